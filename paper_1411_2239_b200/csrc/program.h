// program.h -- internal definition of ltl4c_program (host side) shared by the
// compiler (compiler.cpp) and the runtime (runtime.cu).
#pragma once
#include <string>
#include <vector>

#include "../../include/ltl4c.h"

struct ltl4c_program {
  uint32_t n_formulas = 0, n_levels = 0, n_atoms = 0, n_states = 0, initial = 0;
  uint32_t letter_bits = 0;               // codes < 1 << letter_bits (= n_atoms up to 8 atoms)
  std::vector<uint8_t> letter_class;      // [1 << n_atoms] code of each valuation (> 8 atoms), else empty
  std::vector<uint8_t> delta;             // [n_states][1 << letter_bits]
  std::vector<uint8_t> label;             // [n_formulas][n_states], B6 codes {0,2,3,5}
  std::vector<ltl4c_quantifier> quant;    // [n_formulas][n_levels]
  std::vector<std::string> atom_names;    // [n_atoms]
  std::vector<std::vector<int>> atom_levels;  // [n_atoms]: quantifier level of each argument
  std::vector<const char *> atom_ptrs;    // views into atom_names
  std::vector<std::string> key_names;     // [n_levels]
  std::vector<std::string> texts;         // source formulas
};

namespace ltl4c {
// thread-local error message plumbing (runtime.cu owns the storage)
ltl4c_status fail(ltl4c_status st, const std::string &msg);
}
