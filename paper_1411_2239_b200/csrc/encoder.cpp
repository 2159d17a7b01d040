// encoder.cpp -- host trace encoder: JSON-lines key -> value records to the
// encoded batch layout of ltl4c_batch (include/ltl4c.h).
//
// arXiv:1411.2239 §4.1 "Valuation Extraction": "the trace event is a
// key-value structure"; epsilon(u_i, K) returns the values of the quantified
// keys K.  Def. 1/2: an event is a set of (interpreted) predicates.
// Readings (A12, A25-A27):
//   * guard key p_i of quantifier level i: the event's value of key p_i (a JSON
//     string or number) is its value for x_i; values are identified by their
//     canonical string (strings as written, numbers as canonical decimals,
//     so 12, 12.0, 1.2e1 and "12" are one value); booleans, null, arrays and
//     objects bind no value (the event binds no vector at that level);
//   * 0-ary atom q: holds iff the record maps q to true;
//   * parametric atom q(x_i, ...): holds iff the record maps q to true (the
//     event's own guard values) or binds q to exactly the event's own value of
//     x_i (a scalar for one argument, an array of scalars in argument order for
//     several) -- P:926-932, reading A12;
//   * other keys are ignored.
// Each level keeps one dictionary canonical string -> dense id (0, 1, 2, ... in
// order of first appearance) for the encoder's lifetime, so the batches of an
// online stream share ids.
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>
#include <unordered_map>
#include <vector>

#include "program.h"

struct ltl4c_encoder {
  const ltl4c_program *prog = nullptr;
  std::vector<std::unordered_map<std::string, uint32_t>> dict;  // per level
  struct Atom {
    std::string pred;
    std::vector<int> levels;
  };
  std::vector<Atom> atoms;
  uint64_t line = 0;  // records read so far (error messages)
};

namespace ltl4c {
namespace {

// A parsed JSON value, reduced to what the encoder reads.
struct Val {
  enum Kind { kNone, kTrue, kFalse, kNull, kScalar, kArray, kObject } kind = kNone;
  std::string canon;                 // kScalar: canonical string
  std::vector<std::string> items;    // kArray: canonical strings of scalar items ("\x01" = non-scalar)
};

struct Parser {
  const char *p, *end;
  std::string err;

  void ws() {
    while (p < end && (*p == ' ' || *p == '\t' || *p == '\r')) ++p;
  }
  bool fail(const char *m) {
    if (err.empty()) err = m;
    return false;
  }
  static void put_utf8(std::string &o, uint32_t c) {
    if (c < 0x80) o += (char)c;
    else if (c < 0x800) { o += (char)(0xC0 | (c >> 6)); o += (char)(0x80 | (c & 63)); }
    else if (c < 0x10000) { o += (char)(0xE0 | (c >> 12)); o += (char)(0x80 | ((c >> 6) & 63)); o += (char)(0x80 | (c & 63)); }
    else { o += (char)(0xF0 | (c >> 18)); o += (char)(0x80 | ((c >> 12) & 63)); o += (char)(0x80 | ((c >> 6) & 63)); o += (char)(0x80 | (c & 63)); }
  }
  bool hex4(uint32_t *v) {
    if (end - p < 4) return fail("truncated \\u escape");
    *v = 0;
    for (int i = 0; i < 4; ++i) {
      const char c = p[i];
      *v <<= 4;
      if (c >= '0' && c <= '9') *v |= (uint32_t)(c - '0');
      else if (c >= 'a' && c <= 'f') *v |= (uint32_t)(c - 'a' + 10);
      else if (c >= 'A' && c <= 'F') *v |= (uint32_t)(c - 'A' + 10);
      else return fail("bad \\u escape");
    }
    p += 4;
    return true;
  }
  bool str(std::string &o) {  // at '"'
    ++p;
    o.clear();
    while (p < end && *p != '"') {
      if (*p == '\n') return fail("newline inside a string");
      if (*p != '\\') { o += *p++; continue; }
      if (++p >= end) return fail("truncated escape");
      const char e = *p++;
      switch (e) {
        case '"': o += '"'; break;
        case '\\': o += '\\'; break;
        case '/': o += '/'; break;
        case 'b': o += '\b'; break;
        case 'f': o += '\f'; break;
        case 'n': o += '\n'; break;
        case 'r': o += '\r'; break;
        case 't': o += '\t'; break;
        case 'u': {
          uint32_t c;
          if (!hex4(&c)) return false;
          if (c >= 0xD800 && c < 0xDC00 && end - p >= 6 && p[0] == '\\' && p[1] == 'u') {
            p += 2;
            uint32_t lo;
            if (!hex4(&lo)) return false;
            if (lo >= 0xDC00 && lo < 0xE000) c = 0x10000 + ((c - 0xD800) << 10) + (lo - 0xDC00);
            else { put_utf8(o, c); c = lo; }
          }
          put_utf8(o, c);
          break;
        }
        default: return fail("bad escape");
      }
    }
    if (p >= end) return fail("unterminated string");
    ++p;
    return true;
  }
  // JSON number -> canonical decimal string (value identity: 12 == 12.0 == 1.2e1)
  bool num(std::string &o) {
    const char *s = p;
    bool neg = false;
    if (p < end && *p == '-') { neg = true; ++p; }
    std::string digits;
    long point = 0;
    if (p >= end || !(*p >= '0' && *p <= '9')) return fail("bad number");
    while (p < end && *p >= '0' && *p <= '9') { digits += *p++; ++point; }
    if (p < end && *p == '.') {
      ++p;
      if (p >= end || !(*p >= '0' && *p <= '9')) return fail("bad number");
      while (p < end && *p >= '0' && *p <= '9') digits += *p++;
    }
    if (p < end && (*p == 'e' || *p == 'E')) {
      ++p;
      bool eneg = false;
      if (p < end && (*p == '+' || *p == '-')) eneg = *p++ == '-';
      if (p >= end || !(*p >= '0' && *p <= '9')) return fail("bad number");
      long e = 0;
      while (p < end && *p >= '0' && *p <= '9') {
        e = e * 10 + (*p++ - '0');
        if (e > 4096) return fail("number exponent out of range");
      }
      point += eneg ? -e : e;
    }
    (void)s;
    // strip leading zeros (moving the point) and trailing zeros
    size_t lz = 0;
    while (lz < digits.size() && digits[lz] == '0') ++lz;
    digits.erase(0, lz);
    point -= (long)lz;
    while (!digits.empty() && digits.back() == '0') digits.pop_back();
    if (digits.empty()) { o = "0"; return true; }
    o.clear();
    if (neg) o += '-';
    const long nd = (long)digits.size();
    if (point <= 0) { o += "0."; o.append((size_t)(-point), '0'); o += digits; }
    else if (point >= nd) { o += digits; o.append((size_t)(point - nd), '0'); }
    else { o += digits.substr(0, (size_t)point); o += '.'; o += digits.substr((size_t)point); }
    return true;
  }
  bool lit(const char *w) {
    const size_t n = std::strlen(w);
    if ((size_t)(end - p) < n || std::memcmp(p, w, n) != 0) return fail("bad literal");
    p += n;
    return true;
  }
  // any value; depth-limited; scalars and arrays of scalars are kept
  bool value(Val &v, int depth) {
    ws();
    if (p >= end) return fail("missing value");
    if (depth > 64) return fail("nesting too deep");
    const char c = *p;
    if (c == '"') { v.kind = Val::kScalar; return str(v.canon); }
    if (c == '-' || (c >= '0' && c <= '9')) { v.kind = Val::kScalar; return num(v.canon); }
    if (c == 't') { v.kind = Val::kTrue; return lit("true"); }
    if (c == 'f') { v.kind = Val::kFalse; return lit("false"); }
    if (c == 'n') { v.kind = Val::kNull; return lit("null"); }
    if (c == '[') {
      ++p;
      v.kind = Val::kArray;
      ws();
      if (p < end && *p == ']') { ++p; return true; }
      while (true) {
        Val it;
        if (!value(it, depth + 1)) return false;
        v.items.push_back(it.kind == Val::kScalar ? it.canon : std::string("\x01", 1));
        ws();
        if (p < end && *p == ',') { ++p; continue; }
        if (p < end && *p == ']') { ++p; return true; }
        return fail("expected ',' or ']'");
      }
    }
    if (c == '{') {
      v.kind = Val::kObject;
      return object(nullptr, depth + 1);
    }
    return fail("unexpected character");
  }
  // object at '{'; calls on(key, value) for every member (on == nullptr: skip)
  template <class F>
  bool object_with(F &&on, int depth) {
    ws();
    if (p >= end || *p != '{') return fail("a record must be a JSON object");
    ++p;
    ws();
    if (p < end && *p == '}') { ++p; return true; }
    std::string key;
    while (true) {
      ws();
      if (p >= end || *p != '"') return fail("expected a string key");
      if (!str(key)) return false;
      ws();
      if (p >= end || *p != ':') return fail("expected ':'");
      ++p;
      Val v;
      if (!value(v, depth)) return false;
      on(key, v);
      ws();
      if (p < end && *p == ',') { ++p; continue; }
      if (p < end && *p == '}') { ++p; return true; }
      return fail("expected ',' or '}'");
    }
  }
  bool object(void *, int depth) {
    return object_with([](const std::string &, const Val &) {}, depth);
  }
};

}  // namespace
}  // namespace ltl4c

using namespace ltl4c;

extern "C" {

ltl4c_status ltl4c_encoder_create(const ltl4c_program *prog, ltl4c_encoder **out) {
  if (!prog || !out) return fail(LTL4C_E_INVALID, "null argument");
  auto *e = new ltl4c_encoder();
  e->prog = prog;
  e->dict.resize(prog->n_levels);
  for (uint32_t j = 0; j < prog->n_atoms; ++j) {
    const std::string &nm = prog->atom_names[j];
    ltl4c_encoder::Atom a;
    a.pred = nm.substr(0, nm.find('('));
    a.levels = j < prog->atom_levels.size() ? prog->atom_levels[j] : std::vector<int>();
    e->atoms.push_back(a);
  }
  *out = e;
  return LTL4C_OK;
}

void ltl4c_encoder_free(ltl4c_encoder *enc) { delete enc; }

ltl4c_status ltl4c_encoder_values(const ltl4c_encoder *enc, uint32_t level, uint64_t *count) {
  if (!enc || !count) return fail(LTL4C_E_INVALID, "null argument");
  if (level >= enc->dict.size()) return fail(LTL4C_E_INVALID, "level out of range");
  *count = enc->dict[level].size();
  return LTL4C_OK;
}

ltl4c_status ltl4c_encode_jsonl(ltl4c_encoder *enc, const char *text, uint64_t len, uint32_t *const *keys,
                                uint8_t *letters, uint64_t capacity, uint64_t *n_events, uint64_t *consumed) {
  if (!enc || !n_events || !consumed || (len && !text)) return fail(LTL4C_E_INVALID, "null argument");
  const int K = (int)enc->prog->n_levels;
  if (capacity && (!letters || !keys)) return fail(LTL4C_E_INVALID, "null output buffer");
  for (int l = 0; l < K && capacity; ++l)
    if (!keys[l]) return fail(LTL4C_E_INVALID, "null key buffer");
  *n_events = 0;
  *consumed = 0;
  const char *p = text, *end = text + len;
  uint64_t n = 0;
  std::vector<const Val *> guard(K);
  std::vector<std::pair<std::string, Val>> rec;
  while (p < end && n < capacity) {
    const char *nl = (const char *)std::memchr(p, '\n', (size_t)(end - p));
    const char *le = nl ? nl : end;
    const char *q = p;
    while (q < le && (*q == ' ' || *q == '\t' || *q == '\r')) ++q;
    if (q == le) {  // blank line
      p = nl ? nl + 1 : end;
      continue;
    }
    enc->line++;
    Parser ps{q, le, {}};
    rec.clear();
    bool ok = ps.object_with([&](const std::string &k, const Val &v) { rec.emplace_back(k, v); }, 0);
    ps.ws();
    if (ok && ps.p != le) ok = ps.fail("trailing characters after the record");
    if (!ok)
      return fail(LTL4C_E_SYNTAX, "record " + std::to_string(enc->line) + ": " + ps.err);
    // a repeated key: the last occurrence wins (one value per key, reading A11)
    auto find = [&](const std::string &k) -> const Val * {
      const Val *r = nullptr;
      for (auto &kv : rec)
        if (kv.first == k) r = &kv.second;
      return r;
    };
    for (int l = 0; l < K; ++l) {
      const Val *v = find(enc->prog->key_names[l]);
      guard[l] = v && v->kind == Val::kScalar ? v : nullptr;
      uint32_t id = LTL4C_ABSENT;
      if (guard[l]) {
        auto &d = enc->dict[l];
        auto it = d.find(v->canon);
        if (it == d.end()) {
          if (d.size() >= 0xFFFFFFFFull) return fail(LTL4C_E_BUDGET, "more than 2^32 - 1 values of one key");
          it = d.emplace(v->canon, (uint32_t)d.size()).first;
        }
        id = it->second;
      }
      keys[l][n] = id;
    }
    uint32_t let = 0;  // the atom valuation; its letter code below
    for (size_t j = 0; j < enc->atoms.size(); ++j) {
      const auto &a = enc->atoms[j];
      const Val *v = find(a.pred);
      if (!v) continue;
      bool holds = v->kind == Val::kTrue;
      if (!holds && !a.levels.empty()) {
        if (a.levels.size() == 1 && v->kind == Val::kScalar) {
          const Val *g = guard[a.levels[0]];
          holds = g && g->canon == v->canon;
        } else if (v->kind == Val::kArray && v->items.size() == a.levels.size()) {
          holds = true;
          for (size_t i = 0; i < a.levels.size() && holds; ++i) {
            const Val *g = guard[a.levels[i]];
            holds = g && g->canon == v->items[i];
          }
        }
      }
      if (holds) let |= 1u << j;
    }
    letters[n] = enc->prog->letter_class.empty() ? (uint8_t)let : enc->prog->letter_class[let];
    ++n;
    p = nl ? nl + 1 : end;
  }
  *n_events = n;
  *consumed = (uint64_t)(p - text);
  return LTL4C_OK;
}

}  // extern "C"
