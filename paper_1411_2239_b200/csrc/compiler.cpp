// compiler.cpp -- host formula compiler: LTL4-C text -> LTL4 monitor tables.
//
// arXiv:1411.2239: syntax Def. 3, canonical form Eq. 4/5
// (P:459-474), LTL4 semantics Def. 4, LTL4 monitor Def. 5
// (P:326-336).  The paper synthesises monitors with the construction of
// [bls10-jlc] without giving it; this compiler uses its own
// construction:
//
//  1. states are residual obligations after a prefix u: a Boolean function
//     S_u over variables N(chi) ("there is a next position and chi holds
//     there"), chi ranging over the X-arguments and U-subformulas of psi.
//     S_{ua} = S_u[N(chi) := P(chi, a)], P the one-step expansion
//       P(p,a) = [p in a], P(Xf,a) = N(f), P(f U g,a) = P(g,a) | (P(f,a) & N(f U g)).
//     Boolean functions are truth tables over the <= 12 variables, so states are
//     canonical and finite.
//  2. the FLTL value [u |=_F psi] is S_u with every N(.) false
//     (strong next: there is no next position after u);
//  3. "forall v: uv |= psi" is S_u(tau) = 1 for every type tau realisable by an
//     infinite word; realisable types are computed on the type graph
//     (tau = sub_a(tau')) as the nodes that reach a fair SCC (every U-obligation
//     claimed in the SCC is either dropped or fulfilled inside it);
//  4. lambda(S) = T if valid on realisable types, F if unsatisfiable, else
//     Tp / Fp by the FLTL value (Def. 4); Moore minimisation; traps merge.
//
// Shares no code with oracle/ (which uses a different parser and the textbook
// atom tableau with per-run subset tracking).
#include <algorithm>
#include <cctype>
#include <cstring>
#include <map>
#include <queue>
#include <set>
#include <string>
#include <tuple>
#include <vector>

#include "program.h"

namespace ltl4c {
namespace {

// ----------------------------------------------------------------- lexer
enum class Tk { End, Ident, Number, Percent, LBrack, RBrack, LParen, RParen, Comma, Colon,
                Guard /* => */, Arrow /* -> */, And, Or, Not, Lt, Le, Gt, Ge, Eq, Minus, Bad };

struct Token {
  Tk k;
  std::string s;
  size_t at;
};

std::vector<Token> lex(const std::string &src) {
  std::vector<Token> out;
  size_t i = 0, n = src.size();
  while (true) {
    while (i < n) {
      if (std::isspace((unsigned char)src[i])) { ++i; continue; }
      if (src[i] == '#') { while (i < n && src[i] != '\n') ++i; continue; }
      break;
    }
    if (i >= n) { out.push_back({Tk::End, "", i}); return out; }
    size_t at = i;
    char c = src[i];
    if (std::isalpha((unsigned char)c) || c == '_') {
      size_t j = i;
      while (j < n && (std::isalnum((unsigned char)src[j]) || src[j] == '_')) ++j;
      out.push_back({Tk::Ident, src.substr(i, j - i), at});
      i = j;
      continue;
    }
    if (std::isdigit((unsigned char)c) || (c == '.' && i + 1 < n && std::isdigit((unsigned char)src[i + 1]))) {
      size_t j = i;
      while (j < n && (std::isdigit((unsigned char)src[j]) || src[j] == '.')) ++j;
      out.push_back({Tk::Number, src.substr(i, j - i), at});
      i = j;
      continue;
    }
    auto two = [&](char a, char b) { return c == a && i + 1 < n && src[i + 1] == b; };
    Tk k;
    size_t w = 1;
    if (two('=', '>')) { k = Tk::Guard; w = 2; }
    else if (two('-', '>')) { k = Tk::Arrow; w = 2; }
    else if (two('&', '&')) { k = Tk::And; w = 2; }
    else if (two('|', '|')) { k = Tk::Or; w = 2; }
    else if (two('<', '=')) { k = Tk::Le; w = 2; }
    else if (two('>', '=')) { k = Tk::Ge; w = 2; }
    else if (two('=', '=')) { k = Tk::Eq; w = 2; }
    else switch (c) {
      case '%': k = Tk::Percent; break;
      case '[': k = Tk::LBrack; break;
      case ']': k = Tk::RBrack; break;
      case '(': k = Tk::LParen; break;
      case ')': k = Tk::RParen; break;
      case ',': k = Tk::Comma; break;
      case ':': k = Tk::Colon; break;
      case '&': k = Tk::And; break;
      case '|': k = Tk::Or; break;
      case '!': case '~': k = Tk::Not; break;
      case '<': k = Tk::Lt; break;
      case '>': k = Tk::Gt; break;
      case '=': k = Tk::Eq; break;
      case '-': k = Tk::Minus; break;
      default: k = Tk::Bad; break;
    }
    out.push_back({k, src.substr(i, w), at});
    i += w;
  }
}

// ----------------------------------------------------------------- AST
enum Op { kTrue, kAtom, kNot, kAnd, kNext, kUntil };
struct Node {
  Op op;
  int a, b, atom;
};

struct Quant {
  int kind, cmp;
  uint64_t num, den;
  std::string var, key;
};

struct Formula {
  std::vector<Quant> q;
  std::vector<Node> nodes;
  std::map<std::tuple<int, int, int, int>, int> intern;
  std::vector<std::string> atoms;
  std::vector<std::vector<int>> atom_levels;  // per atom: quantifier level of each argument
  int root = -1;

  int make(Op op, int a = -1, int b = -1, int atom = -1) {
    auto key = std::make_tuple((int)op, a, b, atom);
    auto it = intern.find(key);
    if (it != intern.end()) return it->second;
    nodes.push_back({op, a, b, atom});
    intern[key] = (int)nodes.size() - 1;
    return (int)nodes.size() - 1;
  }
};

struct ParseError {
  ltl4c_status st;
  std::string msg;
};

// ----------------------------------------------------------------- parser
class Parser {
 public:
  explicit Parser(const std::string &text) : toks_(lex(text)) {}

  Formula run() {
    int wrap = 0;
    while (true) {
      // parentheses that enclose a nested quantifier (P:699 writes them)
      size_t k = pos_;
      while (toks_[k].k == Tk::LParen) ++k;
      if (k > pos_ && is_quant(toks_[k])) { wrap += (int)(k - pos_); pos_ = k; }
      if (!is_quant(cur())) break;
      quantifier();
    }
    f_.root = implication();
    for (int i = 0; i < wrap; ++i) expect(Tk::RParen, "expected ')'");
    if (is_quant(cur())) throw ParseError{LTL4C_E_NONCANONICAL, "quantifier after the body"};
    if (cur().k != Tk::End) err(LTL4C_E_SYNTAX, "trailing input");
    return std::move(f_);
  }

 private:
  std::vector<Token> toks_;
  size_t pos_ = 0;
  Formula f_;

  const Token &cur() const { return toks_[pos_]; }
  bool is_word(const Token &t, const char *w) const { return t.k == Tk::Ident && t.s == w; }
  bool is_quant(const Token &t) const { return is_word(t, "forall") || is_word(t, "exists"); }
  [[noreturn]] void err(ltl4c_status st, const std::string &m) {
    throw ParseError{st, m + " at offset " + std::to_string(cur().at)};
  }
  void expect(Tk k, const char *m) {
    if (cur().k != k) err(LTL4C_E_SYNTAX, m);
    ++pos_;
  }
  std::string ident(const char *m) {
    if (cur().k != Tk::Ident) err(LTL4C_E_SYNTAX, m);
    return toks_[pos_++].s;
  }

  void quantifier() {
    if (f_.q.size() >= LTL4C_MAX_LEVELS) err(LTL4C_E_BUDGET, "more than 3 quantifiers");
    Quant q{};
    q.kind = is_word(cur(), "forall") ? LTL4C_QUANT_A : LTL4C_QUANT_E;
    ++pos_;
    // default constraints: A == A_{=1}, E == E_{>=1}
    if (q.kind == LTL4C_QUANT_A) { q.cmp = LTL4C_EQ; q.num = 1; q.den = 1; }
    else { q.cmp = LTL4C_GE; q.num = 1; q.den = 1; }
    if (cur().k == Tk::LBrack) constraint(q);
    q.var = ident("expected the bound variable");
    for (auto &o : f_.q)
      if (o.var == q.var) err(LTL4C_E_SYNTAX, "variable bound twice");
    expect(Tk::Colon, "expected ':'");
    q.key = ident("expected the guard predicate");
    expect(Tk::LParen, "expected '('");
    if (cur().k != Tk::Ident) err(LTL4C_E_SYNTAX, "expected the guard variable");
    if (cur().s != q.var) err(LTL4C_E_UNBOUND, "guard variable differs from the bound variable");
    ++pos_;
    expect(Tk::RParen, "expected ')'");
    expect(Tk::Guard, "expected '=>'");
    f_.q.push_back(q);
  }

  // "[" cmp ["-"] number ["%"] "]"   (readings A5, A6)
  void constraint(Quant &q) {
    ++pos_;
    switch (cur().k) {
      case Tk::Lt: q.cmp = LTL4C_LT; break;
      case Tk::Le: q.cmp = LTL4C_LE; break;
      case Tk::Gt: q.cmp = LTL4C_GT; break;
      case Tk::Ge: q.cmp = LTL4C_GE; break;
      case Tk::Eq: q.cmp = LTL4C_EQ; break;
      default: err(LTL4C_E_SYNTAX, "expected a comparison operator");
    }
    ++pos_;
    bool negative = false;
    if (cur().k == Tk::Minus) { negative = true; ++pos_; }
    if (cur().k != Tk::Number) err(LTL4C_E_SYNTAX, "expected a number");
    std::string lit = toks_[pos_++].s;
    bool pct = false;
    if (cur().k == Tk::Percent) { pct = true; ++pos_; }
    expect(Tk::RBrack, "expected ']'");
    size_t dot = lit.find('.');
    if (dot != std::string::npos && lit.find('.', dot + 1) != std::string::npos)
      err(LTL4C_E_SYNTAX, "malformed number");
    std::string digits;
    int frac = 0;
    for (size_t i = 0; i < lit.size(); ++i) {
      if (lit[i] == '.') continue;
      digits.push_back(lit[i]);
      if (dot != std::string::npos && i > dot) ++frac;
    }
    if (digits.size() > 18) err(LTL4C_E_RANGE, "constant has too many digits");
    uint64_t m = 0;
    for (char d : digits) m = m * 10 + (uint64_t)(d - '0');
    if (negative && m != 0) err(LTL4C_E_RANGE, "negative constant");
    if (q.kind == LTL4C_QUANT_E) {
      if (pct || frac > 0) err(LTL4C_E_RANGE, "E constant must be an integer");
      if (m > (1ull << 40)) err(LTL4C_E_RANGE, "E constant too large");
      q.num = m;
      q.den = 1;
      return;
    }
    if ((!pct && frac > 6) || (pct && frac > 4)) err(LTL4C_E_RANGE, "A constant has too many decimals");
    uint64_t den = 1;
    for (int i = 0; i < frac; ++i) den *= 10;
    if (pct) den *= 100;
    if (m > den) err(LTL4C_E_RANGE, "A constant outside [0,1]");
    uint64_t a = m, b = den;
    while (b) { uint64_t t = a % b; a = b; b = t; }
    uint64_t g = a ? a : den;
    q.num = m / g;
    q.den = den / g;
  }

  // derived operators (P:288 and Boolean identities)
  int mk_not(int a) { return f_.make(kNot, a); }
  int mk_or(int a, int b) { return mk_not(f_.make(kAnd, mk_not(a), mk_not(b))); }
  int mk_F(int a) { return f_.make(kUntil, f_.make(kTrue), a); }

  int implication() {
    int a = disjunction();
    if (cur().k == Tk::Arrow) {
      ++pos_;
      int b = implication();
      return mk_or(mk_not(a), b);
    }
    return a;
  }
  int disjunction() {
    int a = conjunction();
    while (cur().k == Tk::Or) { ++pos_; a = mk_or(a, conjunction()); }
    return a;
  }
  int conjunction() {
    int a = until();
    while (cur().k == Tk::And) { ++pos_; a = f_.make(kAnd, a, until()); }
    return a;
  }
  int until() {
    int a = unary();
    if (is_word(cur(), "U")) { ++pos_; return f_.make(kUntil, a, until()); }
    return a;
  }
  int unary() {
    if (cur().k == Tk::Not) { ++pos_; return mk_not(unary()); }
    if (is_word(cur(), "X")) { ++pos_; return f_.make(kNext, unary()); }
    if (is_word(cur(), "F")) { ++pos_; return mk_F(unary()); }
    if (is_word(cur(), "G")) { ++pos_; return mk_not(mk_F(mk_not(unary()))); }
    return primary();
  }
  int primary() {
    if (cur().k == Tk::LParen) {
      ++pos_;
      int r = implication();
      expect(Tk::RParen, "expected ')'");
      return r;
    }
    if (cur().k != Tk::Ident) err(LTL4C_E_SYNTAX, "expected a proposition");
    if (is_quant(cur())) err(LTL4C_E_NONCANONICAL, "quantifier inside the quantifier-free body");
    if (is_word(cur(), "true")) { ++pos_; return f_.make(kTrue); }
    if (is_word(cur(), "false")) { ++pos_; return mk_not(f_.make(kTrue)); }
    if (is_word(cur(), "U")) err(LTL4C_E_SYNTAX, "unexpected U");
    std::string name = toks_[pos_++].s;
    std::vector<int> levels;
    if (cur().k == Tk::LParen) {
      ++pos_;
      name += "(";
      bool first = true;
      while (true) {
        if (cur().k != Tk::Ident) err(LTL4C_E_SYNTAX, "expected a variable");
        bool bound = false;
        for (size_t l = 0; l < f_.q.size(); ++l)
          if (f_.q[l].var == cur().s) { bound = true; levels.push_back((int)l); }
        if (!bound) err(LTL4C_E_UNBOUND, "unbound variable '" + cur().s + "'");
        name += (first ? "" : ",") + cur().s;
        first = false;
        ++pos_;
        if (cur().k == Tk::Comma) { ++pos_; continue; }
        expect(Tk::RParen, "expected ',' or ')'");
        break;
      }
      name += ")";
    }
    auto it = std::find(f_.atoms.begin(), f_.atoms.end(), name);
    int j = (int)(it - f_.atoms.begin());
    if (it == f_.atoms.end()) {
      if (f_.atoms.size() >= LTL4C_MAX_ATOMS) err(LTL4C_E_BUDGET, "more than 8 atoms");
      f_.atoms.push_back(name);
      f_.atom_levels.push_back(levels);
    }
    return f_.make(kAtom, -1, -1, j);
  }
};

// ------------------------------------------------------ Boolean truth tables
constexpr int kMaxVars = 12;

struct TT {  // truth table over V variables, bit s = value at assignment s
  std::vector<uint64_t> w;
  bool operator<(const TT &o) const { return w < o.w; }
  bool operator==(const TT &o) const { return w == o.w; }
  bool get(uint32_t s) const { return (w[s >> 6] >> (s & 63)) & 1; }
};

struct TTSpace {
  int V;
  uint32_t size;  // 2^V
  int nw;
  uint64_t tail;  // mask of the valid bits of the last word
  explicit TTSpace(int v) : V(v), size(1u << v), nw(v >= 6 ? (1 << (v - 6)) : 1) {
    tail = v >= 6 ? ~0ull : ((1ull << (1u << v)) - 1ull);
  }
  TT constant(bool b) const {
    TT t;
    t.w.assign(nw, b ? ~0ull : 0ull);
    t.w.back() &= tail;
    if (V >= 6 && b) t.w.back() = ~0ull;
    return t;
  }
  TT var(int i) const {
    TT t = constant(false);
    for (uint32_t s = 0; s < size; ++s)
      if ((s >> i) & 1) t.w[s >> 6] |= 1ull << (s & 63);
    return t;
  }
  TT neg(const TT &a) const {
    TT t = a;
    for (auto &x : t.w) x = ~x;
    t.w.back() &= tail;
    return t;
  }
  TT conj(const TT &a, const TT &b) const {
    TT t = a;
    for (int i = 0; i < nw; ++i) t.w[i] &= b.w[i];
    return t;
  }
  TT disj(const TT &a, const TT &b) const {
    TT t = a;
    for (int i = 0; i < nw; ++i) t.w[i] |= b.w[i];
    return t;
  }
};

struct Dfa {
  int Q = 0, A = 0;          // states, letters (2^atoms)
  int initial = 0;
  std::vector<int> delta;    // Q * A
  std::vector<uint8_t> lab;  // Q (B6 codes)
};

// Moore minimisation w.r.t. a label signature per state; renumbers states in
// BFS order from the initial state (so the initial state is 0).
template <class Sig>
Dfa minimise(const Dfa &d, const std::vector<Sig> &sig, std::vector<Sig> *sig_out) {
  int Q = d.Q, A = d.A;
  std::vector<int> cls(Q);
  {
    std::map<Sig, int> m;
    for (int q = 0; q < Q; ++q) {
      auto it = m.find(sig[q]);
      if (it == m.end()) it = m.emplace(sig[q], (int)m.size()).first;
      cls[q] = it->second;
    }
  }
  while (true) {
    std::map<std::vector<int>, int> m;
    std::vector<int> nc(Q);
    for (int q = 0; q < Q; ++q) {
      std::vector<int> key;
      key.reserve(A + 1);
      key.push_back(cls[q]);
      for (int a = 0; a < A; ++a) key.push_back(cls[d.delta[q * A + a]]);
      auto it = m.find(key);
      if (it == m.end()) it = m.emplace(key, (int)m.size()).first;
      nc[q] = it->second;
    }
    bool same = true;
    int ncls = (int)m.size();
    int ocls = *std::max_element(cls.begin(), cls.end()) + 1;
    if (ncls != ocls) same = false;
    cls = nc;
    if (same) break;
  }
  // representative per class and BFS renumbering
  int C = *std::max_element(cls.begin(), cls.end()) + 1;
  std::vector<int> rep(C, -1);
  for (int q = 0; q < Q; ++q) if (rep[cls[q]] < 0) rep[cls[q]] = q;
  std::vector<int> order(C, -1);
  std::vector<int> bfs;
  std::queue<int> qu;
  order[cls[d.initial]] = 0;
  bfs.push_back(cls[d.initial]);
  qu.push(cls[d.initial]);
  while (!qu.empty()) {
    int c = qu.front();
    qu.pop();
    for (int a = 0; a < A; ++a) {
      int c2 = cls[d.delta[rep[c] * A + a]];
      if (order[c2] < 0) { order[c2] = (int)bfs.size(); bfs.push_back(c2); qu.push(c2); }
    }
  }
  Dfa out;
  out.Q = (int)bfs.size();
  out.A = A;
  out.initial = 0;
  out.delta.resize((size_t)out.Q * A);
  out.lab.resize(out.Q);
  if (sig_out) sig_out->resize(out.Q);
  for (int i = 0; i < out.Q; ++i) {
    int q = rep[bfs[i]];
    out.lab[i] = d.lab[q];
    if (sig_out) (*sig_out)[i] = sig[q];
    for (int a = 0; a < A; ++a) out.delta[i * A + a] = order[cls[d.delta[q * A + a]]];
  }
  return out;
}

// ----------------------------------------------------------- synthesis
Dfa synthesise(const Formula &f) {
  const int nAtoms = (int)f.atoms.size();
  const int A = 1 << nAtoms;
  // obligation variables: root, X-arguments, U-subformulas
  std::vector<int> var_of(f.nodes.size(), -1);
  std::vector<int> vars;
  auto add_var = [&](int node) {
    if (var_of[node] < 0) { var_of[node] = (int)vars.size(); vars.push_back(node); }
  };
  add_var(f.root);
  for (size_t i = 0; i < f.nodes.size(); ++i) {
    if (f.nodes[i].op == kNext) add_var(f.nodes[i].a);
    if (f.nodes[i].op == kUntil) add_var((int)i);
  }
  const int V = (int)vars.size();
  if (V > kMaxVars) throw ParseError{LTL4C_E_BUDGET, "formula has more than 12 temporal obligations"};
  TTSpace sp(V);

  // P(node, a) for every node and letter (children precede parents in `nodes`)
  std::vector<std::vector<TT>> P(A, std::vector<TT>(f.nodes.size()));
  for (int a = 0; a < A; ++a) {
    for (size_t i = 0; i < f.nodes.size(); ++i) {
      const Node &n = f.nodes[i];
      switch (n.op) {
        case kTrue: P[a][i] = sp.constant(true); break;
        case kAtom: P[a][i] = sp.constant((a >> n.atom) & 1); break;
        case kNot: P[a][i] = sp.neg(P[a][n.a]); break;
        case kAnd: P[a][i] = sp.conj(P[a][n.a], P[a][n.b]); break;
        case kNext: P[a][i] = sp.var(var_of[n.a]); break;
        case kUntil:
          P[a][i] = sp.disj(P[a][n.b], sp.conj(P[a][n.a], sp.var(var_of[i])));
          break;
      }
    }
  }
  // sub[a][s'] = assignment of the current position from letter a and next type s'
  std::vector<std::vector<uint32_t>> sub(A, std::vector<uint32_t>(sp.size));
  for (int a = 0; a < A; ++a)
    for (uint32_t s = 0; s < sp.size; ++s) {
      uint32_t t = 0;
      for (int v = 0; v < V; ++v) if (P[a][vars[v]].get(s)) t |= 1u << v;
      sub[a][s] = t;
    }

  // --- realisable types: nodes of the type graph that reach a fair SCC
  const uint32_t T = sp.size;
  std::vector<std::vector<std::pair<uint32_t, int>>> out(T);  // tau -> (tau', a)
  for (int a = 0; a < A; ++a)
    for (uint32_t s = 0; s < T; ++s) out[sub[a][s]].push_back({s, a});
  std::vector<int> idx(T, -1), low(T, 0), comp(T, -1), stk;
  std::vector<char> on(T, 0);
  int counter = 0, ncomp = 0;
  for (uint32_t root = 0; root < T; ++root) {
    if (idx[root] >= 0) continue;
    std::vector<std::pair<uint32_t, size_t>> cs{{root, 0}};
    idx[root] = low[root] = counter++;
    stk.push_back(root);
    on[root] = 1;
    while (!cs.empty()) {
      uint32_t v = cs.back().first;
      size_t &it = cs.back().second;
      if (it < out[v].size()) {
        uint32_t w = out[v][it++].first;
        if (idx[w] < 0) {
          idx[w] = low[w] = counter++;
          stk.push_back(w);
          on[w] = 1;
          cs.push_back({w, 0});
        } else if (on[w]) {
          low[v] = std::min(low[v], idx[w]);
        }
        continue;
      }
      if (low[v] == idx[v]) {
        while (true) {
          uint32_t w = stk.back();
          stk.pop_back();
          on[w] = 0;
          comp[w] = ncomp;
          if (w == v) break;
        }
        ++ncomp;
      }
      cs.pop_back();
      if (!cs.empty()) low[cs.back().first] = std::min(low[cs.back().first], low[v]);
    }
  }
  std::vector<int> uvars;  // (var index of each U node)
  for (size_t i = 0; i < f.nodes.size(); ++i)
    if (f.nodes[i].op == kUntil) uvars.push_back((int)i);
  std::vector<char> has_edge(ncomp, 0);
  // per comp and U node: dropped somewhere / fulfilled on an inner edge
  std::vector<std::vector<char>> dropped(ncomp, std::vector<char>(uvars.size(), 0));
  std::vector<std::vector<char>> fulfilled(ncomp, std::vector<char>(uvars.size(), 0));
  for (uint32_t t = 0; t < T; ++t) {
    int c = comp[t];
    for (size_t k = 0; k < uvars.size(); ++k)
      if (!((t >> var_of[uvars[k]]) & 1)) dropped[c][k] = 1;
    for (auto &e : out[t]) {
      if (comp[e.first] != c) continue;
      has_edge[c] = 1;
      for (size_t k = 0; k < uvars.size(); ++k)
        if (P[e.second][f.nodes[uvars[k]].b].get(e.first)) fulfilled[c][k] = 1;
    }
  }
  std::vector<char> real(T, 0);
  std::vector<std::vector<uint32_t>> rev(T);
  for (uint32_t t = 0; t < T; ++t)
    for (auto &e : out[t]) rev[e.first].push_back(t);
  std::queue<uint32_t> bq;
  for (uint32_t t = 0; t < T; ++t) {
    int c = comp[t];
    bool fair = has_edge[c];
    for (size_t k = 0; k < uvars.size() && fair; ++k) fair = dropped[c][k] || fulfilled[c][k];
    if (fair) { real[t] = 1; bq.push(t); }
  }
  while (!bq.empty()) {
    uint32_t t = bq.front();
    bq.pop();
    for (uint32_t p : rev[t]) if (!real[p]) { real[p] = 1; bq.push(p); }
  }

  // --- residual DFA by BFS over truth tables
  std::map<TT, int> id;
  std::vector<TT> states;
  std::vector<int> delta;
  TT s0 = sp.var(var_of[f.root]);
  id[s0] = 0;
  states.push_back(s0);
  for (size_t q = 0; q < states.size(); ++q) {
    if (states.size() > 4096) throw ParseError{LTL4C_E_BUDGET, "monitor too large before minimisation"};
    for (int a = 0; a < A; ++a) {
      TT nxt = sp.constant(false);
      const TT &S = states[q];
      for (uint32_t s = 0; s < sp.size; ++s)
        if (S.get(sub[a][s])) nxt.w[s >> 6] |= 1ull << (s & 63);
      auto it = id.find(nxt);
      int to;
      if (it == id.end()) {
        to = (int)states.size();
        id.emplace(nxt, to);
        states.push_back(nxt);
      } else {
        to = it->second;
      }
      delta.push_back(to);
    }
  }
  Dfa d;
  d.Q = (int)states.size();
  d.A = A;
  d.initial = 0;
  d.delta = delta;
  d.lab.resize(d.Q);
  for (int q = 0; q < d.Q; ++q) {
    bool any1 = false, any0 = false;
    for (uint32_t t = 0; t < T; ++t) {
      if (!real[t]) continue;
      if (states[q].get(t)) any1 = true; else any0 = true;
    }
    if (!any0) d.lab[q] = LTL4C_TRUE;
    else if (!any1) d.lab[q] = LTL4C_FALSE;
    else d.lab[q] = states[q].get(0) ? LTL4C_PRESUMABLY_TRUE : LTL4C_PRESUMABLY_FALSE;
  }
  std::vector<int> sig(d.lab.begin(), d.lab.end());
  return minimise(d, sig, (std::vector<int> *)nullptr);
}

Formula parse(const char *text) {
  if (!text) throw ParseError{LTL4C_E_INVALID, "null formula"};
  Parser p{std::string(text)};
  Formula f = p.run();
  if (f.q.empty())
    throw ParseError{LTL4C_E_BUDGET, "a formula needs at least one counting quantifier in this build"};
  return f;
}

}  // namespace

ltl4c_status compile_many(const char *const *texts, int nf, ltl4c_program **out) {
  if (!out) return fail(LTL4C_E_INVALID, "null output pointer");
  *out = nullptr;
  if (!texts || nf < 1 || nf > LTL4C_MAX_FORMULAS)
    return fail(LTL4C_E_INVALID, "need 1..4 formulas");
  try {
    std::vector<Formula> fs;
    std::vector<Dfa> ds;
    for (int i = 0; i < nf; ++i) {
      fs.push_back(parse(texts[i]));
      ds.push_back(synthesise(fs.back()));
    }
    auto prog = new ltl4c_program();
    prog->n_formulas = nf;
    prog->n_levels = (uint32_t)fs[0].q.size();
    for (int i = 1; i < nf; ++i) {
      bool same = fs[i].q.size() == fs[0].q.size();
      for (size_t l = 0; same && l < fs[0].q.size(); ++l) same = fs[i].q[l].key == fs[0].q[l].key;
      if (!same) {
        delete prog;
        return fail(LTL4C_E_INVALID, "formulas of one batch must share the guard-key string");
      }
    }
    // atom union in order of first occurrence
    std::vector<std::vector<int>> gbit(nf);
    for (int i = 0; i < nf; ++i)
      for (size_t j = 0; j < fs[i].atoms.size(); ++j) {
        const std::string &a = fs[i].atoms[j];
        auto it = std::find(prog->atom_names.begin(), prog->atom_names.end(), a);
        if (it == prog->atom_names.end()) {
          prog->atom_names.push_back(a);
          prog->atom_levels.push_back(fs[i].atom_levels[j]);
          gbit[i].push_back((int)prog->atom_names.size() - 1);
        } else {
          const int g = (int)(it - prog->atom_names.begin());
          if (prog->atom_levels[g] != fs[i].atom_levels[j]) {
            delete prog;
            return fail(LTL4C_E_INVALID, "atom " + a + " binds different quantifier levels in the batch");
          }
          gbit[i].push_back(g);
        }
      }
    if (prog->atom_names.size() > LTL4C_MAX_BATCH_ATOMS) {
      delete prog;
      return fail(LTL4C_E_BUDGET, "more than 16 atoms in the formula batch");
    }
    prog->n_atoms = (uint32_t)prog->atom_names.size();
    const int A = 1 << prog->n_atoms;
    auto project = [&](int i, int g) {
      int l = 0;
      for (size_t j = 0; j < gbit[i].size(); ++j) if ((g >> gbit[i][j]) & 1) l |= 1 << j;
      return l;
    };
    // product automaton over tuples of component states
    std::map<std::vector<int>, int> id;
    std::vector<std::vector<int>> tuples;
    Dfa prod;
    prod.A = A;
    std::vector<int> init(nf);
    for (int i = 0; i < nf; ++i) init[i] = ds[i].initial;
    id[init] = 0;
    tuples.push_back(init);
    for (size_t q = 0; q < tuples.size(); ++q) {
      for (int g = 0; g < A; ++g) {
        std::vector<int> nt(nf);
        for (int i = 0; i < nf; ++i) nt[i] = ds[i].delta[tuples[q][i] * ds[i].A + project(i, g)];
        auto it = id.find(nt);
        int to;
        if (it == id.end()) { to = (int)tuples.size(); id.emplace(nt, to); tuples.push_back(nt); }
        else to = it->second;
        prod.delta.push_back(to);
      }
    }
    prod.Q = (int)tuples.size();
    prod.initial = 0;
    prod.lab.assign(prod.Q, 0);
    std::vector<std::vector<uint8_t>> sig(prod.Q, std::vector<uint8_t>(nf));
    for (int q = 0; q < prod.Q; ++q)
      for (int i = 0; i < nf; ++i) sig[q][i] = ds[i].lab[tuples[q][i]];
    std::vector<std::vector<uint8_t>> sig_min;
    Dfa m = minimise(prod, sig, &sig_min);
    if (m.Q > LTL4C_MAX_STATES) {
      delete prog;
      return fail(LTL4C_E_BUDGET, "monitor has " + std::to_string(m.Q) + " states (> 16)");
    }
    prog->n_states = (uint32_t)m.Q;
    prog->initial = (uint32_t)m.initial;
    if (prog->n_atoms <= LTL4C_MAX_ATOMS) {
      prog->letter_bits = prog->n_atoms;
      prog->delta.resize((size_t)m.Q * A);
      for (size_t i = 0; i < prog->delta.size(); ++i) prog->delta[i] = (uint8_t)m.delta[i];
    } else {
      // letter equivalence classes (NEXT-2): valuations whose columns of the minimised
      // product's transition table are equal act identically on every state -- they
      // are one letter to the monitor (lambda depends on the state only)
      std::map<std::vector<int>, int> cls;
      std::vector<std::vector<int>> cols;
      prog->letter_class.resize(A);
      for (int g = 0; g < A; ++g) {
        std::vector<int> col(m.Q);
        for (int q = 0; q < m.Q; ++q) col[q] = m.delta[(size_t)q * A + g];
        auto it = cls.find(col);
        if (it == cls.end()) {
          if (cols.size() >= 256) {
            delete prog;
            return fail(LTL4C_E_BUDGET, "more than 256 letter classes in the formula batch");
          }
          it = cls.emplace(col, (int)cols.size()).first;
          cols.push_back(col);
        }
        prog->letter_class[g] = (uint8_t)it->second;
      }
      int bits = 1;
      while ((1u << bits) < cols.size()) ++bits;
      prog->letter_bits = (uint32_t)bits;
      const int C = 1 << bits;
      prog->delta.resize((size_t)m.Q * C);
      for (int q = 0; q < m.Q; ++q)
        for (int c = 0; c < C; ++c)  // (codes past the classes repeat class 0: never produced)
          prog->delta[(size_t)q * C + c] = (uint8_t)cols[c < (int)cols.size() ? c : 0][q];
    }
    prog->label.resize((size_t)nf * m.Q);
    for (int i = 0; i < nf; ++i)
      for (int q = 0; q < m.Q; ++q) prog->label[i * m.Q + q] = sig_min[q][i];
    for (int i = 0; i < nf; ++i)
      for (auto &q : fs[i].q) {
        ltl4c_quantifier lq{};
        lq.kind = q.kind;
        lq.cmp = q.cmp;
        lq.num = q.num;
        lq.den = q.den;
        std::snprintf(lq.key, sizeof lq.key, "%s", q.key.c_str());
        prog->quant.push_back(lq);
      }
    for (auto &q : fs[0].q) prog->key_names.push_back(q.key);
    for (auto &a : prog->atom_names) prog->atom_ptrs.push_back(a.c_str());
    for (int i = 0; i < nf; ++i) prog->texts.push_back(texts[i]);
    *out = prog;
    return LTL4C_OK;
  } catch (const ParseError &e) {
    return fail(e.st, e.msg);
  } catch (const std::bad_alloc &) {
    return fail(LTL4C_E_BUDGET, "out of host memory while compiling");
  }
}

}  // namespace ltl4c

extern "C" ltl4c_status ltl4c_compile(const char *formula_utf8, ltl4c_program **out) {
  const char *one[1] = {formula_utf8};
  return ltl4c::compile_many(one, 1, out);
}

extern "C" ltl4c_status ltl4c_compile_batch(const char *const *formulas_utf8, int n_formulas,
                                            ltl4c_program **out) {
  return ltl4c::compile_many(formulas_utf8, n_formulas, out);
}

extern "C" ltl4c_status ltl4c_program_tables(const ltl4c_program *prog, ltl4c_tables *view) {
  if (!prog || !view) return ltl4c::fail(LTL4C_E_INVALID, "null argument");
  view->n_formulas = prog->n_formulas;
  view->n_levels = prog->n_levels;
  view->n_atoms = prog->n_atoms;
  view->n_states = prog->n_states;
  view->initial = prog->initial;
  view->delta = prog->delta.data();
  view->label = prog->label.data();
  view->quant = prog->quant.data();
  view->atom_names = prog->atom_ptrs.data();
  view->letter_bits = prog->letter_bits;
  view->letter_class = prog->letter_class.empty() ? nullptr : prog->letter_class.data();
  return LTL4C_OK;
}

extern "C" void ltl4c_program_free(ltl4c_program *prog) { delete prog; }
