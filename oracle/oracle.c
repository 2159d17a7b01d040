/*
 * oracle.c -- TEST INFRASTRUCTURE ONLY (see oracle.h).
 *
 * Plain, slow CPU interpreter of LTL4-C (arXiv:1411.2239).  Everything here
 * follows the paper's definitions in the paper's order:
 *
 *   parse        Def. 3, canonical prefix form Eq. 4/5,
 *                derived operators F/G
 *   leaf verdict Def. 4: [u |=_4 psi] via
 *                  - the textbook LTL tableau (Lichtenstein-Pnueli atoms over the
 *                    elementary subformulas, self-fulfilling SCCs) to decide
 *                    "forall v in Sigma^omega: uv |= psi" and its dual; the
 *                    prefix u is followed through the tableau with a subset of
 *                    atoms per run (the construction of [bls10-jlc]);
 *                  - FLTL evaluated by its definition on u itself.
 *   slices       value vectors and u^D, Eq. D
 *   tree         P, B, S (Eq. S)
 *   node verdict Def. 6 under readings A1-A4, A9:
 *                the forall-v clauses are the permanence rules of Table 1
 *                 and P:690.
 *
 * Parity unpinned: none of the functions below is unpinned; see DESIGN.md
 * "Oracle pins" for the test that pins each one.
 */
#include "oracle.h"

#include <ctype.h>
#include <pthread.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------ */
/* formula nodes (desugared: TRUE, ATOM, NOT, AND, X, U -- P:288)      */
/* ------------------------------------------------------------------------ */
enum { N_TRUE = 0, N_ATOM, N_NOT, N_AND, N_X, N_U };

#define MAXNODES 256
#define MAXATOMS 8
#define MAXE 12

typedef struct { int op, a, b, atom; } node_t;

typedef struct {
  int kind, cmp;
  uint64_t num, den; /* A: num/den reduced in [0,1]; E: num = constant, den = 1 */
  char var[64];
  char key[64];
} quant_t;

struct orc_prop {
  int nq;
  quant_t q[ORC_MAX_LEVELS];
  int nnodes;
  node_t nodes[MAXNODES];
  int root;
  int natoms;
  char atoms[MAXATOMS][128];
  /* tableau over elementary formulas (built once after parsing) */
  int nX, nU, E, nA;
  int xnode[MAXNODES], unode[MAXNODES];
  uint8_t *val;        /* val[A * nnodes + node] */
  uint8_t *consistent; /* consistent[A] */
  uint32_t *sig_req;   /* what atom A requires of its successor */
  uint32_t *sig_prov;  /* what atom A provides to its predecessor */
  uint8_t *good;       /* good[A]: A starts an infinite fulfilling path */
};

/* ------------------------------------------------------------------------ */
/* parser                                                                    */
/* ------------------------------------------------------------------------ */
enum { T_EOF = 0, T_IDENT, T_NUM, T_PCT, T_LBR, T_RBR, T_LP, T_RP, T_COMMA, T_COLON,
       T_IMPLIES_Q, T_ARROW, T_AND, T_OR, T_NOT, T_LT, T_LE, T_GT, T_GE, T_EQ, T_MINUS,
       T_BAD };

typedef struct {
  const char *s;
  int pos;
  int tok;
  char text[128];
  int tstart;
  orc_prop *p;
  int err;
  char *errbuf;
  int errlen;
  int nvars; /* number of quantifier variables declared so far */
} parser_t;

static void perr(parser_t *ps, int code, const char *msg) {
  if (ps->err) return;
  ps->err = code;
  if (ps->errbuf && ps->errlen > 0)
    snprintf(ps->errbuf, (size_t)ps->errlen, "%s at offset %d", msg, ps->tstart);
}

static void next(parser_t *ps) {
  const char *s = ps->s;
  for (;;) {
    while (s[ps->pos] && isspace((unsigned char)s[ps->pos])) ps->pos++;
    if (s[ps->pos] == '#') { /* comment to end of line */
      while (s[ps->pos] && s[ps->pos] != '\n') ps->pos++;
      continue;
    }
    break;
  }
  ps->tstart = ps->pos;
  ps->text[0] = 0;
  char c = s[ps->pos];
  if (!c) { ps->tok = T_EOF; return; }
  if (isalpha((unsigned char)c) || c == '_') {
    int n = 0;
    while (isalnum((unsigned char)s[ps->pos]) || s[ps->pos] == '_') {
      if (n < 127) ps->text[n++] = s[ps->pos];
      ps->pos++;
    }
    ps->text[n] = 0;
    ps->tok = T_IDENT;
    return;
  }
  if (isdigit((unsigned char)c) || (c == '.' && isdigit((unsigned char)s[ps->pos + 1]))) {
    int n = 0;
    while (isdigit((unsigned char)s[ps->pos]) || s[ps->pos] == '.') {
      if (n < 127) ps->text[n++] = s[ps->pos];
      ps->pos++;
    }
    ps->text[n] = 0;
    ps->tok = T_NUM;
    return;
  }
  ps->pos++;
  char d = s[ps->pos];
  switch (c) {
    case '%': ps->tok = T_PCT; return;
    case '[': ps->tok = T_LBR; return;
    case ']': ps->tok = T_RBR; return;
    case '(': ps->tok = T_LP; return;
    case ')': ps->tok = T_RP; return;
    case ',': ps->tok = T_COMMA; return;
    case ':': ps->tok = T_COLON; return;
    case '!': ps->tok = T_NOT; return;
    case '~': ps->tok = T_NOT; return;
    case '&': if (d == '&') ps->pos++; ps->tok = T_AND; return;
    case '|': if (d == '|') ps->pos++; ps->tok = T_OR; return;
    case '<': if (d == '=') { ps->pos++; ps->tok = T_LE; } else ps->tok = T_LT; return;
    case '>': if (d == '=') { ps->pos++; ps->tok = T_GE; } else ps->tok = T_GT; return;
    case '=':
      if (d == '>') { ps->pos++; ps->tok = T_IMPLIES_Q; return; }
      if (d == '=') ps->pos++;
      ps->tok = T_EQ; return;
    case '-':
      if (d == '>') { ps->pos++; ps->tok = T_ARROW; return; }
      ps->tok = T_MINUS; return;
    default: ps->tok = T_BAD; return;
  }
}

static int is_kw(parser_t *ps, const char *kw) {
  return ps->tok == T_IDENT && strcmp(ps->text, kw) == 0;
}

/* hash-consed node constructor (identical subformulas share one node) */
static int mk(parser_t *ps, int op, int a, int b, int atom) {
  orc_prop *p = ps->p;
  for (int i = 0; i < p->nnodes; i++) {
    node_t *n = &p->nodes[i];
    if (n->op == op && n->a == a && n->b == b && n->atom == atom) return i;
  }
  if (p->nnodes >= MAXNODES) { perr(ps, ORC_E_BUDGET, "formula too large"); return 0; }
  node_t *n = &p->nodes[p->nnodes];
  n->op = op; n->a = a; n->b = b; n->atom = atom;
  return p->nnodes++;
}
static int mk_not(parser_t *ps, int a) { return mk(ps, N_NOT, a, -1, -1); }
static int mk_and(parser_t *ps, int a, int b) { return mk(ps, N_AND, a, b, -1); }
static int mk_true(parser_t *ps) { return mk(ps, N_TRUE, -1, -1, -1); }
/* a || b  ==  !( !a && !b ) */
static int mk_or(parser_t *ps, int a, int b) { return mk_not(ps, mk_and(ps, mk_not(ps, a), mk_not(ps, b))); }
/* F a == true U a ; G a == !F !a */
static int mk_F(parser_t *ps, int a) { return mk(ps, N_U, mk_true(ps), a, -1); }
static int mk_G(parser_t *ps, int a) { return mk_not(ps, mk_F(ps, mk_not(ps, a))); }

static int var_bound(parser_t *ps, const char *v) {
  for (int i = 0; i < ps->nvars; i++)
    if (strcmp(ps->p->q[i].var, v) == 0) return 1;
  return 0;
}

static int parse_impl(parser_t *ps);

static int parse_primary(parser_t *ps) {
  if (ps->err) return 0;
  if (ps->tok == T_LP) {
    next(ps);
    int r = parse_impl(ps);
    if (ps->tok != T_RP) { perr(ps, ORC_E_SYNTAX, "expected ')'"); return 0; }
    next(ps);
    return r;
  }
  if (ps->tok != T_IDENT) { perr(ps, ORC_E_SYNTAX, "expected a proposition"); return 0; }
  if (is_kw(ps, "forall") || is_kw(ps, "exists")) {
    perr(ps, ORC_E_NONCANONICAL, "quantifier inside the quantifier-free body");
    return 0;
  }
  if (is_kw(ps, "true")) { next(ps); return mk_true(ps); }
  if (is_kw(ps, "false")) { next(ps); return mk_not(ps, mk_true(ps)); }
  if (is_kw(ps, "U")) { perr(ps, ORC_E_SYNTAX, "unexpected U"); return 0; }
  /* predicate application name or name(args) -> an atomic proposition */
  char name[128];
  snprintf(name, sizeof name, "%s", ps->text);
  next(ps);
  char full[128];
  snprintf(full, sizeof full, "%s", name);
  if (ps->tok == T_LP) {
    next(ps);
    size_t len = strlen(full);
    full[len++] = '(';
    full[len] = 0;
    int first = 1;
    for (;;) {
      if (ps->tok != T_IDENT) { perr(ps, ORC_E_SYNTAX, "expected a variable"); return 0; }
      if (!var_bound(ps, ps->text)) { perr(ps, ORC_E_UNBOUND, "unbound variable"); return 0; }
      len = strlen(full);
      snprintf(full + len, sizeof full - len, "%s%s", first ? "" : ",", ps->text);
      first = 0;
      next(ps);
      if (ps->tok == T_COMMA) { next(ps); continue; }
      if (ps->tok == T_RP) { next(ps); break; }
      perr(ps, ORC_E_SYNTAX, "expected ',' or ')'");
      return 0;
    }
    len = strlen(full);
    snprintf(full + len, sizeof full - len, ")");
  }
  orc_prop *p = ps->p;
  int j;
  for (j = 0; j < p->natoms; j++)
    if (strcmp(p->atoms[j], full) == 0) break;
  if (j == p->natoms) {
    if (p->natoms >= MAXATOMS) { perr(ps, ORC_E_BUDGET, "more than 8 atoms"); return 0; }
    snprintf(p->atoms[p->natoms++], 128, "%s", full);
  }
  return mk(ps, N_ATOM, -1, -1, j);
}

static int parse_unary(parser_t *ps) {
  if (ps->err) return 0;
  if (ps->tok == T_NOT) { next(ps); return mk_not(ps, parse_unary(ps)); }
  if (is_kw(ps, "X")) { next(ps); int a = parse_unary(ps); return mk(ps, N_X, a, -1, -1); }
  if (is_kw(ps, "F")) { next(ps); return mk_F(ps, parse_unary(ps)); }
  if (is_kw(ps, "G")) { next(ps); return mk_G(ps, parse_unary(ps)); }
  return parse_primary(ps);
}

static int parse_until(parser_t *ps) {
  int a = parse_unary(ps);
  if (ps->err) return 0;
  if (is_kw(ps, "U")) {
    next(ps);
    int b = parse_until(ps); /* right associative */
    return mk(ps, N_U, a, b, -1);
  }
  return a;
}

static int parse_and(parser_t *ps) {
  int a = parse_until(ps);
  while (!ps->err && ps->tok == T_AND) {
    next(ps);
    a = mk_and(ps, a, parse_until(ps));
  }
  return a;
}

static int parse_or(parser_t *ps) {
  int a = parse_and(ps);
  while (!ps->err && ps->tok == T_OR) {
    next(ps);
    a = mk_or(ps, a, parse_and(ps));
  }
  return a;
}

static int parse_impl(parser_t *ps) {
  int a = parse_or(ps);
  if (!ps->err && ps->tok == T_ARROW) {
    next(ps);
    int b = parse_impl(ps); /* right associative; a -> b == !a || b */
    return mk_or(ps, mk_not(ps, a), b);
  }
  return a;
}

static uint64_t gcd64(uint64_t a, uint64_t b) {
  while (b) { uint64_t t = a % b; a = b; b = t; }
  return a;
}

/* constraint "[" cmp number ["%"] "]" of Def. 3; A5/A6 readings */
static void parse_constraint(parser_t *ps, quant_t *q) {
  next(ps); /* past '[' */
  switch (ps->tok) {
    case T_LT: q->cmp = ORC_LT; break;
    case T_LE: q->cmp = ORC_LE; break;
    case T_GT: q->cmp = ORC_GT; break;
    case T_GE: q->cmp = ORC_GE; break;
    case T_EQ: q->cmp = ORC_EQ; break;
    default: perr(ps, ORC_E_SYNTAX, "expected a comparison operator"); return;
  }
  next(ps);
  int neg = 0;
  if (ps->tok == T_MINUS) { neg = 1; next(ps); }
  if (ps->tok != T_NUM) { perr(ps, ORC_E_SYNTAX, "expected a number"); return; }
  char num[128];
  snprintf(num, sizeof num, "%s", ps->text);
  next(ps);
  int pct = 0;
  if (ps->tok == T_PCT) { pct = 1; next(ps); }
  if (ps->tok != T_RBR) { perr(ps, ORC_E_SYNTAX, "expected ']'"); return; }
  next(ps);
  /* exact decimal -> mantissa / 10^frac */
  uint64_t mant = 0;
  int frac = -1, ndig = 0, dots = 0;
  for (const char *c = num; *c; c++) {
    if (*c == '.') { dots++; frac = 0; continue; }
    if (ndig >= 18) { perr(ps, ORC_E_RANGE, "constant has too many digits"); return; }
    mant = mant * 10 + (uint64_t)(*c - '0');
    ndig++;
    if (frac >= 0) frac++;
  }
  if (dots > 1) { perr(ps, ORC_E_SYNTAX, "malformed number"); return; }
  if (frac < 0) frac = 0;
  if (neg && mant != 0) { perr(ps, ORC_E_RANGE, "negative constant"); return; }
  if (q->kind == ORC_Q_E) {
    /* l in Z (>= 0, reading A6) */
    if (pct || frac > 0) { perr(ps, ORC_E_RANGE, "E constant must be an integer"); return; }
    if (mant > (1ull << 40)) { perr(ps, ORC_E_RANGE, "E constant too large"); return; }
    q->num = mant;
    q->den = 1;
    return;
  }
  /* A: k in [0,1] as an exact reduced fraction (reading A5) */
  if ((!pct && frac > 6) || (pct && frac > 4)) {
    perr(ps, ORC_E_RANGE, "A constant has too many decimals"); return;
  }
  uint64_t den = 1;
  for (int i = 0; i < frac; i++) den *= 10;
  if (pct) den *= 100;
  if (mant > den) { perr(ps, ORC_E_RANGE, "A constant outside [0,1]"); return; }
  uint64_t g = gcd64(mant, den);
  if (g == 0) g = den; /* mant == 0 -> 0/1 */
  q->num = mant / g;
  q->den = den / g;
}

/* quant := ('forall'|'exists') constraint? VAR ':' KEY '(' VAR ')' '=>' */
static int parse_property(parser_t *ps) {
  int open_parens = 0;
  for (;;) {
    if (ps->err) return 0;
    /* optional parentheses that wrap a nested quantifier */
    if (ps->tok == T_LP) {
      int save_pos = ps->pos, save_tok = ps->tok, save_start = ps->tstart;
      char save_text[128];
      memcpy(save_text, ps->text, sizeof save_text);
      int k = 0;
      while (ps->tok == T_LP) { next(ps); k++; }
      if (is_kw(ps, "forall") || is_kw(ps, "exists")) {
        open_parens += k;
      } else { /* not a quantifier: rewind, it is the body */
        ps->pos = save_pos; ps->tok = save_tok; ps->tstart = save_start;
        memcpy(ps->text, save_text, sizeof save_text);
      }
    }
    if (!(is_kw(ps, "forall") || is_kw(ps, "exists"))) break;
    orc_prop *p = ps->p;
    if (p->nq >= ORC_MAX_LEVELS) { perr(ps, ORC_E_BUDGET, "more than 3 quantifiers"); return 0; }
    quant_t *q = &p->q[p->nq];
    q->kind = is_kw(ps, "forall") ? ORC_Q_A : ORC_Q_E;
    /* defaults: A means A_{=1}, E means E_{>=1} */
    if (q->kind == ORC_Q_A) { q->cmp = ORC_EQ; q->num = 1; q->den = 1; }
    else { q->cmp = ORC_GE; q->num = 1; q->den = 1; }
    next(ps);
    if (ps->tok == T_LBR) parse_constraint(ps, q);
    if (ps->err) return 0;
    if (ps->tok != T_IDENT) { perr(ps, ORC_E_SYNTAX, "expected the bound variable"); return 0; }
    snprintf(q->var, sizeof q->var, "%s", ps->text);
    for (int i = 0; i < p->nq; i++)
      if (strcmp(p->q[i].var, q->var) == 0) { perr(ps, ORC_E_SYNTAX, "variable bound twice"); return 0; }
    next(ps);
    if (ps->tok != T_COLON) { perr(ps, ORC_E_SYNTAX, "expected ':'"); return 0; }
    next(ps);
    if (ps->tok != T_IDENT) { perr(ps, ORC_E_SYNTAX, "expected the guard predicate"); return 0; }
    snprintf(q->key, sizeof q->key, "%s", ps->text);
    next(ps);
    if (ps->tok != T_LP) { perr(ps, ORC_E_SYNTAX, "expected '('"); return 0; }
    next(ps);
    if (ps->tok != T_IDENT) { perr(ps, ORC_E_SYNTAX, "expected the guard variable"); return 0; }
    if (strcmp(ps->text, q->var) != 0) { perr(ps, ORC_E_UNBOUND, "guard variable differs"); return 0; }
    next(ps);
    if (ps->tok != T_RP) { perr(ps, ORC_E_SYNTAX, "expected ')'"); return 0; }
    next(ps);
    if (ps->tok != T_IMPLIES_Q) { perr(ps, ORC_E_SYNTAX, "expected '=>'"); return 0; }
    next(ps);
    p->nq++;
    ps->nvars = p->nq;
  }
  int body = parse_impl(ps);
  if (ps->err) return 0;
  for (int i = 0; i < open_parens; i++) {
    if (ps->tok != T_RP) { perr(ps, ORC_E_SYNTAX, "expected ')'"); return 0; }
    next(ps);
  }
  if (ps->tok == T_IDENT && (is_kw(ps, "forall") || is_kw(ps, "exists"))) {
    perr(ps, ORC_E_NONCANONICAL, "quantifier after the body");
    return 0;
  }
  if (ps->tok != T_EOF) { perr(ps, ORC_E_SYNTAX, "trailing input"); return 0; }
  return body;
}

/* ------------------------------------------------------------------------ */
/* LTL tableau (textbook: atoms = consistent valuations of the elementary     */
/* formulas, edges by the X rule, self-fulfilling SCCs).  Used to decide      */
/* "forall v: uv |= psi" / "forall v: uv |/= psi" of Def. 4.                  */
/* ------------------------------------------------------------------------ */

/* variable index of an elementary formula inside an atom (bit position) */
static int xvar(const orc_prop *p, int xi) { return p->natoms + xi; }
static int uvar(const orc_prop *p, int ui) { return p->natoms + p->nX + ui; }
static int xuvar(const orc_prop *p, int ui) { return p->natoms + p->nX + p->nU + ui; }

static int build_tableau(orc_prop *p) {
  p->nX = p->nU = 0;
  for (int i = 0; i < p->nnodes; i++) {
    if (p->nodes[i].op == N_X) p->xnode[p->nX++] = i;
    if (p->nodes[i].op == N_U) p->unode[p->nU++] = i;
  }
  p->E = p->natoms + p->nX + 2 * p->nU;
  if (p->E > MAXE) return ORC_E_BUDGET;
  p->nA = 1 << p->E;
  int nA = p->nA, nn = p->nnodes;
  p->val = (uint8_t *)calloc((size_t)nA * nn, 1);
  p->consistent = (uint8_t *)calloc((size_t)nA, 1);
  p->sig_req = (uint32_t *)calloc((size_t)nA, 4);
  p->sig_prov = (uint32_t *)calloc((size_t)nA, 4);
  p->good = (uint8_t *)calloc((size_t)nA, 1);
  if (!p->val || !p->consistent || !p->sig_req || !p->sig_prov || !p->good) return ORC_E_BUDGET;

  /* value of every node under atom A; nodes are created children-first, so
   * increasing node id is a topological order */
  int xi_of[MAXNODES], ui_of[MAXNODES];
  for (int i = 0; i < nn; i++) xi_of[i] = ui_of[i] = -1;
  for (int k = 0; k < p->nX; k++) xi_of[p->xnode[k]] = k;
  for (int k = 0; k < p->nU; k++) ui_of[p->unode[k]] = k;
  for (int A = 0; A < nA; A++) {
    uint8_t *v = &p->val[(size_t)A * nn];
    for (int i = 0; i < nn; i++) {
      node_t *n = &p->nodes[i];
      switch (n->op) {
        case N_TRUE: v[i] = 1; break;
        case N_ATOM: v[i] = (A >> n->atom) & 1; break;
        case N_NOT: v[i] = !v[n->a]; break;
        case N_AND: v[i] = v[n->a] && v[n->b]; break;
        case N_X: v[i] = (A >> xvar(p, xi_of[i])) & 1; break;
        case N_U: v[i] = (A >> uvar(p, ui_of[i])) & 1; break;
      }
    }
    /* consistency: phi U psi <-> psi || (phi && X(phi U psi))  (expansion law) */
    int ok = 1;
    for (int k = 0; k < p->nU; k++) {
      node_t *n = &p->nodes[p->unode[k]];
      int xu = (A >> xuvar(p, k)) & 1;
      int rhs = v[n->b] || (v[n->a] && xu);
      if (v[p->unode[k]] != rhs) ok = 0;
    }
    p->consistent[A] = (uint8_t)ok;
    /* successor constraint: X phi in A <-> phi in B ; X(U) in A <-> U in B */
    uint32_t req = 0, prov = 0;
    for (int k = 0; k < p->nX; k++) {
      if ((A >> xvar(p, k)) & 1) req |= 1u << k;
      if (v[p->nodes[p->xnode[k]].a]) prov |= 1u << k;
    }
    for (int k = 0; k < p->nU; k++) {
      if ((A >> xuvar(p, k)) & 1) req |= 1u << (p->nX + k);
      if (v[p->unode[k]]) prov |= 1u << (p->nX + k);
    }
    p->sig_req[A] = req;
    p->sig_prov[A] = prov;
  }

  /* edges A -> B  iff  both consistent and sig_req[A] == sig_prov[B].
   * Tarjan SCC (iterative) over consistent atoms. */
  int *index = (int *)malloc(sizeof(int) * nA), *low = (int *)malloc(sizeof(int) * nA);
  int *onstk = (int *)calloc((size_t)nA, sizeof(int)), *stk = (int *)malloc(sizeof(int) * nA);
  int *comp = (int *)malloc(sizeof(int) * nA);
  int *cs_node = (int *)malloc(sizeof(int) * nA), *cs_it = (int *)malloc(sizeof(int) * nA);
  for (int A = 0; A < nA; A++) { index[A] = -1; comp[A] = -1; }
  int idx = 0, sp = 0, ncomp = 0;
  for (int s = 0; s < nA; s++) {
    if (!p->consistent[s] || index[s] >= 0) continue;
    int csp = 0;
    cs_node[csp] = s; cs_it[csp] = 0; csp++;
    index[s] = low[s] = idx++; stk[sp++] = s; onstk[s] = 1;
    while (csp > 0) {
      int A = cs_node[csp - 1];
      int advanced = 0;
      while (cs_it[csp - 1] < nA) {
        int B = cs_it[csp - 1]++;
        if (!p->consistent[B] || p->sig_prov[B] != p->sig_req[A]) continue;
        if (index[B] < 0) {
          index[B] = low[B] = idx++; stk[sp++] = B; onstk[B] = 1;
          cs_node[csp] = B; cs_it[csp] = 0; csp++;
          advanced = 1;
          break;
        } else if (onstk[B] && index[B] < low[A]) {
          low[A] = index[B];
        }
      }
      if (advanced) continue;
      if (low[A] == index[A]) {
        int B;
        do { B = stk[--sp]; onstk[B] = 0; comp[B] = ncomp; } while (B != A);
        ncomp++;
      }
      csp--;
      if (csp > 0) {
        int P = cs_node[csp - 1];
        if (low[A] < low[P]) low[P] = low[A];
      }
    }
  }
  /* fair (self-fulfilling) nontrivial SCCs */
  uint8_t *fair = (uint8_t *)calloc((size_t)(ncomp + 1), 1);
  int *csize = (int *)calloc((size_t)(ncomp + 1), sizeof(int));
  uint8_t *cedge = (uint8_t *)calloc((size_t)(ncomp + 1), 1);
  for (int A = 0; A < nA; A++) if (comp[A] >= 0) csize[comp[A]]++;
  for (int A = 0; A < nA; A++) {
    if (comp[A] < 0) continue;
    for (int B = 0; B < nA; B++)
      if (comp[B] == comp[A] && p->sig_prov[B] == p->sig_req[A]) { cedge[comp[A]] = 1; break; }
  }
  for (int c = 0; c < ncomp; c++) {
    if (!cedge[c]) continue; /* trivial SCC: no edge inside */
    int ok = 1;
    for (int k = 0; k < p->nU && ok; k++) {
      node_t *n = &p->nodes[p->unode[k]];
      int has_u = 0, has_psi = 0;
      for (int A = 0; A < nA; A++) {
        if (comp[A] != c) continue;
        const uint8_t *v = &p->val[(size_t)A * nn];
        if (v[p->unode[k]]) has_u = 1;
        if (v[n->b]) has_psi = 1;
      }
      if (has_u && !has_psi) ok = 0;
    }
    fair[c] = (uint8_t)ok;
  }
  /* good = can reach a fair SCC (backward closure) */
  for (int A = 0; A < nA; A++) if (comp[A] >= 0 && fair[comp[A]]) p->good[A] = 1;
  /* sig values have nX + nU <= MAXE bits: a flag per sig value of a good atom */
  uint8_t *goodprov = (uint8_t *)calloc((size_t)1 << (p->nX + p->nU), 1);
  for (int B = 0; B < nA; B++) if (p->good[B]) goodprov[p->sig_prov[B]] = 1;
  int changed = 1;
  while (changed) {
    changed = 0;
    for (int A = 0; A < nA; A++) {
      if (!p->consistent[A] || p->good[A] || !goodprov[p->sig_req[A]]) continue;
      p->good[A] = 1;
      goodprov[p->sig_prov[A]] = 1;
      changed = 1;
    }
  }
  free(goodprov);
  free(index); free(low); free(onstk); free(stk); free(comp); free(cs_node); free(cs_it);
  free(fair); free(csize); free(cedge);
  return ORC_OK;
}

int orc_parse(const char *text, orc_prop **out, char *err, int errlen) {
  *out = NULL;
  if (err && errlen > 0) err[0] = 0;
  orc_prop *p = (orc_prop *)calloc(1, sizeof(orc_prop));
  if (!p) return ORC_E_BUDGET;
  parser_t ps;
  memset(&ps, 0, sizeof ps);
  ps.s = text; ps.p = p; ps.errbuf = err; ps.errlen = errlen;
  next(&ps);
  p->root = parse_property(&ps);
  if (ps.err) { orc_prop_free(p); return ps.err; }
  int rc = build_tableau(p);
  if (rc) {
    if (err && errlen > 0) snprintf(err, (size_t)errlen, "tableau too large");
    orc_prop_free(p);
    return rc;
  }
  *out = p;
  return ORC_OK;
}

void orc_prop_free(orc_prop *p) {
  if (!p) return;
  free(p->val); free(p->consistent); free(p->sig_req); free(p->sig_prov); free(p->good);
  free(p);
}

int orc_num_levels(const orc_prop *p) { return p->nq; }
int orc_num_atoms(const orc_prop *p) { return p->natoms; }
int orc_atom_name(const orc_prop *p, int j, char *buf, int buflen) {
  if (j < 0 || j >= p->natoms) return -1;
  snprintf(buf, (size_t)buflen, "%s", p->atoms[j]);
  return 0;
}
int orc_quantifier(const orc_prop *p, int i, int *kind, int *cmp, uint64_t *num, uint64_t *den,
                   char *key, int keylen) {
  if (i < 0 || i >= p->nq) return -1;
  *kind = p->q[i].kind; *cmp = p->q[i].cmp; *num = p->q[i].num; *den = p->q[i].den;
  snprintf(key, (size_t)keylen, "%s", p->q[i].key);
  return 0;
}

/* ------------------------------------------------------------------------ */
/* per-instance (LTL4 submonitor) run state: the set of tableau atoms that   */
/* can be at the current position of a run over u with psi true (pos) and   */
/* with psi false (neg) at position 0.                                       */
/* ------------------------------------------------------------------------ */
typedef struct { uint64_t *pos, *neg; } runset_t;

static int words_of(const orc_prop *p) { return (p->nA + 63) / 64; }

static void run_first(const orc_prop *p, uint8_t a, uint64_t *pos, uint64_t *neg) {
  int W = words_of(p);
  memset(pos, 0, sizeof(uint64_t) * W);
  memset(neg, 0, sizeof(uint64_t) * W);
  uint32_t lmask = (1u << p->natoms) - 1u;
  for (int A = 0; A < p->nA; A++) {
    if (!p->consistent[A] || ((uint32_t)A & lmask) != (a & lmask)) continue;
    if (p->val[(size_t)A * p->nnodes + p->root]) pos[A >> 6] |= 1ull << (A & 63);
    else neg[A >> 6] |= 1ull << (A & 63);
  }
}

/* S' = { B consistent : letter(B) = a and exists A in S with A -> B }.
 * A -> B iff sig_req[A] == sig_prov[B], so S' is the set of atoms with letter a
 * whose sig_prov is one of the sig_req values of S. */
static void run_step(const orc_prop *p, uint8_t a, uint64_t *set, uint64_t *tmp) {
  int W = words_of(p);
  uint32_t req[64];
  int nreq = 0, overflow = 0;
  for (int A = 0; A < p->nA && !overflow; A++) {
    if (!((set[A >> 6] >> (A & 63)) & 1)) continue;
    int k;
    for (k = 0; k < nreq; k++) if (req[k] == p->sig_req[A]) break;
    if (k == nreq) { if (nreq == 64) overflow = 1; else req[nreq++] = p->sig_req[A]; }
  }
  memset(tmp, 0, sizeof(uint64_t) * W);
  uint32_t lmask = (1u << p->natoms) - 1u;
  for (int B = 0; B < p->nA; B++) {
    if (!p->consistent[B] || ((uint32_t)B & lmask) != (a & lmask)) continue;
    int hit = 0;
    if (!overflow) {
      for (int k = 0; k < nreq; k++) if (req[k] == p->sig_prov[B]) { hit = 1; break; }
    } else {
      for (int A = 0; A < p->nA; A++)
        if (((set[A >> 6] >> (A & 63)) & 1) && p->sig_req[A] == p->sig_prov[B]) { hit = 1; break; }
    }
    if (hit) tmp[B >> 6] |= 1ull << (B & 63);
  }
  memcpy(set, tmp, sizeof(uint64_t) * W);
}

static int any_good(const orc_prop *p, const uint64_t *set) {
  for (int A = 0; A < p->nA; A++)
    if (((set[A >> 6] >> (A & 63)) & 1) && p->good[A]) return 1;
  return 0;
}

/* FLTL on a nonempty word, evaluated backwards over positions:
 *   [u_i |= X phi]      = (i+1 < n) && [u_{i+1} |= phi]          (strong next)
 *   [u_i |= phi U psi]  = exists k in [i,n-1]: [u_k |= psi] && forall l in [i,k): [u_l |= phi]
 *                       = [u_i |= psi] || ([u_i |= phi] && i+1 < n && [u_{i+1} |= phi U psi])
 * (the second line is the first unrolled at k = i). */
static int fltl_eval(const orc_prop *p, const uint8_t *w, int n) {
  int nn = p->nnodes;
  uint8_t cur[MAXNODES], nxt[MAXNODES];
  memset(nxt, 0, sizeof nxt);
  for (int i = n - 1; i >= 0; i--) {
    for (int k = 0; k < nn; k++) {
      const node_t *d = &p->nodes[k];
      switch (d->op) {
        case N_TRUE: cur[k] = 1; break;
        case N_ATOM: cur[k] = (w[i] >> d->atom) & 1; break;
        case N_NOT: cur[k] = !cur[d->a]; break;
        case N_AND: cur[k] = cur[d->a] && cur[d->b]; break;
        case N_X: cur[k] = (i + 1 < n) ? nxt[d->a] : 0; break;
        case N_U: cur[k] = cur[d->b] || (cur[d->a] && (i + 1 < n) && nxt[k]); break;
      }
    }
    memcpy(nxt, cur, sizeof cur);
  }
  return nxt[p->root];
}

int orc_fltl_word(const orc_prop *p, const uint8_t *word, int len) {
  if (len <= 0) return 0; /* reading A14: empty trace -> false */
  return fltl_eval(p, word, len);
}

/* Def. 4: T if every infinite extension satisfies, F if none does, else
 * Tp / Fp by the FLTL value of u. */
static int ltl4_verdict(const orc_prop *p, const uint64_t *pos, const uint64_t *neg,
                        const uint8_t *w, int n) {
  int sat_ext = any_good(p, pos);   /* exists v: uv |= psi   */
  int vio_ext = any_good(p, neg);   /* exists v: uv |/= psi  */
  if (!vio_ext) return 5;           /* forall v: uv |= psi   -> T  */
  if (!sat_ext) return 0;           /* forall v: uv |/= psi  -> F  */
  return fltl_eval(p, w, n) ? 3 : 2;
}

int orc_ltl4_word(const orc_prop *p, const uint8_t *word, int len) {
  int W = words_of(p);
  uint64_t *pos = (uint64_t *)calloc((size_t)W, 8), *neg = (uint64_t *)calloc((size_t)W, 8);
  uint64_t *tmp = (uint64_t *)calloc((size_t)W, 8);
  int r;
  if (len <= 0) {
    /* empty prefix: u = epsilon; run sets are "any atom" */
    uint8_t sat = 0, vio = 0;
    for (int A = 0; A < p->nA; A++) {
      if (!p->consistent[A] || !p->good[A]) continue;
      if (p->val[(size_t)A * p->nnodes + p->root]) sat = 1; else vio = 1;
    }
    r = !vio ? 5 : (!sat ? 0 : 2); /* FLTL on epsilon is false (A14) */
  } else {
    run_first(p, word[0], pos, neg);
    for (int i = 1; i < len; i++) {
      run_step(p, word[i], pos, tmp);
      run_step(p, word[i], neg, tmp);
    }
    r = ltl4_verdict(p, pos, neg, word, len);
  }
  free(pos); free(neg); free(tmp);
  return r;
}

/* ------------------------------------------------------------------------ */
/* Eq. S and Def. 6                                                          */
/* ------------------------------------------------------------------------ */
typedef unsigned __int128 u128;

/* S(B) with B the up-set {v >= t} (every B in Def. 6 is one): count ~ c*|P|
 * for A (exact rational: count*den ~ num*N, reading A5), count ~ c for E. */
static int S_upset(int kind, int cmp, uint64_t num, uint64_t den, const uint64_t h[6], int t) {
  uint64_t count = 0, N = 0;
  for (int v = 0; v < 6; v++) { N += h[v]; if (v >= t) count += h[v]; }
  u128 lhs, rhs;
  if (kind == ORC_Q_A) { lhs = (u128)count * den; rhs = (u128)num * N; }
  else { lhs = count; rhs = num; }
  switch (cmp) {
    case ORC_LT: return lhs < rhs;
    case ORC_LE: return lhs <= rhs;
    case ORC_GT: return lhs > rhs;
    case ORC_GE: return lhs >= rhs;
    default: return lhs == rhs;
  }
}

/* forall-v clause of Def. 6 row T (reading A2): the constraint on {T} stays
 * satisfied for every continuation.  Table 1 (E rows) and the same argument
 * for A: h[5] (# permanently true children) and h[0] (# permanently false)
 * can only grow; other children and new instances can become anything. */
static int forall_v_top(int kind, int cmp, uint64_t num, uint64_t den, const uint64_t h[6]) {
  if (kind == ORC_Q_E) {
    if (cmp == ORC_GT) return h[5] > num;        /* Table 1: "> c"  -> if > c   */
    if (cmp == ORC_GE) return h[5] >= num;       /* Table 1: ">= c" -> if >= c  */
    return 0;                                    /* =, <, <= never perm. true   */
  }
  /* A: count*den ~ num*N must hold for all future (count, N) */
  if (cmp == ORC_GE && num == 0) return 1;       /* A_{>=0}: always           */
  if (cmp == ORC_LE && num == den) return 1;     /* A_{<=1}: always           */
  if (cmp == ORC_GT && num == 0) return h[5] >= 1; /* A_{>0}: one T child     */
  if (cmp == ORC_LT && num == den) return h[0] >= 1; /* A_{<1}: one F child   */
  return 0;
}

/* forall-v clause of Def. 6 row F: the constraint on B6-{F} stays violated. */
static int forall_v_bot(int kind, int cmp, uint64_t num, uint64_t den, const uint64_t h[6]) {
  if (kind == ORC_Q_E) {
    if (cmp == ORC_EQ) return h[5] > num;        /* Table 1: "= c"  -> if > c   */
    if (cmp == ORC_LT) return h[5] >= num;       /* Table 1: "< c"  -> if >= c  */
    if (cmp == ORC_LE) return h[5] > num;        /* Table 1: "<= c" -> if > c   */
    return 0;
  }
  if ((cmp == ORC_EQ || cmp == ORC_GE) && num == den) return h[0] >= 1;
  if ((cmp == ORC_EQ || cmp == ORC_LE) && num == 0) return h[5] >= 1;   /* A_{=0}  */
  if (cmp == ORC_GT && num == den) return 1;     /* A_{>1}: unsatisfiable       */
  if (cmp == ORC_LT && num == 0) return 1;       /* A_{<0}: unsatisfiable       */
  return 0;
}

/* Def. 6 with readings A1 (Fp row), A2 (forall/exists clauses),
 * A3 (first match in lattice-descending order). */
int orc_rule(int kind, int cmp, uint64_t num, uint64_t den, const uint64_t h[6]) {
  /* T  : S({T}) = 1 and forall v */
  if (S_upset(kind, cmp, num, den, h, 5) && forall_v_top(kind, cmp, num, den, h)) return 5;
  /* F  : S(B6 - {F}) = 0 and forall v */
  if (!S_upset(kind, cmp, num, den, h, 1) && forall_v_bot(kind, cmp, num, den, h)) return 0;
  /* Tc : S({T, Tc}) = 1 */
  if (S_upset(kind, cmp, num, den, h, 4)) return 4;
  /* Tp : S({T, Tc, Tp}) = 1 and S({T, Tc}) = 0 */
  if (S_upset(kind, cmp, num, den, h, 3)) return 3;
  /* Fp : S({T, Tc, Tp}) = 0 and S(B6 - {F, Fc}) = 1   (reading A1) */
  if (S_upset(kind, cmp, num, den, h, 2)) return 2;
  /* Fc : S(B6 - {F, Fc}) = 0 */
  return 1;
}

/* ------------------------------------------------------------------------ */
/* Algorithm 1, plain sequential version                       */
/* ------------------------------------------------------------------------ */
typedef struct {
  int K;          /* key words per entry */
  uint64_t cap, n;
  uint32_t *keys; /* cap * K */
  int64_t *val;
} vmap_t;

static uint64_t hash_keys(const uint32_t *k, int K) {
  uint64_t h = 1469598103934665603ull;
  for (int i = 0; i < K; i++) { h ^= k[i]; h *= 1099511628211ull; h ^= h >> 29; }
  return h;
}

static void vmap_init(vmap_t *m, int K) {
  m->K = K; m->cap = 1024; m->n = 0;
  m->keys = (uint32_t *)malloc(sizeof(uint32_t) * m->cap * (K ? K : 1));
  m->val = (int64_t *)malloc(sizeof(int64_t) * m->cap);
  for (uint64_t i = 0; i < m->cap; i++) m->val[i] = -1;
}
static void vmap_free(vmap_t *m) { free(m->keys); free(m->val); }

static int64_t vmap_find(const vmap_t *m, const uint32_t *k) {
  int K = m->K;
  uint64_t i = hash_keys(k, K) & (m->cap - 1);
  for (;;) {
    if (m->val[i] < 0) return -1;
    if (memcmp(&m->keys[i * K], k, sizeof(uint32_t) * K) == 0) return m->val[i];
    i = (i + 1) & (m->cap - 1);
  }
}

static void vmap_put(vmap_t *m, const uint32_t *k, int64_t v);
static void vmap_grow(vmap_t *m) {
  vmap_t n2;
  n2.K = m->K; n2.cap = m->cap * 2; n2.n = 0;
  n2.keys = (uint32_t *)malloc(sizeof(uint32_t) * n2.cap * (m->K ? m->K : 1));
  n2.val = (int64_t *)malloc(sizeof(int64_t) * n2.cap);
  for (uint64_t i = 0; i < n2.cap; i++) n2.val[i] = -1;
  for (uint64_t i = 0; i < m->cap; i++)
    if (m->val[i] >= 0) vmap_put(&n2, &m->keys[i * m->K], m->val[i]);
  vmap_free(m);
  *m = n2;
}
static void vmap_put(vmap_t *m, const uint32_t *k, int64_t v) {
  if ((m->n + 1) * 2 > m->cap) vmap_grow(m);
  int K = m->K;
  uint64_t i = hash_keys(k, K) & (m->cap - 1);
  while (m->val[i] >= 0) {
    if (memcmp(&m->keys[i * K], k, sizeof(uint32_t) * K) == 0) { m->val[i] = v; return; }
    i = (i + 1) & (m->cap - 1);
  }
  memcpy(&m->keys[i * K], k, sizeof(uint32_t) * K);
  m->val[i] = v;
  m->n++;
}

struct orc_monitor {
  const orc_prop *p;
  int n;                 /* levels */
  vmap_t vec;            /* D -> vector id (the cache of value vectors, Alg. 1 "D") */
  uint64_t nvec, capvec;
  uint32_t *vkeys;       /* nvec * n */
  uint64_t *runs;        /* per vector: pos[W], neg[W] */
  uint64_t nev, capev;   /* bound events, in trace order */
  int64_t *ev_vid;
  uint8_t *ev_letter;
  uint64_t seen;
  /* tree after orc_evaluate */
  vmap_t level[ORC_MAX_LEVELS + 1];
  int8_t *lvl_verdict[ORC_MAX_LEVELS + 1];
  uint64_t lvl_count[ORC_MAX_LEVELS + 1];
  int evaluated;
};

orc_monitor *orc_monitor_new(const orc_prop *p) {
  orc_monitor *m = (orc_monitor *)calloc(1, sizeof(orc_monitor));
  m->p = p;
  m->n = p->nq;
  vmap_init(&m->vec, m->n);
  return m;
}

static void clear_tree(orc_monitor *m) {
  if (!m->evaluated) return;
  for (int l = 0; l <= m->n; l++) { vmap_free(&m->level[l]); free(m->lvl_verdict[l]); }
  m->evaluated = 0;
}

void orc_monitor_free(orc_monitor *m) {
  if (!m) return;
  clear_tree(m);
  vmap_free(&m->vec);
  free(m->vkeys); free(m->runs); free(m->ev_vid); free(m->ev_letter);
  free(m);
}

int orc_feed(orc_monitor *m, uint64_t n, const uint32_t *const *keys, const uint8_t *letters) {
  const orc_prop *p = m->p;
  int W = words_of(p);
  uint64_t *tmp = (uint64_t *)malloc(sizeof(uint64_t) * W);
  uint32_t D[ORC_MAX_LEVELS];
  for (uint64_t j = 0; j < n; j++) {
    m->seen++;
    /* epsilon(u_j, K): the event's value vector if every guard key is
     * bound in this event (Eq. D), else the event is in no slice (A10) */
    int complete = 1;
    for (int i = 0; i < m->n; i++) {
      D[i] = keys[i][j];
      if (D[i] == ORC_ABSENT) complete = 0;
    }
    if (!complete) continue;
    uint8_t a = letters[j];
    int64_t vid = vmap_find(&m->vec, D);
    if (vid < 0) {
      /* SpawnMonitors: first occurrence of D creates its submonitor */
      if (m->nvec == m->capvec) {
        m->capvec = m->capvec ? m->capvec * 2 : 1024;
        m->vkeys = (uint32_t *)realloc(m->vkeys, sizeof(uint32_t) * m->capvec * (m->n ? m->n : 1));
        m->runs = (uint64_t *)realloc(m->runs, sizeof(uint64_t) * m->capvec * 2 * W);
      }
      vid = (int64_t)m->nvec++;
      vmap_put(&m->vec, D, vid);
      memcpy(&m->vkeys[vid * m->n], D, sizeof(uint32_t) * m->n);
      run_first(p, a, &m->runs[(uint64_t)vid * 2 * W], &m->runs[(uint64_t)vid * 2 * W + W]);
    } else {
      /* UpdateMonitor on the slice u^D, in trace order */
      run_step(p, a, &m->runs[(uint64_t)vid * 2 * W], tmp);
      run_step(p, a, &m->runs[(uint64_t)vid * 2 * W + W], tmp);
    }
    if (m->nev == m->capev) {
      m->capev = m->capev ? m->capev * 2 : 4096;
      m->ev_vid = (int64_t *)realloc(m->ev_vid, sizeof(int64_t) * m->capev);
      m->ev_letter = (uint8_t *)realloc(m->ev_letter, m->capev);
    }
    m->ev_vid[m->nev] = vid;
    m->ev_letter[m->nev] = a;
    m->nev++;
  }
  free(tmp);
  m->evaluated = m->evaluated; /* tree is recomputed by orc_evaluate */
  return 0;
}

int orc_evaluate(orc_monitor *m, int *verdict, uint64_t hist[ORC_MAX_LEVELS + 1][6],
                 uint64_t *events_seen, uint64_t *events_bound) {
  const orc_prop *p = m->p;
  int n = m->n, W = words_of(p);
  clear_tree(m);
  memset(hist, 0, sizeof(uint64_t) * (ORC_MAX_LEVELS + 1) * 6);
  *events_seen = m->seen;
  *events_bound = m->nev;

  /* slices u^D: events of each vector in trace order */
  uint64_t V = m->nvec;
  uint64_t *start = (uint64_t *)calloc(V + 1, sizeof(uint64_t));
  for (uint64_t e = 0; e < m->nev; e++) start[m->ev_vid[e] + 1]++;
  for (uint64_t v = 0; v < V; v++) start[v + 1] += start[v];
  uint64_t *fill = (uint64_t *)malloc(sizeof(uint64_t) * (V + 1));
  memcpy(fill, start, sizeof(uint64_t) * (V + 1));
  uint8_t *slice = (uint8_t *)malloc(m->nev + 1);
  for (uint64_t e = 0; e < m->nev; e++) slice[fill[m->ev_vid[e]]++] = m->ev_letter[e];

  /* leaf verdicts [u^D |=_4 psi] (Def. 4) */
  int8_t *leaf = (int8_t *)malloc(V + 1);
  for (uint64_t v = 0; v < V; v++) {
    leaf[v] = (int8_t)ltl4_verdict(p, &m->runs[v * 2 * W], &m->runs[v * 2 * W + W],
                                   &slice[start[v]], (int)(start[v + 1] - start[v]));
  }

  /* tree levels: node at depth l = distinct D|^l (P); depth n = leaves */
  int64_t *par[ORC_MAX_LEVELS + 1];
  for (int l = 0; l <= n; l++) {
    vmap_init(&m->level[l], l);
    m->lvl_count[l] = 0;
    par[l] = NULL;
  }
  /* node ids per level and parent links */
  int64_t *node_of = (int64_t *)malloc(sizeof(int64_t) * (V + 1) * (n + 1));
  for (uint64_t v = 0; v < V; v++) {
    const uint32_t *D = &m->vkeys[v * n];
    for (int l = 0; l <= n; l++) {
      int64_t id;
      if (l == 0) id = 0;
      else {
        id = vmap_find(&m->level[l], D);
        if (id < 0) { id = (int64_t)m->lvl_count[l]; vmap_put(&m->level[l], D, id); }
      }
      if (l == 0 && m->lvl_count[0] == 0) m->lvl_count[0] = 1;
      if (l > 0 && id == (int64_t)m->lvl_count[l]) m->lvl_count[l]++;
      node_of[v * (n + 1) + l] = id;
    }
  }
  if (m->lvl_count[0] == 0) m->lvl_count[0] = 1; /* the root always exists */
  for (int l = 1; l <= n; l++) {
    par[l] = (int64_t *)malloc(sizeof(int64_t) * (m->lvl_count[l] + 1));
    for (uint64_t v = 0; v < V; v++)
      par[l][node_of[v * (n + 1) + l]] = node_of[v * (n + 1) + l - 1];
  }
  for (int l = 0; l <= n; l++)
    m->lvl_verdict[l] = (int8_t *)calloc(m->lvl_count[l] + 1, 1);
  /* leaves: the level-n node of vector v is v itself (distinct vectors) */
  for (uint64_t v = 0; v < V; v++) m->lvl_verdict[n][node_of[v * (n + 1) + n]] = leaf[v];
  if (n == 0) m->lvl_verdict[0][0] = V ? leaf[0] : (int8_t)orc_ltl4_word(p, NULL, 0);

  /* ApplyQuantifiers: depth n-1 down to 0; the truth vector v of
   * each node (Def. 7) counts its children per verdict (B) */
  for (int l = n - 1; l >= 0; l--) {
    uint64_t cnt = m->lvl_count[l];
    uint64_t (*h)[6] = (uint64_t (*)[6])calloc(cnt + 1, sizeof(uint64_t[6]));
    for (uint64_t c = 0; c < m->lvl_count[l + 1]; c++) h[par[l + 1][c]][m->lvl_verdict[l + 1][c]]++;
    const quant_t *q = &p->q[l];
    for (uint64_t x = 0; x < cnt; x++)
      m->lvl_verdict[l][x] = (int8_t)orc_rule(q->kind, q->cmp, q->num, q->den, h[x]);
    free(h);
  }
  for (int l = 0; l <= n; l++)
    for (uint64_t x = 0; x < m->lvl_count[l]; x++) hist[l][m->lvl_verdict[l][x]]++;
  *verdict = m->lvl_verdict[0][0];

  for (int l = 1; l <= n; l++) free(par[l]);
  free(node_of); free(leaf); free(slice); free(fill); free(start);
  m->evaluated = 1;
  return 0;
}

int orc_node_verdict(orc_monitor *m, int m_len, const uint32_t *prefix) {
  if (!m->evaluated || m_len < 0 || m_len > m->n) return -1;
  if (m_len == 0) return m->lvl_verdict[0][0];
  int64_t id = vmap_find(&m->level[m_len], prefix);
  if (id < 0) return -1;
  return m->lvl_verdict[m_len][id];
}

/* ------------------------------------------------------------------------ */
/* Timing mode: T threads, level-0 subtrees partitioned by a hash of k0.    */
/* Every node below the root has a value vector starting with k0 (P), */
/* so thread t's monitor holds exactly the subtrees whose k0 it owns and    */
/* the depth-l node counts (l >= 1) are sums over threads; the root's        */
/* children are the depth-1 nodes, so the root verdict is Def. 6 applied to  */
/* the summed depth-1 histogram (the same orc_rule).                         */
/* ------------------------------------------------------------------------ */
typedef struct {
  const orc_prop *p;
  uint64_t n;
  const uint32_t *const *keys;
  const uint8_t *letters;
  int t, T;
  int verdict;
  uint64_t hist[ORC_MAX_LEVELS + 1][6];
  uint64_t seen, bound;
} orc_job_t;

static uint32_t owner_of(uint32_t k0, int T) {
  uint64_t h = (uint64_t)k0 * 0x9E3779B97F4A7C15ull;
  return (uint32_t)((h >> 32) % (uint64_t)T);
}

static void *orc_job(void *arg) {
  orc_job_t *j = (orc_job_t *)arg;
  orc_monitor *m = orc_monitor_new(j->p);
  int n = j->p->nq;
  const uint64_t chunk = 1u << 16;
  uint32_t *kb[ORC_MAX_LEVELS];
  for (int i = 0; i < n; i++) kb[i] = (uint32_t *)malloc(sizeof(uint32_t) * chunk);
  uint8_t *lb = (uint8_t *)malloc(chunk);
  /* feed this thread's events in trace order, in chunks */
  for (uint64_t lo = 0; lo < j->n; lo += chunk) {
    uint64_t hi = lo + chunk < j->n ? lo + chunk : j->n, c = 0;
    for (uint64_t e = lo; e < hi; e++) {
      if (owner_of(j->keys[0][e], j->T) != (uint32_t)j->t) continue;
      for (int i = 0; i < n; i++) kb[i][c] = j->keys[i][e];
      lb[c++] = j->letters[e];
    }
    orc_feed(m, c, (const uint32_t *const *)kb, lb);
  }
  orc_evaluate(m, &j->verdict, j->hist, &j->seen, &j->bound);
  orc_monitor_free(m);
  for (int i = 0; i < n; i++) free(kb[i]);
  free(lb);
  return NULL;
}

int orc_run_threads(const orc_prop *p, uint64_t n, const uint32_t *const *keys, const uint8_t *letters,
                    int T, int *verdict, uint64_t hist[ORC_MAX_LEVELS + 1][6], uint64_t *events_seen,
                    uint64_t *events_bound) {
  if (T < 1 || p->nq < 1) return -1;
  orc_job_t *jobs = (orc_job_t *)calloc((size_t)T, sizeof(orc_job_t));
  pthread_t *th = (pthread_t *)calloc((size_t)T, sizeof(pthread_t));
  for (int t = 0; t < T; t++) {
    jobs[t].p = p; jobs[t].n = n; jobs[t].keys = keys; jobs[t].letters = letters;
    jobs[t].t = t; jobs[t].T = T;
    if (T == 1) orc_job(&jobs[0]);
    else pthread_create(&th[t], NULL, orc_job, &jobs[t]);
  }
  if (T > 1) for (int t = 0; t < T; t++) pthread_join(th[t], NULL);
  memset(hist, 0, sizeof(uint64_t) * (ORC_MAX_LEVELS + 1) * 6);
  *events_bound = 0;
  for (int t = 0; t < T; t++) {
    for (int l = 1; l <= p->nq; l++)
      for (int v = 0; v < 6; v++) hist[l][v] += jobs[t].hist[l][v];
    *events_bound += jobs[t].bound;
  }
  const quant_t *q = &p->q[0];
  *verdict = orc_rule(q->kind, q->cmp, q->num, q->den, hist[1]);
  hist[0][*verdict] = 1;
  *events_seen = n;
  free(jobs); free(th);
  return 0;
}

/* ------------------------------------------------------------------------ */
/* Records: the oracle's own reader of key -> value events (P:922-935,       */
/* "the trace event is a key-value structure"), one JSON object per line.    */
/* Written independently of the product's encoder; readings (A12,  */
/* A25-A27): a guard key's value is a JSON string or number, identified by   */
/* its canonical text (numbers as canonical decimals); a 0-ary atom q holds  */
/* iff q maps to true; q(x_i, ...) holds iff q maps to true or to the       */
/* event's own value(s) of x_i, ... (array in argument order for several).  */
/* Value ids are the oracle's own (first-appearance order per level); the    */
/* verdicts and counts do not depend on the labelling.                       */
/* ------------------------------------------------------------------------ */
typedef struct { char *s; uint32_t id; } ostr_t;
typedef struct { ostr_t *slot; uint64_t cap, n; } odict_t;

static uint64_t str_hash(const char *s) {
  uint64_t h = 0xcbf29ce484222325ull;
  for (; *s; s++) { h ^= (unsigned char)*s; h *= 0x100000001b3ull; }
  return h;
}
static uint32_t odict_id(odict_t *d, const char *s) {
  if ((d->n + 1) * 2 > d->cap) {
    uint64_t nc = d->cap ? d->cap * 2 : 1024;
    ostr_t *ns = (ostr_t *)calloc(nc, sizeof(ostr_t));
    for (uint64_t i = 0; i < d->cap; i++) {
      if (!d->slot[i].s) continue;
      uint64_t j = str_hash(d->slot[i].s) & (nc - 1);
      while (ns[j].s) j = (j + 1) & (nc - 1);
      ns[j] = d->slot[i];
    }
    free(d->slot); d->slot = ns; d->cap = nc;
  }
  uint64_t j = str_hash(s) & (d->cap - 1);
  while (d->slot[j].s) {
    if (strcmp(d->slot[j].s, s) == 0) return d->slot[j].id;
    j = (j + 1) & (d->cap - 1);
  }
  size_t sl = strlen(s) + 1;
  d->slot[j].s = (char *)malloc(sl);
  memcpy(d->slot[j].s, s, sl);
  d->slot[j].id = (uint32_t)d->n++;
  return d->slot[j].id;
}

/* a JSON value as the reader keeps it */
enum { JV_OTHER = 0, JV_TRUE, JV_SCALAR, JV_ARRAY };
#define JV_MAXITEMS 8
typedef struct {
  int kind;
  char text[256];                 /* JV_SCALAR: canonical text */
  int nitems;
  char items[JV_MAXITEMS][256];   /* JV_ARRAY: canonical text of scalar items ("" if not scalar) */
} jval_t;

typedef struct { const char *p, *e; int bad; } jrd_t;

static void jws(jrd_t *r) { while (r->p < r->e && (*r->p == ' ' || *r->p == '\t' || *r->p == '\r')) r->p++; }

/* string at '"' into out (UTF-8, escapes decoded; truncated to outlen - 1) */
static void jstring(jrd_t *r, char *out, int outlen) {
  int n = 0;
  r->p++;
  while (r->p < r->e && *r->p != '"') {
    unsigned int c = (unsigned char)*r->p++;
    if (c == '\\') {
      if (r->p >= r->e) { r->bad = 1; return; }
      char e = *r->p++;
      if (e == 'u') {
        unsigned int u = 0;
        for (int i = 0; i < 4; i++) {
          if (r->p >= r->e || !isxdigit((unsigned char)*r->p)) { r->bad = 1; return; }
          char h = *r->p++;
          u = u * 16 + (unsigned)(isdigit((unsigned char)h) ? h - '0' : (tolower((unsigned char)h) - 'a' + 10));
        }
        if (u >= 0xD800 && u < 0xDC00 && r->e - r->p >= 6 && r->p[0] == '\\' && r->p[1] == 'u') {
          unsigned int lo = 0;
          const char *save = r->p;
          r->p += 2;
          for (int i = 0; i < 4; i++) {
            char h = *r->p++;
            if (!isxdigit((unsigned char)h)) { r->bad = 1; return; }
            lo = lo * 16 + (unsigned)(isdigit((unsigned char)h) ? h - '0' : (tolower((unsigned char)h) - 'a' + 10));
          }
          if (lo >= 0xDC00 && lo < 0xE000) u = 0x10000 + ((u - 0xD800) << 10) + (lo - 0xDC00);
          else r->p = save;
        }
        /* UTF-8 encode */
        unsigned char b[4]; int nb;
        if (u < 0x80) { b[0] = (unsigned char)u; nb = 1; }
        else if (u < 0x800) { b[0] = (unsigned char)(0xC0 | (u >> 6)); b[1] = (unsigned char)(0x80 | (u & 63)); nb = 2; }
        else if (u < 0x10000) { b[0] = (unsigned char)(0xE0 | (u >> 12)); b[1] = (unsigned char)(0x80 | ((u >> 6) & 63)); b[2] = (unsigned char)(0x80 | (u & 63)); nb = 3; }
        else { b[0] = (unsigned char)(0xF0 | (u >> 18)); b[1] = (unsigned char)(0x80 | ((u >> 12) & 63)); b[2] = (unsigned char)(0x80 | ((u >> 6) & 63)); b[3] = (unsigned char)(0x80 | (u & 63)); nb = 4; }
        for (int i = 0; i < nb; i++) if (n < outlen - 1) out[n++] = (char)b[i];
        continue;
      }
      switch (e) {
        case 'n': c = '\n'; break; case 't': c = '\t'; break; case 'r': c = '\r'; break;
        case 'b': c = '\b'; break; case 'f': c = '\f'; break;
        case '"': case '\\': case '/': c = (unsigned char)e; break;
        default: r->bad = 1; return;
      }
    }
    if (n < outlen - 1) out[n++] = (char)c;
  }
  if (r->p >= r->e) { r->bad = 1; return; }
  r->p++;
  out[n] = 0;
}

/* number -> canonical decimal text: the value m x 10^(x) with m an integer whose
 * digits have no leading or trailing zeros, written positionally */
static void jnumber(jrd_t *r, char *out, int outlen) {
  int neg = 0;
  char dig[512]; int nd = 0;
  long exp10 = 0;
  if (*r->p == '-') { neg = 1; r->p++; }
  if (r->p >= r->e || !isdigit((unsigned char)*r->p)) { r->bad = 1; return; }
  while (r->p < r->e && isdigit((unsigned char)*r->p)) { if (nd < 500) dig[nd++] = *r->p; else exp10++; r->p++; }
  if (r->p < r->e && *r->p == '.') {
    r->p++;
    if (r->p >= r->e || !isdigit((unsigned char)*r->p)) { r->bad = 1; return; }
    while (r->p < r->e && isdigit((unsigned char)*r->p)) { if (nd < 500) { dig[nd++] = *r->p; exp10--; } r->p++; }
  }
  if (r->p < r->e && (*r->p == 'e' || *r->p == 'E')) {
    r->p++;
    int es = 1; long ev = 0;
    if (r->p < r->e && (*r->p == '+' || *r->p == '-')) { if (*r->p == '-') es = -1; r->p++; }
    if (r->p >= r->e || !isdigit((unsigned char)*r->p)) { r->bad = 1; return; }
    while (r->p < r->e && isdigit((unsigned char)*r->p)) { ev = ev * 10 + (*r->p++ - '0'); if (ev > 4096) { r->bad = 1; return; } }
    exp10 += es * ev;
  }
  /* value = digits x 10^exp10; drop leading zeros, fold trailing zeros into exp10 */
  int a = 0;
  while (a < nd && dig[a] == '0') a++;
  while (nd > a && dig[nd - 1] == '0') { nd--; exp10++; }
  if (a == nd) { snprintf(out, (size_t)outlen, "0"); return; }
  int m = nd - a;            /* significant digits */
  long ip = m + exp10;       /* digits before the decimal point */
  char buf[12000]; int k = 0;
  if (neg) buf[k++] = '-';
  if (ip <= 0) {
    buf[k++] = '0'; buf[k++] = '.';
    for (long i = 0; i < -ip && k < 11000; i++) buf[k++] = '0';
    for (int i = a; i < nd && k < 11990; i++) buf[k++] = dig[i];
  } else {
    for (long i = 0; i < ip && k < 11990; i++) buf[k++] = i < m ? dig[a + i] : '0';
    if (ip < m) { buf[k++] = '.'; for (int i = a + (int)ip; i < nd && k < 11990; i++) buf[k++] = dig[i]; }
  }
  buf[k] = 0;
  snprintf(out, (size_t)outlen, "%s", buf);
}

static void jvalue(jrd_t *r, jval_t *v, int depth);

static void jskip_container(jrd_t *r, char open, int depth) {
  (void)open;
  jval_t tmp;
  if (*r->p == '[') {
    r->p++; jws(r);
    if (r->p < r->e && *r->p == ']') { r->p++; return; }
    for (;;) {
      jvalue(r, &tmp, depth + 1); if (r->bad) return;
      jws(r);
      if (r->p < r->e && *r->p == ',') { r->p++; continue; }
      if (r->p < r->e && *r->p == ']') { r->p++; return; }
      r->bad = 1; return;
    }
  }
  r->p++; jws(r);
  if (r->p < r->e && *r->p == '}') { r->p++; return; }
  for (;;) {
    char key[256];
    jws(r);
    if (r->p >= r->e || *r->p != '"') { r->bad = 1; return; }
    jstring(r, key, sizeof key); if (r->bad) return;
    jws(r);
    if (r->p >= r->e || *r->p != ':') { r->bad = 1; return; }
    r->p++;
    jvalue(r, &tmp, depth + 1); if (r->bad) return;
    jws(r);
    if (r->p < r->e && *r->p == ',') { r->p++; continue; }
    if (r->p < r->e && *r->p == '}') { r->p++; return; }
    r->bad = 1; return;
  }
}

static void jvalue(jrd_t *r, jval_t *v, int depth) {
  jws(r);
  v->kind = JV_OTHER;
  v->nitems = 0;
  if (r->p >= r->e || depth > 64) { r->bad = 1; return; }
  char c = *r->p;
  if (c == '"') { v->kind = JV_SCALAR; jstring(r, v->text, sizeof v->text); return; }
  if (c == '-' || isdigit((unsigned char)c)) { v->kind = JV_SCALAR; jnumber(r, v->text, sizeof v->text); return; }
  if (c == 't' && r->e - r->p >= 4 && strncmp(r->p, "true", 4) == 0) { r->p += 4; v->kind = JV_TRUE; return; }
  if (c == 'f' && r->e - r->p >= 5 && strncmp(r->p, "false", 5) == 0) { r->p += 5; return; }
  if (c == 'n' && r->e - r->p >= 4 && strncmp(r->p, "null", 4) == 0) { r->p += 4; return; }
  if (c == '[') {
    /* keep the scalar items (for parametric atoms with several arguments) */
    v->kind = JV_ARRAY;
    r->p++; jws(r);
    if (r->p < r->e && *r->p == ']') { r->p++; return; }
    for (;;) {
      jval_t it;
      jvalue(r, &it, depth + 1); if (r->bad) return;
      if (v->nitems < JV_MAXITEMS) snprintf(v->items[v->nitems], 256, "%s", it.kind == JV_SCALAR ? it.text : "\x01");
      v->nitems++;
      jws(r);
      if (r->p < r->e && *r->p == ',') { r->p++; continue; }
      if (r->p < r->e && *r->p == ']') { r->p++; return; }
      r->bad = 1; return;
    }
  }
  if (c == '{') { jskip_container(r, '{', depth); return; }
  r->bad = 1;
}

struct orc_reader {
  const orc_prop *p;
  odict_t dict[ORC_MAX_LEVELS];
  /* per atom: predicate name and the level of each argument */
  char pred[MAXATOMS][128];
  int nargs[MAXATOMS];
  int argl[MAXATOMS][ORC_MAX_LEVELS];
};

orc_reader *orc_reader_new(const orc_prop *p) {
  orc_reader *r = (orc_reader *)calloc(1, sizeof(orc_reader));
  r->p = p;
  for (int j = 0; j < p->natoms; j++) {
    const char *nm = p->atoms[j];
    const char *lp = strchr(nm, '(');
    int len = lp ? (int)(lp - nm) : (int)strlen(nm);
    snprintf(r->pred[j], sizeof r->pred[j], "%.*s", len, nm);
    r->nargs[j] = 0;
    if (lp) {
      const char *a = lp + 1;
      while (*a && *a != ')') {
        char var[64]; int k = 0;
        while (*a && *a != ',' && *a != ')' && k < 63) var[k++] = *a++;
        var[k] = 0;
        for (int i = 0; i < p->nq; i++)
          if (strcmp(p->q[i].var, var) == 0 && r->nargs[j] < ORC_MAX_LEVELS) r->argl[j][r->nargs[j]++] = i;
        if (*a == ',') a++;
      }
    }
  }
  return r;
}

void orc_reader_free(orc_reader *r) {
  if (!r) return;
  for (int l = 0; l < ORC_MAX_LEVELS; l++) {
    for (uint64_t i = 0; i < r->dict[l].cap; i++) free(r->dict[l].slot[i].s);
    free(r->dict[l].slot);
  }
  free(r);
}

/* Read every record of text[0, len) and feed the monitor one event per record.
 * Returns the number of records, or -(line number) of the first malformed one. */
int64_t orc_feed_jsonl(orc_reader *rd, orc_monitor *m, const char *text, uint64_t len) {
  const orc_prop *p = rd->p;
  const char *s = text, *end = text + len;
  int64_t nrec = 0, line = 0;
  enum { MAXKV = 64 };
  static __thread char keys[MAXKV][128];
  static __thread jval_t vals[MAXKV];
  while (s < end) {
    const char *nl = memchr(s, '\n', (size_t)(end - s));
    const char *le = nl ? nl : end;
    line++;
    jrd_t r = {s, le, 0};
    jws(&r);
    if (r.p == le) { s = nl ? nl + 1 : end; continue; }
    int nkv = 0;
    if (*r.p != '{') return -line;
    r.p++; jws(&r);
    if (r.p < le && *r.p == '}') r.p++;
    else {
      for (;;) {
        char key[128]; jval_t v;
        jws(&r);
        if (r.p >= le || *r.p != '"') return -line;
        jstring(&r, key, sizeof key); if (r.bad) return -line;
        jws(&r);
        if (r.p >= le || *r.p != ':') return -line;
        r.p++;
        jvalue(&r, &v, 0); if (r.bad) return -line;
        /* one value per key (reading A11): a repeated key keeps its last value */
        int at = -1;
        for (int i = 0; i < nkv; i++) if (strcmp(keys[i], key) == 0) at = i;
        if (at < 0 && nkv < MAXKV) at = nkv++;
        if (at >= 0) { snprintf(keys[at], 128, "%s", key); vals[at] = v; }
        jws(&r);
        if (r.p < le && *r.p == ',') { r.p++; continue; }
        if (r.p < le && *r.p == '}') { r.p++; break; }
        return -line;
      }
    }
    jws(&r);
    if (r.p != le) return -line;
    /* epsilon(u_j, K): the value of each guard key p_i */
    uint32_t D[ORC_MAX_LEVELS];
    const char *gv[ORC_MAX_LEVELS];
    for (int i = 0; i < p->nq; i++) {
      gv[i] = NULL;
      for (int k = 0; k < nkv; k++)
        if (strcmp(keys[k], p->q[i].key) == 0 && vals[k].kind == JV_SCALAR) gv[i] = vals[k].text;
      D[i] = gv[i] ? odict_id(&rd->dict[i], gv[i]) : ORC_ABSENT;
    }
    uint8_t a = 0;
    for (int j = 0; j < p->natoms; j++) {
      const jval_t *v = NULL;
      for (int k = 0; k < nkv; k++) if (strcmp(keys[k], rd->pred[j]) == 0) v = &vals[k];
      if (!v) continue;
      int holds = v->kind == JV_TRUE;
      if (!holds && rd->nargs[j] == 1 && v->kind == JV_SCALAR)
        holds = gv[rd->argl[j][0]] && strcmp(gv[rd->argl[j][0]], v->text) == 0;
      if (!holds && rd->nargs[j] >= 1 && v->kind == JV_ARRAY && v->nitems == rd->nargs[j]) {
        holds = 1;
        for (int i = 0; i < rd->nargs[j]; i++) {
          const char *g = gv[rd->argl[j][i]];
          if (!g || strcmp(g, v->items[i]) != 0) holds = 0;
        }
      }
      if (holds) a |= (uint8_t)(1u << j);
    }
    const uint32_t *kp[ORC_MAX_LEVELS];
    uint32_t col[ORC_MAX_LEVELS][1];
    for (int i = 0; i < p->nq; i++) { col[i][0] = D[i]; kp[i] = col[i]; }
    orc_feed(m, 1, kp, &a);
    nrec++;
    s = nl ? nl + 1 : end;
  }
  return nrec;
}
