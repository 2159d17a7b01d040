/*
 * oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, obviously-correct CPU interpreter of the LTL4-C semantics of
 * Medhat, Joshi, Bonakdarpour, Fischmeister, "Accelerated Runtime Verification
 * of LTL Specifications with Counting Semantics" (arXiv:1411.2239).
 * `P:n` below is line n of the paper text; readings of ambiguous
 * passages are listed in DESIGN.md ("Readings") and tagged A1..A20.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * `--impl reference` leg may load this library.  It shares no code, header,
 * table or constant with the product (paper_1411_2239_b200/).
 *
 * Verdict codes follow the B6 lattice order of P:366:
 *   0 = FALSE (⊥), 1 = CURRENTLY_FALSE (⊥c), 2 = PRESUMABLY_FALSE (⊥p),
 *   3 = PRESUMABLY_TRUE (⊤p), 4 = CURRENTLY_TRUE (⊤c), 5 = TRUE (⊤).
 */
#ifndef LTL4C_ORACLE_H
#define LTL4C_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ORC_MAX_LEVELS 3
#define ORC_ABSENT 0xFFFFFFFFu

/* error codes of orc_parse (same meaning as SPEC's parse errors) */
enum { ORC_OK = 0, ORC_E_SYNTAX = 1, ORC_E_NONCANONICAL = 2, ORC_E_UNBOUND = 3,
       ORC_E_RANGE = 4, ORC_E_BUDGET = 5 };

/* quantifier kinds / comparison operators (Def. 3) */
enum { ORC_Q_A = 0, ORC_Q_E = 1 };
enum { ORC_LT = 0, ORC_LE = 1, ORC_GT = 2, ORC_GE = 3, ORC_EQ = 4 };

typedef struct orc_prop orc_prop;
typedef struct orc_monitor orc_monitor;

int  orc_parse(const char *text, orc_prop **out, char *err, int errlen);
void orc_prop_free(orc_prop *p);
int  orc_num_levels(const orc_prop *p);
int  orc_num_atoms(const orc_prop *p);
/* writes "name(args)" of atom j (bit j of a letter) */
int  orc_atom_name(const orc_prop *p, int j, char *buf, int buflen);
/* quantifier i: kind, cmp, num, den (E: den = 1), guard key name */
int  orc_quantifier(const orc_prop *p, int i, int *kind, int *cmp, uint64_t *num,
                    uint64_t *den, char *key, int keylen);

/* [u |=_4 psi] of the inner formula on a single word (Def. 4) */
int  orc_ltl4_word(const orc_prop *p, const uint8_t *word, int len);
/* [u |=_F psi] (FLTL); 1 = true, 0 = false; len >= 1 */
int  orc_fltl_word(const orc_prop *p, const uint8_t *word, int len);

/* Def. 6 node verdict for one quantifier from the child-verdict histogram */
int  orc_rule(int kind, int cmp, uint64_t num, uint64_t den, const uint64_t h[6]);

/* Algorithm 1 over a stream of events (offline = one feed, online = many) */
orc_monitor *orc_monitor_new(const orc_prop *p);
void orc_monitor_free(orc_monitor *m);
/* keys[i][j] = value of guard key i in event j (ORC_ABSENT if unbound) */
int  orc_feed(orc_monitor *m, uint64_t n, const uint32_t *const *keys,
              const uint8_t *letters);
/* verdict of the root, hist[l][v] = #nodes at depth l with verdict v
 * (l = 0 root ... l = n leaves), events seen / guard-complete */
int  orc_evaluate(orc_monitor *m, int *verdict, uint64_t hist[ORC_MAX_LEVELS + 1][6],
                  uint64_t *events_seen, uint64_t *events_bound);
/* verdict of the node identified by a partial vector D|^m (m <= n);
 * returns -1 if the vector is not in the tree (after orc_evaluate) */
int  orc_node_verdict(orc_monitor *m, int m_len, const uint32_t *prefix);

/* Timing mode: the same result computed by T threads,
 * level-0 subtrees partitioned by a hash of k0 (results identical for every T). */
int  orc_run_threads(const orc_prop *p, uint64_t n, const uint32_t *const *keys,
                     const uint8_t *letters, int T, int *verdict,
                     uint64_t hist[ORC_MAX_LEVELS + 1][6], uint64_t *events_seen,
                     uint64_t *events_bound);

/* Records (JSON lines, one key -> value object per line) read by the oracle's
 * own reader and fed to a monitor one event per record; returns the number of
 * records, or -(line) of the first malformed record. */
typedef struct orc_reader orc_reader;
orc_reader *orc_reader_new(const orc_prop *p);
void orc_reader_free(orc_reader *r);
int64_t orc_feed_jsonl(orc_reader *r, orc_monitor *m, const char *text, uint64_t len);

#ifdef __cplusplus
}
#endif
#endif
