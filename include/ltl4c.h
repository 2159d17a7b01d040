/*
 * ltl4c.h -- C ABI of the B200-native LTL4-C verifier (libltl4c.so).
 *
 * Method: Medhat, Joshi, Bonakdarpour, Fischmeister, "Accelerated Runtime
 * Verification of LTL Specifications with Counting Semantics", arXiv:1411.2239.
 * `P:n` = line n of the paper text.  Readings of ambiguous passages (A1..A20)
 * are listed in DESIGN.md.
 *
 * Conventions for every entry point:
 *   - all calls return ltl4c_status; nothing throws across the ABI;
 *   - on a non-OK status, ltl4c_last_error() returns a thread-local message;
 *   - "device pointer" = CUDA global memory on the state's device, owned by the
 *     caller, read-only to the library, not retained after the call returns;
 *   - programs are immutable and may be shared between threads; a state has a
 *     single writer (calls on one state must not overlap).
 */
#ifndef LTL4C_H
#define LTL4C_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LTL4C_MAX_LEVELS 3      /* quantifier string length n (Eq. 5)        */
#define LTL4C_MAX_ATOMS 8       /* atoms of one formula's psi                       */
#define LTL4C_MAX_BATCH_ATOMS 16 /* atoms of a formula batch (letter classes > 8)    */
#define LTL4C_MAX_STATES 16     /* LTL4 monitor states (after minimisation/product) */
#define LTL4C_MAX_FORMULAS 4    /* formulas verified together (ltl4c_compile_batch) */
#define LTL4C_ABSENT 0xFFFFFFFFu /* key value meaning "the event does not bind it"  */

typedef enum {
  LTL4C_OK = 0,
  LTL4C_E_SYNTAX = 1,        /* bad token or grammar violation (Def. 3)      */
  LTL4C_E_NONCANONICAL = 2,  /* quantifier below a temporal/boolean operator    */
  LTL4C_E_UNBOUND = 3,       /* predicate argument not bound by the quantifier prefix   */
  LTL4C_E_RANGE = 4,         /* A constant outside [0,1] / >6 decimals, E constant < 0  */
  LTL4C_E_BUDGET = 5,        /* > 3 levels, > 8 atoms, > 16 monitor states, n = 0       */
  LTL4C_E_INVALID = 6,       /* null pointer, bad argument, non-contiguous online batch */
  LTL4C_E_CUDA = 7,          /* CUDA runtime error (message in ltl4c_last_error)        */
  LTL4C_E_NCCL = 8,          /* NCCL error                                              */
  LTL4C_E_OOM = 9,           /* device allocation failed                                */
  LTL4C_E_POISONED = 10      /* a previous verify failed mid-way; call ltl4c_state_reset */
} ltl4c_status;

/* six verdicts B6 in lattice order bottom < ... < top */
typedef enum {
  LTL4C_FALSE = 0,
  LTL4C_CURRENTLY_FALSE = 1,
  LTL4C_PRESUMABLY_FALSE = 2,
  LTL4C_PRESUMABLY_TRUE = 3,
  LTL4C_CURRENTLY_TRUE = 4,
  LTL4C_TRUE = 5
} ltl4c_verdict;

typedef enum { LTL4C_QUANT_A = 0, LTL4C_QUANT_E = 1 } ltl4c_quant_kind; /* A: percentage, E: instance */
typedef enum { LTL4C_LT = 0, LTL4C_LE = 1, LTL4C_GT = 2, LTL4C_GE = 3, LTL4C_EQ = 4 } ltl4c_cmp;

typedef struct ltl4c_program ltl4c_program;
typedef struct ltl4c_state ltl4c_state;

/* One counting quantifier Q_i = <Q_i, ~_i, c_i, x_i, p_i> (Eq. 5).
 * A: c = num/den, a reduced fraction in [0,1] (reading A5);  E: c = num, den = 1. */
typedef struct {
  int32_t kind; /* ltl4c_quant_kind */
  int32_t cmp;  /* ltl4c_cmp        */
  uint64_t num, den;
  char key[64]; /* guard predicate p_i = the event key holding x_i's value */
} ltl4c_quantifier;

/* Read-only view of a compiled program (host memory owned by the program).
 * Letters: a valuation of the atoms is a bitmask m (bit j = atom j, Def. 1/2);
 * the batches carry its LETTER CODE: m itself when n_atoms <= 8 (letter_bits =
 * n_atoms, letter_class = NULL); for a formula batch over 9..16 atoms, the class
 * letter_class[m] of m, letters of one class acting identically on every state of
 * the product monitor (letter equivalence classes; at most
 * 256 classes, else E_BUDGET), codes < 1 << letter_bits.
 * delta[q * (1 << letter_bits) + code] is the LTL4 monitor transition (Def. 5,
 * P:326-336) of the (product) automaton; label[f * n_states + q] is lambda_f(q) in
 * B6 codes {0,2,3,5}; states with label 0/5 are traps. */
typedef struct {
  uint32_t n_formulas, n_levels, n_atoms, n_states, initial;
  const uint8_t *delta;
  const uint8_t *label;
  const ltl4c_quantifier *quant; /* [n_formulas][n_levels] */
  const char *const *atom_names; /* [n_atoms], bit j of a valuation = atom j          */
  uint32_t letter_bits;          /* codes are < 1 << letter_bits                      */
  const uint8_t *letter_class;   /* [1 << n_atoms] code of each valuation, or NULL    */
} ltl4c_tables;

/* A trace batch u (Def. 2) in encoded form, n_events events.
 * keys[i][j]  : value of guard key i (quantifier level i) in event j, or LTL4C_ABSENT;
 *               an event binding every key has value vector D = (keys[0][j] ...
 *               keys[n-1][j]) (epsilon; Eq. D); others bind no vector.
 * letters[j]  : the letter code of event j: bit k set iff atom k of the program holds
 *               (programs of <= 8 atoms), else the class of that valuation
 *               (ltl4c_tables.letter_class).
 * first_index : global index of event 0; for an online state it must equal the
 *               previous batch's first_index + n_events (else LTL4C_E_INVALID).
 * Pointers are device pointers for ltl4c_verify and host pointers for
 * ltl4c_verify_host.  n_events may be 0 (pointers may then be NULL). */
typedef struct {
  uint64_t n_events;
  uint64_t first_index;
  const uint32_t *keys[LTL4C_MAX_LEVELS];
  const uint8_t *letters;
} ltl4c_batch;

/* Result of Algorithm 1 after the batch, per formula.
 * hist[l][v] = number of depth-l nodes of the submonitor tree (Fig. 2) with
 * verdict v: l = 0 is the root (one-hot of `verdict`), l = n_levels the leaves
 * (LTL4 submonitors, verdicts in {0,2,3,5}).  For an online state these are the
 * values for the concatenation of all batches since create/reset. */
typedef struct {
  int32_t verdict; /* ltl4c_verdict of the root */
  uint32_t n_levels;
  uint64_t hist[LTL4C_MAX_LEVELS + 1][6];
  uint64_t events_seen;  /* events consumed so far            */
  uint64_t events_bound; /* of those, events binding every key */
} ltl4c_result;

/* Per-state counters for benchmarking (kernel launches and CUDA-event times of
 * the library's kernels, accumulated while profiling is enabled). */
#define LTL4C_MAX_KERNELS 16
typedef struct {
  uint64_t verifies;
  uint64_t launches;                 /* kernels launched by the library */
  uint32_t n_kernels;
  char kernel_name[LTL4C_MAX_KERNELS][32];
  uint64_t kernel_launches[LTL4C_MAX_KERNELS];
  double kernel_ms[LTL4C_MAX_KERNELS]; /* sum of CUDA-event durations          */
} ltl4c_stats;

/* --- programs (host only) -------------------------------------------------- */

/* Parse an LTL4-C property (Def. 3; grammar in DESIGN.md "Surface syntax") and
 * synthesise its LTL4 monitor (Def. 5; construction in DESIGN.md "Compiler").
 * Errors: E_SYNTAX, E_NONCANONICAL, E_UNBOUND, E_RANGE, E_BUDGET, E_INVALID. */
ltl4c_status ltl4c_compile(const char *formula_utf8, ltl4c_program **out);

/* F <= LTL4C_MAX_FORMULAS formulas with the same guard-key string, verified in
 * one pass (reading A20).  Atoms are the union in order of first occurrence
 * (formula 0's atoms first); the monitor is the minimised product automaton. */
ltl4c_status ltl4c_compile_batch(const char *const *formulas_utf8, int n_formulas,
                                 ltl4c_program **out);

/* Fill *view with pointers into the program (valid until ltl4c_program_free). */
ltl4c_status ltl4c_program_tables(const ltl4c_program *prog, ltl4c_tables *view);

void ltl4c_program_free(ltl4c_program *prog);

/* --- states (device) ------------------------------------------------------- */

#define LTL4C_STATE_ONLINE 1u /* carry the submonitor tree across verify calls */

/* Create a verification state on CUDA device `device`.  capacity_hint: expected
 * events per batch (buffers grow on demand).  flags: 0 = offline (every verify
 * evaluates its batch alone), LTL4C_STATE_ONLINE = online. */
ltl4c_status ltl4c_state_create(const ltl4c_program *prog, int device, uint64_t capacity_hint,
                                uint32_t flags, ltl4c_state **out);

/* Multi-GPU: rank 0 creates a 128-byte ncclUniqueId with
 * ltl4c_nccl_unique_id and the caller broadcasts it (e.g. torch.distributed);
 * every rank then calls ltl4c_state_comm before its first verify.  n_ranks must
 * be a power of two <= 256.  Afterwards each ltl4c_verify call takes this rank's
 * contiguous slice of the trace (rank r's events precede rank r+1's), routes
 * every bound event to its owner rank (a hash of k0: every tree node below the
 * root lives on one rank), exchanges them with NCCL send/recv over NVLink, runs
 * the local pipeline on the owned events and all-reduces the per-level counts;
 * every rank returns the global result.  Errors: E_INVALID, E_NCCL, E_OOM. */
ltl4c_status ltl4c_nccl_unique_id(void *out128);
ltl4c_status ltl4c_state_comm(ltl4c_state *st, const void *nccl_id, int n_ranks, int rank);

/* Run Algorithm 1 on one batch of device-resident events.  Work is enqueued on
 * `cuda_stream` (a cudaStream_t; NULL = legacy default stream); the call returns
 * after the <= 200-byte result has been copied to *out (one per formula: out
 * must hold n_formulas results).  On error the state is poisoned (online) or
 * unchanged (offline). */
ltl4c_status ltl4c_verify(ltl4c_state *st, const ltl4c_batch *batch, void *cuda_stream,
                          ltl4c_result *out);

/* As ltl4c_verify, but batch pointers are HOST pointers: the library copies the
 * events to device buffers it owns (cudaMemcpyAsync on `cuda_stream`; pinned
 * host memory gives asynchronous copies), then verifies. */
ltl4c_status ltl4c_verify_host(ltl4c_state *st, const ltl4c_batch *batch, void *cuda_stream,
                               ltl4c_result *out);

/* Pipelined online monitoring (a stream of batches): enqueue one batch
 * of an online state on `cuda_stream` and return at once with a ticket; the
 * result is read later with ltl4c_result_get(ticket) (which waits for that
 * batch only).  All batches of a state go on the same stream.  Batches must be
 * contiguous as for ltl4c_verify, their device
 * buffers must stay valid until the result is read, and at most 8 results may
 * be outstanding (E_INVALID otherwise).  Single-GPU states only.  Carried tables
 * grow on the bound "leaves of the last read result + events enqueued since".
 * Errors: E_INVALID (offline state, communicator, too many outstanding, bad
 * ticket), E_CUDA, E_OOM (table overflow: the state is poisoned). */
ltl4c_status ltl4c_verify_async(ltl4c_state *st, const ltl4c_batch *batch, void *cuda_stream,
                                uint64_t *ticket);
ltl4c_status ltl4c_result_get(ltl4c_state *st, uint64_t ticket, ltl4c_result *out);

/* Forget all carried state (online) and clear the poisoned flag. */
ltl4c_status ltl4c_state_reset(ltl4c_state *st);

void ltl4c_state_free(ltl4c_state *st);

/* Checkpoint / restore of an ONLINE state's carried state (
 * the paper keeps the submonitor tree across invocations): the submonitor
 * set 𝔻 (every leaf's value vector and monitor state, Def. 5), every
 * quantifier node with its child histogram and verdict (Def. 6/7), the
 * per-level counts and the stream position.  The blob is host memory owned by the
 * caller, opaque, for the same program (checked by a fingerprint of its tables).
 *   ltl4c_state_checkpoint_size: bytes a checkpoint of `st` takes now;
 *   ltl4c_state_checkpoint: drains the state's batches in flight, writes the blob
 *     to buf[0 .. cap) (*written = its size);
 *   ltl4c_state_restore: replaces the carried state of an online state created
 *     from the same program (tables reallocated to the checkpoint's capacities);
 *     later batches continue the stream exactly as the checkpointed state would.
 * Errors: E_INVALID (null argument, offline state, cap too small, not a
 * checkpoint, other program), E_CUDA, E_OOM. */
ltl4c_status ltl4c_state_checkpoint_size(ltl4c_state *st, uint64_t *bytes);
ltl4c_status ltl4c_state_checkpoint(ltl4c_state *st, void *buf, uint64_t cap, uint64_t *written);
ltl4c_status ltl4c_state_restore(ltl4c_state *st, const void *buf, uint64_t len);

/* Compaction of an ONLINE state's carried tables (NEXT-3): the tables are rehashed
 * into the smallest power-of-two capacities that hold the live leaves and nodes
 * at load <= 1/2 (they only ever grow while batches run); results are unchanged.
 * Drains batches in flight.  Errors: E_INVALID (null or offline state), E_CUDA, E_OOM. */
ltl4c_status ltl4c_state_compact(ltl4c_state *st);

/* Explain / dump of an ONLINE state's carried tree (the
 * quantifier tree of §3.3, Fig. 2): the nodes of depth `level`
 * (1 <= level <= n_levels; depth n_levels = the leaves, i.e. the submonitors of
 * 𝔻) with their current verdict for formula `formula` -- Def. 6 for inner nodes
 * (P:648-675), lambda of the monitor state for leaves (Def. 5).
 * Writes at most `cap` nodes: keys[i][j] (i < level) = the value vector of node j,
 * verdicts[j] = its B6 code (ltl4c_verdict); *count = the nodes at that depth (all
 * of them, even beyond cap).  Order unspecified.  Buffers are HOST memory owned by
 * the caller (keys: `level` arrays of cap u32; either may be null when cap = 0).
 * Errors: E_INVALID (null state/count, offline state, level or formula out of
 * range), E_CUDA. */
ltl4c_status ltl4c_state_nodes(ltl4c_state *st, uint32_t level, uint32_t formula, uint32_t *const *keys,
                               uint8_t *verdicts, uint64_t cap, uint64_t *count);

/* Kernel-level profiling: when enabled, every library kernel launch is bracketed
 * by CUDA events on the stream it runs on; ltl4c_state_stats sums them (this
 * synchronises the stream).  ltl4c_state_stats_reset zeroes the counters. */
ltl4c_status ltl4c_state_profile(ltl4c_state *st, int enable);
ltl4c_status ltl4c_state_stats(ltl4c_state *st, ltl4c_stats *out);
ltl4c_status ltl4c_state_stats_reset(ltl4c_state *st);

/* --- trace encoder (host) ------------------------------------------------- */

/* Turns key -> value records into the encoded batch layout above: arXiv:1411.2239
 * §4.1 "Valuation Extraction" ("the trace event is a key-value
 * structure"; epsilon(u_i, K)), Def. 1/2.  Input: JSON lines, one
 * object per line (UTF-8; blank lines skipped; other JSON values are E_SYNTAX).
 *   keys[l][j]  = dense id of event j's value of guard key p_l (the key named by
 *                 quantifier l), or LTL4C_ABSENT if the record maps p_l to no
 *                 string/number.  Values are identified by their canonical string
 *                 (strings as written; numbers as canonical decimals: 12, 12.0,
 *                 1.2e1 and "12" are one value).  Ids are 0, 1, 2, ... per level in
 *                 order of first appearance and persist for the encoder's life
 *                 (the batches of an online stream share them).
 *   letters[j]  bit a = atom a of the program holds: a 0-ary atom q holds iff the
 *                 record maps q to true; a parametric atom q(x_i, ...) holds iff
 *                 the record maps q to true or to the event's own value(s) of
 *                 x_i, ... (a scalar for one argument, an array in argument order
 *                 for several) -- reading A12.  Other keys are ignored.
 * Reads whole lines from text[0 .. len) until `capacity` events are written;
 * *consumed = bytes read (resume there), *n_events = events written.  Buffers are
 * HOST memory owned by the caller (keys: n_levels arrays of `capacity` u32).
 * Errors: E_INVALID (null argument), E_SYNTAX (malformed record; the message
 * names the record number; nothing of that record is written), E_BUDGET (more
 * than 2^32 - 1 distinct values of one key).  An encoder is single-threaded. */
typedef struct ltl4c_encoder ltl4c_encoder;
ltl4c_status ltl4c_encoder_create(const ltl4c_program *prog, ltl4c_encoder **out);
ltl4c_status ltl4c_encode_jsonl(ltl4c_encoder *enc, const char *text, uint64_t len,
                                uint32_t *const *keys, uint8_t *letters, uint64_t capacity,
                                uint64_t *n_events, uint64_t *consumed);
/* number of distinct values of guard key `level` seen so far */
ltl4c_status ltl4c_encoder_values(const ltl4c_encoder *enc, uint32_t level, uint64_t *count);
void ltl4c_encoder_free(ltl4c_encoder *enc);

/* --- trace ingest on the device ----------------------- */

/* The host encoder's semantics (above; §4.1 Valuation Extraction, P:915-935,
 * reading A12) run on the GPU over JSON-lines text in DEVICE memory -- the stage
 * upstream of the hot path that the paper measures as its strace parsing module
 * (P:1087-1094).  One record per line; blank lines are skipped.
 * Dictionary ids are dense per level (0, 1, ... < ltl4c_dencoder_values) and
 * persist across calls of one encoder, but are assigned in the order concurrent
 * threads first claim a value (not first appearance): only the partition of values
 * into ids is the host encoder's, and verdicts and counts depend on nothing else.
 * Values are identified by a 64-bit hash of their canonical string (DESIGN.md
 * A28).  `max_values` = capacity of each level's dictionary.
 * ltl4c_dencode_jsonl: text = DEVICE pointer, len bytes; keys (n_levels DEVICE
 * arrays) and letters (DEVICE) receive one event per record in line order;
 * capacity = their length.  The call synchronises `cuda_stream`.  Errors:
 * E_INVALID (null argument; more records than capacity: *n_events = the number
 * needed, nothing written), E_SYNTAX (malformed record: the message names the
 * first bad line, nothing written), E_BUDGET (a dictionary is full), E_CUDA, E_OOM. */
typedef struct ltl4c_dencoder ltl4c_dencoder;
ltl4c_status ltl4c_dencoder_create(const ltl4c_program *prog, int device, uint64_t max_values, ltl4c_dencoder **out);
ltl4c_status ltl4c_dencode_jsonl(ltl4c_dencoder *enc, const char *text, uint64_t len, uint32_t *const *keys,
                                 uint8_t *letters, uint64_t capacity, uint64_t *n_events, void *cuda_stream);
ltl4c_status ltl4c_dencoder_values(const ltl4c_dencoder *enc, uint32_t level, uint64_t *count);
void ltl4c_dencoder_free(ltl4c_dencoder *enc);

/* Thread-local message of the last non-OK status ("" if none). */
const char *ltl4c_last_error(void);

/* Library version string, e.g. "ltl4c 0.1 sm_100a". */
const char *ltl4c_version(void);

#ifdef __cplusplus
}
#endif
#endif /* LTL4C_H */
