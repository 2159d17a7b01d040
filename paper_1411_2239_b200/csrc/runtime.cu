// runtime.cu -- C ABI (include/ltl4c.h): states, buffers, launch orchestration.
//
// One ltl4c_verify = Algorithm 1 of arXiv:1411.2239 on a batch:
//   SortTrace       -> P stable LSD passes (part_count, part_scan, part_scatter)
//                      + bucket_bounds (mu) + unit_start          (a1, a2)
//   SpawnMonitors,
//   Distribute,
//   ApplyQuantifiers -> offline: bucket_warp -> bucket_warp_big -> bucket_fast
//                      -> heavy (each takes what the previous one spills);
//                      online: online_leaf + online_nodes per level  (a3-a5)
//   return           -> finalize + one <= 1 KB D2H copy              (a6)
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "kernels.cuh"
#include "program.h"

namespace ltl4c {

static thread_local std::string g_err;

ltl4c_status fail(ltl4c_status st, const std::string &msg) {
  g_err = msg;
  return st;
}

#define CU(expr)                                                                          \
  do {                                                                                    \
    cudaError_t e_ = (expr);                                                              \
    if (e_ != cudaSuccess)                                                                \
      return fail(e_ == cudaErrorMemoryAllocation ? LTL4C_E_OOM : LTL4C_E_CUDA,           \
                  std::string(#expr) + ": " + cudaGetErrorString(e_));                    \
  } while (0)

template <class T>
struct DevBuf {
  T *p = nullptr;
  size_t n = 0;
  cudaError_t ensure(size_t want) {
    if (want <= n && p) return cudaSuccess;
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
    size_t cap = std::max<size_t>(want, 1);
    cudaError_t e = cudaMalloc((void **)&p, cap * sizeof(T));
    if (e != cudaSuccess) return e;
    n = cap;
    // zero once per allocation: 16-byte staging loads read the padding past N and the
    // result copy reads unused DevOut fields (harmless values, but defined for initcheck)
    e = cudaMemset(p, 0, cap * sizeof(T));
    if (e == cudaSuccess) e = cudaStreamSynchronize(0);
    return e;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
};

struct Tables {
  DevTables d{};
  DevBuf<uint4> leaf_slot;
  DevBuf<uint8_t> leaf_state;
  DevBuf<uint32_t> leaf_aux;
  DevBuf<uint32_t> node_aux[kMaxLevels];
  DevBuf<uint4> node_slot[kMaxLevels];
  DevBuf<uint32_t> node_verdict[kMaxLevels];
  DevBuf<uint32_t> node_hist[kMaxLevels];
  void release() {
    leaf_slot.release();
    leaf_state.release();
    leaf_aux.release();
    for (int l = 0; l < kMaxLevels; ++l) {
      node_aux[l].release();
      node_slot[l].release();
      node_verdict[l].release();
      node_hist[l].release();
    }
    d = DevTables{};
  }
};

struct PendingTiming {
  int kernel;
  cudaEvent_t a, b;
};

// NCCL, resolved at run time (the copy torch already loaded, else the system one)
struct NcclId { char internal[128]; };
struct Nccl {
  void *h = nullptr;
  int (*GetUniqueId)(NcclId *) = nullptr;
  int (*CommInitRank)(void **, int, NcclId, int) = nullptr;
  int (*CommDestroy)(void *) = nullptr;
  int (*Send)(const void *, size_t, int, int, void *, cudaStream_t) = nullptr;
  int (*Recv)(void *, size_t, int, int, void *, cudaStream_t) = nullptr;
  int (*GroupStart)() = nullptr;
  int (*GroupEnd)() = nullptr;
  int (*AllReduce)(const void *, void *, size_t, int, int, void *, cudaStream_t) = nullptr;
  int (*AllGather)(const void *, void *, size_t, int, void *, cudaStream_t) = nullptr;
  const char *(*ErrStr)(int) = nullptr;
};
enum { kNcclUint8 = 1, kNcclUint32 = 3, kNcclUint64 = 5, kNcclSum = 0 };

Nccl *nccl() {
  static Nccl n;
  static bool tried = false;
  if (tried) return n.h ? &n : nullptr;
  tried = true;
  const char *names[] = {"libnccl.so.2", "libnccl.so", "/usr/lib/x86_64-linux-gnu/libnccl.so.2"};
  for (const char *nm : names) {
    n.h = dlopen(nm, RTLD_NOW | RTLD_GLOBAL);
    if (n.h) break;
  }
  if (!n.h) return nullptr;
  n.GetUniqueId = (decltype(n.GetUniqueId))dlsym(n.h, "ncclGetUniqueId");
  n.CommInitRank = (decltype(n.CommInitRank))dlsym(n.h, "ncclCommInitRank");
  n.CommDestroy = (decltype(n.CommDestroy))dlsym(n.h, "ncclCommDestroy");
  n.Send = (decltype(n.Send))dlsym(n.h, "ncclSend");
  n.Recv = (decltype(n.Recv))dlsym(n.h, "ncclRecv");
  n.GroupStart = (decltype(n.GroupStart))dlsym(n.h, "ncclGroupStart");
  n.GroupEnd = (decltype(n.GroupEnd))dlsym(n.h, "ncclGroupEnd");
  n.AllReduce = (decltype(n.AllReduce))dlsym(n.h, "ncclAllReduce");
  n.AllGather = (decltype(n.AllGather))dlsym(n.h, "ncclAllGather");
  n.ErrStr = (decltype(n.ErrStr))dlsym(n.h, "ncclGetErrorString");
  if (!n.GetUniqueId || !n.CommInitRank || !n.Send || !n.Recv || !n.GroupStart || !n.GroupEnd || !n.AllReduce ||
      !n.AllGather) {
    dlclose(n.h);
    n.h = nullptr;
    return nullptr;
  }
  return &n;
}

#define NC(expr)                                                                                   \
  do {                                                                                             \
    int r_ = (expr);                                                                               \
    if (r_ != 0) return fail(LTL4C_E_NCCL, std::string(#expr) + ": " + (nccl()->ErrStr ? nccl()->ErrStr(r_) : "error")); \
  } while (0)

}  // namespace ltl4c

using namespace ltl4c;

struct ltl4c_state {
  const ltl4c_program *prog = nullptr;
  int device = 0;
  uint32_t flags = 0;
  bool poisoned = false;
  uint64_t next_index = 0;
  bool have_index = false;
  uint64_t events_seen = 0;
  uint32_t epoch = 1;
  DevProg hprog{};
  DevBuf<DevProg> d_prog;
  DevBuf<DevAcc> d_acc;
  DevBuf<DevOut> d_out;
  DevOut *h_out = nullptr;  // pinned
  DevBuf<unsigned long long> d_nvalid;
  DevBuf<uint32_t> bufkey[2][kMaxLevels];
  DevBuf<uint8_t> buflet[2];
  DevBuf<uint32_t> totals, counts, bucket_off, oversize_list, medium_list, large_list, sched, unit_start;
  int n_sms = 148;
  int warp_cfg[4] = {4, 1, 1, 1};  // {warps/CTA, CTAs/SM} of the unit and the medium warp kernels
  int online_cfg[2] = {4, 1};      // {warps/CTA, CTAs/SM} of online_leaf
  // pipelined online batches (ltl4c_verify_async / ltl4c_result_get): results land
  // in a ring of pinned slots; table growth uses an upper bound of the carried
  // leaves (the last read result + every event enqueued after it)
  static constexpr int kRing = 8;
  DevOut *ring_out = nullptr;                 // pinned [kRing]
  cudaEvent_t ring_ev[kRing] = {};
  uint64_t ring_ticket[kRing] = {};           // 0: free / consumed
  uint64_t ring_seen[kRing] = {}, ring_cum[kRing] = {};
  uint64_t next_ticket = 1, enq_events = 0, outstanding = 0;
  uint64_t known_leaves = 0, known_nodes[kMaxLevels] = {}, known_cum = 0;
  uint32_t batch_id = 0;           // online: touch mark of the current batch
  DevBuf<uint32_t> tlist[kMaxLevels], tcnt;
  DevBuf<uint32_t> d_bid;          // online: the batch id as the kernels read it (set per batch, graphs replay)
  DevBuf<uint32_t> hkeys[kMaxLevels];  // staging for ltl4c_verify_host
  DevBuf<uint8_t> hlet;
  uint8_t *h_pack = nullptr;       // small host batches: pinned staging block (one H2D copy per verify)
  cudaEvent_t pack_done = nullptr; //   recorded after its copy (the block is not refilled before)
  DevBuf<uint8_t> d_pack;          //   its device copy (fixed size: the same layout every call)
  Tables tab;
  // multi-GPU (ltl4c_state_comm)
  void *comm = nullptr;
  int n_ranks = 1, rank = 0, owner_bits = 0;
  bool force_exchange = false;  // LTL4C_FORCE_EXCHANGE: run the exchange path with 1 rank (tests)
  // tuning / test knobs, read from the environment once per state (ltl4c_state_create)
  uint64_t bucket_mul = 6;         // LTL4C_BUCKET_MUL: buckets per kWarpCap events
  int max_bits = kMaxPasses * kMaxDigitBits;  // LTL4C_MAX_BITS: cap on the bucket bits
  bool max_bits_set = false;
  uint32_t warp_grid = 0;          // LTL4C_WARP_GRID: cap on the warp kernels' grids (0 = none)
  int vshards = 1;                 // LTL4C_VIRTUAL_SHARDS: test-only owner shards on one GPU (run_virtual)
  int rank_ballot = 1;             // LTL4C_RANK_BALLOT: stable rank by ballots (1) or match.any (0)
  bool hot = true;                 // LTL4C_NO_HOT: no heavy-hitter path for K = 1 (hot.cu)
  DevBuf<uint32_t> hot_cnt, hot_tab, hot_partial;  // sample counts [2][cap], slot keys + nhot, chunk maps
  DevBuf<uint32_t> hot_chunk;      // cold events per chunk
  DevBuf<unsigned long long> hot_n;  // cold events in the batch
  int hot_per_sm = 2;              // resident hot_compose CTAs per SM
  int hot_mapk = -1;               // map kind of the program (hot.cu), -1: no hot path
  bool seg = true;                 // LTL4C_NO_SEG: K = 1 units through bucket_warp instead of bucket_seg
  uint32_t seg_unit = 1024;        // LTL4C_SEG_UNIT: events per bucket_seg unit
  bool coarse = true;              // LTL4C_NO_COARSE: no one-pass mode for K = 1 hot batches
  int coarse_per_sm = 2;
  int force_onepass = 0;           // LTL4C_FORCE_ONEPASS (tests): one-pass mode whatever the sample says
  DevBuf<uint32_t> coarse_off;     // one-pass mode: coarse bucket offsets
  DevBuf<uint32_t> unit_start2;    // bucket_seg units
  int seg_per_sm = 4;              // resident bucket_seg CTAs per SM
  DevBuf<DevAcc> d_gacc, d_sacc;                 // all-reduced result, shard-pass scratch
  DevBuf<uint32_t> exkey[kMaxLevels];
  DevBuf<uint8_t> exlet;
  DevBuf<unsigned long long> dc_cnt;             // [G] own counts, [G][G] all-gathered
  unsigned long long *hc_cnt = nullptr;          // pinned [G + G*G]
  // heavy path buffers
  DevBuf<uint4> h_part, h_lists;
  DevBuf<uint32_t> h_u32;  // seg_base | leaf_slot_of | leaf_npart | leaf_off | leaf_fill | long_list | scan_tmp | node lists
  DevBuf<unsigned long long> h_cnt;
  // stats / profiling
  bool profiling = false;
  uint64_t verifies = 0, launches = 0;
  uint64_t k_launches[kKNumKernels] = {};
  double k_ms[kKNumKernels] = {};
  std::vector<PendingTiming> pending;
  std::vector<cudaEvent_t> event_pool;
  cudaStream_t cur_stream = nullptr;
  // CUDA graph of the offline launch sequence
  bool graphs = true;
  cudaStream_t cap_stream = nullptr;
  cudaGraphExec_t graph_exec = nullptr;
  std::vector<uintptr_t> graph_key;
  std::vector<uintptr_t> graph_pending;  // online: the last layout run directly (captured if seen again)
  uint64_t graph_kernels = 0;
  uint64_t k_launches_saved[kKNumKernels] = {};
};

namespace {

cudaEvent_t take_event(ltl4c_state *st) {
  if (!st->event_pool.empty()) {
    cudaEvent_t e = st->event_pool.back();
    st->event_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}

void before_launch(void *ctx, int k) {
  auto *st = (ltl4c_state *)ctx;
  if (!st->profiling) return;
  PendingTiming t{k, take_event(st), take_event(st)};
  cudaEventRecord(t.a, st->cur_stream);
  st->pending.push_back(t);
}

void after_launch(void *ctx, int k) {
  auto *st = (ltl4c_state *)ctx;
  st->launches++;
  st->k_launches[k]++;
  static const bool sync_debug = std::getenv("LTL4C_SYNC_DEBUG") != nullptr;
  if (sync_debug) {
    std::fprintf(stderr, "[ltl4c] launched %s ...", kKernelNames[k]);
    cudaError_t e = cudaStreamSynchronize(st->cur_stream);
    std::fprintf(stderr, " done (%s)\n", cudaGetErrorString(e));
  }
  if (!st->profiling || st->pending.empty()) return;
  cudaEventRecord(st->pending.back().b, st->cur_stream);
}

void drain_timings(ltl4c_state *st) {
  for (auto &t : st->pending) {
    float ms = 0.f;
    cudaEventSynchronize(t.b);
    if (cudaEventElapsedTime(&ms, t.a, t.b) == cudaSuccess) st->k_ms[t.kernel] += ms;
    st->event_pool.push_back(t.a);
    st->event_pool.push_back(t.b);
  }
  st->pending.clear();
}

int ceil_log2(uint64_t x) {
  int b = 0;
  while ((1ull << b) < x) ++b;
  return b;
}

ltl4c_status alloc_tables(ltl4c_state *st, Tables &t, uint64_t leaf_cap, uint64_t node_cap, cudaStream_t s,
                          bool aux = false, bool node_marks = false) {
  const int nl = (int)st->prog->n_levels;
  CU(t.leaf_slot.ensure(leaf_cap));
  CU(t.leaf_state.ensure(leaf_cap));
  if (aux) {
    CU(t.leaf_aux.ensure(leaf_cap));
    t.d.leaf_aux = t.leaf_aux.p;
  }
  CU(cudaMemsetAsync(t.leaf_slot.p, 0, sizeof(uint4) * leaf_cap, s));
  t.d.leaf_cap = leaf_cap;
  t.d.leaf_slot = t.leaf_slot.p;
  t.d.leaf_state = t.leaf_state.p;
  for (int l = 1; l < nl; ++l) {
    CU(t.node_slot[l].ensure(node_cap));
    CU(t.node_verdict[l].ensure(node_cap));
    CU(t.node_hist[l].ensure(node_cap * kMaxFormulas * 6));
    CU(cudaMemsetAsync(t.node_slot[l].p, 0, sizeof(uint4) * node_cap, s));
    if (aux || node_marks) {
      CU(t.node_aux[l].ensure(node_cap));
      t.d.node_aux[l] = t.node_aux[l].p;
      if (node_marks) CU(cudaMemsetAsync(t.node_aux[l].p, 0, sizeof(uint32_t) * node_cap, s));
    }
    t.d.node_cap[l] = node_cap;
    t.d.node_slot[l] = t.node_slot[l].p;
    t.d.node_verdict[l] = t.node_verdict[l].p;
    t.d.node_hist[l] = t.node_hist[l].p;
  }
  return LTL4C_OK;
}

// Online: make sure the carried tables can absorb `extra` more leaves/nodes at
// load <= 1/2, rehashing the carried entries into larger tables if needed.
ltl4c_status ensure_online_tables(ltl4c_state *st, uint64_t extra, cudaStream_t s, const Launcher &L) {
  Tables &t = st->tab;
  uint64_t want_leaf = 0, want_node = 0;
  bool fits = false;
  for (int pass = 0; pass < 2; ++pass) {
    // carried leaves / nodes: the last result read, plus (pipelined batches) every
    // event enqueued since -- an upper bound, each event adds at most one of each
    const uint64_t inflight = st->enq_events - st->known_cum;
    const uint64_t have = st->known_leaves + inflight;
    uint64_t need_nodes = 0;
    for (int l = 1; l < (int)st->prog->n_levels; ++l) need_nodes = std::max<uint64_t>(need_nodes, st->known_nodes[l] + inflight);
    // load <= 1/2 after this batch; grow 4x at a time (rehash = alloc + copy + sync)
    const uint64_t need_leaf = 2 * (have + extra) + 1, need_node = 2 * (need_nodes + extra) + 1;
    want_leaf = 1ull << std::max(20, ceil_log2(need_leaf));
    want_node = 1ull << std::max(16, ceil_log2(need_node));
    if (t.d.leaf_cap && t.d.leaf_cap < want_leaf) want_leaf = std::max<uint64_t>(want_leaf, 4 * t.d.leaf_cap);
    if (t.d.leaf_cap == 0) want_leaf = std::max<uint64_t>(want_leaf, 1ull << ceil_log2(8 * extra + 1));
    fits = t.d.leaf_cap && t.d.leaf_cap >= want_leaf;
    for (int l = 1; l < (int)st->prog->n_levels; ++l) fits &= t.d.node_cap[l] >= want_node;
    if (fits || inflight == 0 || t.d.leaf_cap == 0) break;
    // the bound says grow while batches are in flight: wait for them and use the
    // exact carried counts instead (growth is rare; the bound alone would over-allocate)
    CU(cudaStreamSynchronize(s));
    unsigned long long cnt[1 + kMaxLevels + 1];
    CU(cudaMemcpy(cnt, &st->d_acc.p->leaves, sizeof cnt, cudaMemcpyDeviceToHost));
    st->known_leaves = cnt[0];
    for (int l = 0; l < kMaxLevels; ++l) st->known_nodes[l] = cnt[1 + l];
    st->known_cum = st->enq_events;
  }
  if (fits) return LTL4C_OK;
  bool fresh = t.d.leaf_cap == 0;
  if (fresh) {
    ltl4c_status r = alloc_tables(st, t, want_leaf, want_node, s, false, true);
    if (r) return r;
    t.d.epoch = st->epoch;
    return LTL4C_OK;
  }
  Tables nt;
  ltl4c_status r = alloc_tables(st, nt, std::max<uint64_t>(want_leaf, t.d.leaf_cap), std::max<uint64_t>(want_node, t.d.node_cap[1]), s,
                                false, true);
  if (r) return r;
  nt.d.epoch = st->epoch;
  CU(launch_rehash(t.d, nt.d, (int)st->prog->n_levels, (int)st->prog->n_formulas,
                   &st->d_acc.p->table_overflow, L));
  CU(cudaStreamSynchronize(s));
  t.release();
  t = nt;
  nt = Tables{};  // ownership moved (DevBuf members copied; prevent double free)
  return LTL4C_OK;
}


// Heavy path for the oversize buckets of an offline verify (sizes known on the
// host from the first result copy).
ltl4c_status run_heavy(ltl4c_state *st, const BucketParams &bp, int K, cudaStream_t s, const Launcher &L) {
  const uint64_t ev = st->h_out->oversize_events;
  const uint64_t nb = st->h_out->oversize_buckets;
  const uint64_t cap = 1ull << std::max(12, ceil_log2(2 * ev + 1));
  if (st->tab.d.leaf_cap < cap || !st->tab.d.leaf_aux || (K > 1 && st->tab.d.node_cap[1] < cap)) {
    st->tab.release();
    ltl4c_status r = alloc_tables(st, st->tab, cap, cap, s, true);
    if (r) return r;
  }
  st->tab.d.epoch = ++st->epoch;
  const uint64_t nblk = (ev + 1023) / 1024 + 1;
  const size_t nseg = nb + 1;
  const size_t u32_need = nseg + 5 * ev + nblk + (size_t)(K - 1) * cap + 16;
  CU(st->h_part.ensure(ev + 1));
  CU(st->h_lists.ensure(ev + 1));
  CU(st->h_u32.ensure(u32_need));
  CU(st->h_cnt.ensure(16));
  HeavyParams h{};
  for (int k = 0; k < K; ++k) h.key[k] = bp.key[k];
  h.let = bp.let;
  h.bucket_off = bp.bucket_off;
  h.list = bp.oversize_list;
  h.list_len = &st->d_acc.p->oversize_buckets;
  h.prog = bp.prog;
  h.acc = bp.acc;
  h.tab = st->tab.d;
  uint32_t *u = st->h_u32.p;
  h.seg_base = u; u += nseg;
  h.leaf_slot_of = u; u += ev;
  h.leaf_npart = u; u += ev;
  h.leaf_off = u; u += ev;
  h.leaf_fill = u; u += ev;
  h.long_list = u; u += ev;
  h.scan_tmp = u; u += nblk;
  for (int l = 1; l < K; ++l) { h.node_list[l] = u; u += cap; }
  h.ctr = u; u += 8;
  h.part = st->h_part.p;
  h.lists = st->h_lists.p;
  unsigned long long *c = st->h_cnt.p;
  h.n_part = c;
  h.n_leaves = c + 1;
  h.n_nodes = c + 4;  // [kMaxLevels]
  h.cap_leaves = ev;
  CU(cudaMemsetAsync(h.leaf_npart, 0, sizeof(uint32_t) * 2 * ev, s));  // npart, off
  CU(cudaMemsetAsync(h.leaf_fill, 0, sizeof(uint32_t) * ev, s));
  CU(cudaMemsetAsync(h.ctr, 0, sizeof(uint32_t) * 8, s));
  CU(cudaMemsetAsync(c, 0, sizeof(unsigned long long) * 16, s));
  CU(launch_heavy(h, K, (int)st->prog->n_formulas, (int)st->prog->n_states, st->n_sms, L));
  return LTL4C_OK;
}

struct Plan {
  uint64_t N = 0;
  int B = 0, P = 0;
  uint32_t NB = 0, n_tiles = 0;
};

// K = 1 offline batches of >= kHotMinBatch events take the heavy-hitter path
// (hot.cu) for monitors of <= 8 states (below that the batch is launch-bound and
// the sampling kernels are pure overhead)
constexpr uint64_t kHotMinBatch = 1u << 17;  // (C1 sweep: 2^16 faster without, 2^17 with)
bool use_hot(const ltl4c_state *st, uint64_t N) {
  return st->hot && st->hot_mapk >= 0 && st->prog->n_levels == 1 && !(st->flags & LTL4C_STATE_ONLINE) &&
         N >= kHotMinBatch;
}
// hot_compose chunks: one per warp of the resident grid, multiples of 512 events
uint64_t hot_chunk_ev(const ltl4c_state *st, uint64_t N) {
  const uint64_t g = (uint64_t)st->hot_per_sm * st->n_sms * kHotCtaWarps;
  return std::max<uint64_t>(512, ((N + g - 1) / g + 511) / 512 * 512);
}

// Buffer sizes for a batch of N events (all allocation happens here, outside
// any stream capture).
ltl4c_status plan_batch(ltl4c_state *st, uint64_t N, Plan *pl) {
  const int K = (int)st->prog->n_levels;
  pl->N = N;
  if (N == 0) return LTL4C_OK;
  const uint64_t target = std::max<uint64_t>(2, (st->bucket_mul * N + kWarpCap - 1) / kWarpCap);
  pl->B = std::min(std::min(kMaxPasses * kMaxDigitBits, st->max_bits), std::max(1, ceil_log2(target)));
  // one level (leaves only, no node tables in the warp kernels): two partition
  // passes with larger buckets beat a third pass (C3: 5.17 -> 4.62 ms; with inner
  // levels the medium tiers fill up instead: C4 9.43 -> 10.0 ms)
  if (K == 1 && !(st->flags & LTL4C_STATE_ONLINE) && !st->max_bits_set)
    pl->B = std::min(pl->B, 2 * kMaxDigitBits);
  pl->P = (pl->B + kMaxDigitBits - 1) / kMaxDigitBits;
  pl->NB = 1u << pl->B;
  pl->n_tiles = (uint32_t)((N + kTileEv - 1) / kTileEv);
  for (int i = 0; i < 2; ++i) {
    for (int l = 0; l < K; ++l) CU(st->bufkey[i][l].ensure(N + 16));
    CU(st->buflet[i].ensure(N + 16));
  }
  CU(st->counts.ensure((size_t)kMaxDigits * pl->n_tiles));
  CU(st->totals.ensure(kMaxPasses * kMaxDigits + 16));
  CU(st->bucket_off.ensure((size_t)pl->NB + 1));
  CU(st->oversize_list.ensure(pl->NB));
  CU(st->medium_list.ensure(pl->NB));
  CU(st->large_list.ensure(pl->NB));
  CU(st->unit_start.ensure(N / kUnitTarget + 4));
  if (K == 1) CU(st->unit_start2.ensure(N / st->seg_unit + 4));
  if (K == 1) CU(st->coarse_off.ensure(2 * ((1u << kCoarseBits) + 1)));  // offsets | order
  if (use_hot(st, N)) {
    const uint64_t nch = (N + hot_chunk_ev(st, N) - 1) / hot_chunk_ev(st, N);
    CU(st->hot_cnt.ensure(2 * (size_t)kHotCountCap));
    CU(st->hot_tab.ensure(hot_slots(st->hot_mapk) + 72));  // slot keys, nhot + count bins
    CU(st->hot_partial.ensure((nch * hot_slots(st->hot_mapk) * hot_map_bytes(st->hot_mapk) + 3) / 4));
    CU(st->hot_chunk.ensure(2 * nch));
    CU(st->hot_n.ensure(1));
  }
  return LTL4C_OK;
}

// grid of a warp kernel: every resident CTA slot (LTL4C_WARP_GRID caps it: tests
// that push many units through one warp)
uint32_t warp_grid(const ltl4c_state *st, int ctas_per_sm) {
  const uint32_t g = (uint32_t)(st->n_sms * ctas_per_sm);
  return st->warp_grid ? std::min(g, st->warp_grid) : g;
}

BucketParams bucket_params(ltl4c_state *st, const Plan &pl) {
  const int K = (int)st->prog->n_levels;
  BucketParams bp{};
  const int fin = (pl.P - 1) & 1;
  for (int l = 0; l < K; ++l) bp.key[l] = st->bufkey[fin][l].p;
  bp.let = st->buflet[fin].p;
  bp.bucket_off = st->bucket_off.p;
  bp.n_buckets = pl.NB;
  bp.oversize_list = st->oversize_list.p;
  bp.medium_list = st->medium_list.p;
  bp.bucket_counter = st->totals.p + kMaxPasses * kMaxDigits + 8;
  bp.warps_per_cta = st->warp_cfg[0];
  bp.warp_hdr = bucket_warp_hdr((int)st->prog->n_states, (int)st->prog->letter_bits);
  bp.spill_list = st->medium_list.p;
  bp.spill_len = &st->d_acc.p->medium_buckets;
  bp.unit_start = st->unit_start.p;
  bp.n_units = (uint32_t)(pl.N / kUnitTarget + 2);
  bp.unit_target = kUnitTarget;
  bp.nvalid = st->d_nvalid.p;
  bp.prog = st->d_prog.p;
  bp.acc = st->d_acc.p;
  bp.tab = st->tab.d;
  return bp;
}

// the one-pass mode's coarse buckets: the first pass's output and its digit offsets
BucketParams coarse_params(ltl4c_state *st, const Plan &pl, const BucketParams &bp, int width) {
  BucketParams cp = bp;
  cp.key[0] = st->bufkey[0][0].p;
  cp.let = st->buflet[0].p;
  cp.bucket_off = st->coarse_off.p;
  cp.n_buckets = 1u << width;
  cp.bucket_counter = st->totals.p + kMaxPasses * kMaxDigits + 10;
  cp.list = st->coarse_off.p + (1u << kCoarseBits) + 1;  // the buckets, largest first (coarse_order)
  cp.coarse_hist = st->totals.p;                          // (pass 0's digit totals: coarse_order writes the offsets)
  return cp;
}

// the heavy path's buckets: coarse when the batch took the one-pass mode
BucketParams heavy_params(ltl4c_state *st, const Plan &pl) {
  BucketParams bp = bucket_params(st, pl);
  if (st->h_out->onepass) bp = coarse_params(st, pl, bp, kCoarseBits);
  return bp;
}

// Everything of one verify up to the first result copy, enqueued on s:
// memsets, SortTrace (count / scan / scatter per pass), mu, the bucket kernels,
// finalize and the D2H copy of the result record.
ltl4c_status enqueue_main(ltl4c_state *st, const Plan &plan, const uint32_t *const *keys, const uint8_t *letters,
                          cudaStream_t s, const Launcher &L, bool finalize_now = true, DevOut *dst = nullptr,
                          bool zero_acc = true) {
  const ltl4c_program *prog = st->prog;
  const int K = (int)prog->n_levels;
  const bool online = st->flags & LTL4C_STATE_ONLINE;
  CU(launch_reset(!online && zero_acc ? st->d_acc.p : nullptr, st->d_nvalid.p, plan.N > 0 ? st->totals.p : nullptr,
                  kMaxPasses * kMaxDigits + 16, L));
  if (plan.N > 0) {
    PartPlan pl{};
    for (int l = 0; l < K; ++l) {
      pl.in_key[l] = keys[l];
      pl.buf_key[0][l] = st->bufkey[0][l].p;
      pl.buf_key[1][l] = st->bufkey[1][l].p;
    }
    pl.in_let = letters;
    pl.buf_let[0] = st->buflet[0].p;
    pl.buf_let[1] = st->buflet[1].p;
    pl.n = plan.N;
    pl.n_tiles = plan.n_tiles;
    pl.n_sms = st->n_sms;
    pl.K = K;
    pl.bits = plan.B;
    pl.salt = kBucketSalt;
    pl.hk = online ? K - 1 : 0;  // online: buckets by the deepest key (balanced leaves)
    pl.hcol[0] = pl.buf_key[0][pl.hk];
    pl.hcol[1] = pl.buf_key[1][pl.hk];
    pl.rank_ballot = st->rank_ballot;
    pl.let_mask = (1u << prog->letter_bits) - 1u;
    pl.passes = plan.P;
    int lo = 0;
    for (int pass = 0; pass < plan.P; ++pass) {
      const int width = (plan.B - lo + (plan.P - pass) - 1) / (plan.P - pass);
      pl.lo[pass] = lo;
      pl.width[pass] = width;
      lo += width;
    }
    pl.digit_hist = st->totals.p;
    pl.counts = st->counts.p;
    pl.nvalid = st->d_nvalid.p;
    pl.acc = st->d_acc.p;
    HotParams hp{};
    const bool hot = use_hot(st, plan.N);
    if (hot) {
      // heavy hitters: sampled, composed where they lie; the rest, gathered into a
      // dense stream (bufkey[1] / buflet[1], free until pass 1), is partitioned
      const int S = hot_slots(st->hot_mapk);
      hp.k0 = keys[0];
      hp.let = letters;
      hp.n = plan.N;
      hp.n_samples = (uint32_t)std::min<uint64_t>(plan.N, kHotSamplesMax);
      hp.cnt_cap = 4096;
      while (hp.cnt_cap < 2 * hp.n_samples && hp.cnt_cap < (uint32_t)kHotCountCap) hp.cnt_cap <<= 1;
      hp.mapk = st->hot_mapk;
      hp.slots = S;
      hp.let_mask = pl.let_mask;
      hp.cnt_key = st->hot_cnt.p;
      hp.cnt_val = st->hot_cnt.p + kHotCountCap;
      hp.slot_key = st->hot_tab.p;
      hp.nhot = st->hot_tab.p + S;
      hp.partial = st->hot_partial.p;
      hp.cold_key = st->bufkey[0][0].p;
      hp.cold_let = st->buflet[0].p;
      hp.dense_key = st->bufkey[1][0].p;
      hp.dense_let = st->buflet[1].p;
      hp.chunk_cold = st->hot_chunk.p;
      hp.chunk_pre = st->hot_chunk.p + (st->hot_chunk.n / 2);
      hp.n_cold = st->hot_n.p;
      hp.chunk_ev = hot_chunk_ev(st, plan.N);
      hp.n_chunks = (int)((plan.N + hp.chunk_ev - 1) / hp.chunk_ev);
      hp.force_onepass = st->force_onepass;
      hp.prog = st->d_prog.p;
      hp.acc = st->d_acc.p;
      CU(cudaMemsetAsync(hp.cnt_key, 0xFF, sizeof(uint32_t) * hp.cnt_cap, s));
      CU(cudaMemsetAsync(hp.cnt_val, 0, sizeof(uint32_t) * hp.cnt_cap, s));
      CU(cudaMemsetAsync(hp.slot_key, 0xFF, sizeof(uint32_t) * S, s));
      CU(cudaMemsetAsync(hp.nhot, 0, sizeof(uint32_t) * 72, s));
      CU(cudaMemsetAsync(hp.n_cold, 0, sizeof(unsigned long long), s));
      CU(launch_hot_select(hp, L));
      CU(launch_hot_compose(hp, L));
      pl.dense_key = hp.dense_key;
      pl.dense_let = hp.dense_let;
      pl.dense_n = hp.n_cold;
      pl.dense_flag = hp.nhot + 2;
    }
    // one-pass mode (decided on the device: some key is hot): the cold stream is
    // partitioned once into coarse buckets, each taken by a CTA (bucket_coarse);
    // otherwise the second pass and the warp kernels run
    const bool onepass = hot && st->hot_mapk == 0 && st->coarse && plan.P == 2;
    const uint32_t *one = onepass ? hp.nhot + 3 : nullptr;  // the one-pass flag (device)
    if (onepass) pl.skip_flag = one;
    if (!hot && plan.N <= (uint64_t)kTinyBatch) {
      // a tiny batch (a verdict stream of single events): one bucket, staged by one CTA
      CU(launch_tiny_stage(pl, st->bucket_off.p, plan.NB, L));
    } else {
      for (int pass = 0; pass < plan.P; ++pass) {
        CU(launch_part_count(pl, pass, L));
        CU(launch_part_scan(pl, pass, L));
        CU(launch_part_scatter(pl, pass, L));
      }
      if (hot) CU(launch_hot_finish(hp, L));
      CU(launch_bucket_bounds(pl, st->bucket_off.p, plan.NB, L, one, 0));
    }
    BucketParams bp = bucket_params(st, plan);
    if (!online) {
      // a warp per unit (<= kWarpCap events); buckets above that go to the same
      // kernel with kWarpCapBig, above that to the CTA kernel, and above kCap to
      // the heavy path (after the first result copy)
      if (K == 1 && st->seg) {
        // one level: units of ~seg_unit events streamed through warp tables by
        // segmented map scans (seg.cu); units with too many distinct keys go to the CTA kernel
        const uint32_t nu = (uint32_t)(plan.N / st->seg_unit + 2);
        CU(launch_unit_start(st->bucket_off.p, plan.NB, st->unit_start2.p, nu, L, st->seg_unit,
                             one, 0));
        if (onepass) {
          BucketParams cp = coarse_params(st, plan, bp, pl.width[0]);
          cp.gate = one;
          cp.gate_want = 1;
          CU(launch_bucket_coarse(cp, (int)prog->n_formulas, warp_grid(st, st->coarse_per_sm), L));
        }
        BucketParams sp = bp;
        sp.gate = one;
        sp.unit_start = st->unit_start2.p;
        sp.n_units = nu;
        sp.unit_target = st->seg_unit;
        sp.spill_list = st->large_list.p;
        sp.spill_len = &st->d_acc.p->large_buckets;
        CU(launch_bucket_seg(sp, (int)prog->n_states, (int)prog->n_formulas, warp_grid(st, st->seg_per_sm), L));
        BucketParams fp = bp;
        fp.list = st->large_list.p;
        fp.list_len = &st->d_acc.p->large_buckets;
        CU(launch_bucket_fast(fp, K, (int)prog->n_formulas, st->n_sms, L));
      } else {
        CU(launch_unit_start(st->bucket_off.p, plan.NB, st->unit_start.p, bp.n_units, L));
        CU(launch_bucket_warp(bp, K, (int)prog->n_formulas, warp_grid(st, st->warp_cfg[1]), L));
        BucketParams mp = bp;
        mp.list = st->medium_list.p;
        mp.list_len = &st->d_acc.p->medium_buckets;
        mp.spill_list = st->large_list.p;
        mp.spill_len = &st->d_acc.p->large_buckets;
        mp.bucket_counter = bp.bucket_counter + 1;
        mp.warps_per_cta = st->warp_cfg[2];
        CU(launch_bucket_warp(mp, K, (int)prog->n_formulas, warp_grid(st, st->warp_cfg[3]), L));
        BucketParams fp = bp;
        fp.list = st->large_list.p;
        fp.list_len = &st->d_acc.p->large_buckets;
        CU(launch_bucket_fast(fp, K, (int)prog->n_formulas, st->n_sms, L));
      }
    } else {
      // carried state: leaves (warp per unit), then touched nodes depth K-1 .. 1
      OnlineParams op{};
      op.b = bp;
      op.b.warps_per_cta = st->online_cfg[0];
      op.bid = st->batch_id;
      op.bid_dev = st->d_bid.p;  // (set by the caller before this sequence runs)
      for (int l = 1; l < K; ++l) op.tlist[l] = st->tlist[l].p;
      op.tcnt = st->tcnt.p;
      CU(cudaMemsetAsync(st->tcnt.p, 0, sizeof(uint32_t) * kMaxLevels, s));
      CU(launch_unit_start(st->bucket_off.p, plan.NB, st->unit_start.p, bp.n_units, L));
      CU(launch_online_leaf(op, K, (int)prog->n_formulas, (uint32_t)(st->n_sms * st->online_cfg[1]), L));
      for (int l = K - 1; l >= 1; --l)
        CU(launch_online_nodes(op, (int)prog->n_formulas, l, (uint32_t)(st->n_sms * 8), L));
    }
  }
  if (finalize_now) {
    CU(launch_finalize(st->d_prog.p, st->d_acc.p, st->d_out.p, L));
    CU(cudaMemcpyAsync(dst ? dst : st->h_out, st->d_out.p, sizeof(DevOut), cudaMemcpyDeviceToHost, s));
  }
  return LTL4C_OK;
}

// Multi-GPU step 1a: one stable partition pass of the bound events
// by owner = top `bits` bits of an (independent) hash of k0 -- every tree node
// below the root lives on one owner -- into (okey, olet); the per-owner counts
// are left in totals[0 .. 2^bits) (u32, device).
ltl4c_status owner_partition(ltl4c_state *st, const uint32_t *const *keys, const uint8_t *letters, uint64_t N,
                             int bits, uint32_t *const *okey, uint8_t *olet, cudaStream_t s, const Launcher &L) {
  const int K = (int)st->prog->n_levels;
  const uint32_t n_tiles = (uint32_t)std::max<uint64_t>(1, (N + kTileEv - 1) / kTileEv);
  CU(st->counts.ensure((size_t)kMaxDigits * n_tiles));
  CU(st->totals.ensure(kMaxPasses * kMaxDigits + 16));
  CU(st->d_sacc.ensure(1));  // (virtual shards run without a communicator)
  CU(cudaMemsetAsync(st->totals.p, 0, sizeof(uint32_t) * (kMaxPasses * kMaxDigits + 16), s));
  CU(cudaMemsetAsync(st->d_nvalid.p, 0, sizeof(unsigned long long), s));
  CU(cudaMemsetAsync(st->d_sacc.p, 0, sizeof(DevAcc), s));
  if (N == 0) return LTL4C_OK;
  PartPlan pl{};
  for (int l = 0; l < K; ++l) {
    pl.in_key[l] = keys[l];
    pl.buf_key[0][l] = okey[l];
    pl.buf_key[1][l] = okey[l];
  }
  pl.in_let = letters;
  pl.buf_let[0] = olet;
  pl.buf_let[1] = olet;
  pl.n = N;
  pl.n_tiles = n_tiles;
  pl.n_sms = st->n_sms;
  pl.K = K;
  pl.bits = bits;
  pl.passes = 1;
  pl.salt = kOwnerSalt;
  pl.hk = 0;  // owner by level-0 key: whole subtrees per owner
  pl.hcol[0] = okey[0];
  pl.hcol[1] = okey[0];
  pl.rank_ballot = st->rank_ballot;
  pl.let_mask = (1u << st->prog->letter_bits) - 1u;
  pl.lo[0] = 0;
  pl.width[0] = bits;
  pl.digit_hist = st->totals.p;
  pl.counts = st->counts.p;
  pl.nvalid = st->d_nvalid.p;
  pl.acc = st->d_sacc.p;
  CU(launch_part_count(pl, 0, L));
  CU(launch_part_scan(pl, 0, L));
  CU(launch_part_scatter(pl, 0, L));
  return LTL4C_OK;
}

// Multi-GPU step 1b: route this rank's bound events to their owner rank and
// exchange them with grouped NCCL send/recv.  The per-owner counts are
// all-gathered from device memory (one host synchronisation to size the
// transfers).  Receive buffers are concatenated in source-rank order; rank r holds
// the trace range preceding rank r+1's, so every slice keeps its trace order.
ltl4c_status exchange(ltl4c_state *st, const uint32_t *const *keys, const uint8_t *letters, uint64_t N,
                      cudaStream_t s, const Launcher &L, uint64_t *M) {
  const int K = (int)st->prog->n_levels, G = st->n_ranks;
  Nccl *nc = nccl();
  if (!nc) return fail(LTL4C_E_NCCL, "NCCL library not found");
  for (int l = 0; l < K; ++l) CU(st->bufkey[0][l].ensure(N + 16));
  CU(st->buflet[0].ensure(N + 16));
  CU(st->dc_cnt.ensure((size_t)G * G));
  uint32_t *ok[kMaxLevels] = {st->bufkey[0][0].p, K > 1 ? st->bufkey[0][1].p : nullptr,
                              K > 2 ? st->bufkey[0][2].p : nullptr};
  {
    ltl4c_status r = owner_partition(st, keys, letters, N, st->owner_bits, ok, st->buflet[0].p, s, L);
    if (r) return r;
  }
  // per-owner counts (u32, device) -> all-gathered G x G matrix (row = source rank)
  uint32_t *mat_d = reinterpret_cast<uint32_t *>(st->dc_cnt.p);
  NC(nc->AllGather(st->totals.p, mat_d, (size_t)G, kNcclUint32, st->comm, s));
  uint32_t *mat = reinterpret_cast<uint32_t *>(st->hc_cnt);
  CU(cudaMemcpyAsync(mat, mat_d, sizeof(uint32_t) * G * G, cudaMemcpyDeviceToHost, s));
  CU(cudaStreamSynchronize(s));
  std::vector<uint64_t> soff(G), scnt(G), roff(G), rcnt(G);
  uint64_t so = 0, ro = 0;
  for (int r = 0; r < G; ++r) {
    scnt[r] = mat[(size_t)st->rank * G + r];
    soff[r] = so;
    so += scnt[r];
    rcnt[r] = mat[(size_t)r * G + st->rank];
    roff[r] = ro;
    ro += rcnt[r];
  }
  *M = ro;
  for (int l = 0; l < K; ++l) CU(st->exkey[l].ensure(ro));
  CU(st->exlet.ensure(ro));
  NC(nc->GroupStart());
  for (int r = 0; r < G; ++r) {
    for (int l = 0; l < K; ++l) {
      if (scnt[r]) NC(nc->Send(st->bufkey[0][l].p + soff[r], scnt[r], kNcclUint32, r, st->comm, s));
      if (rcnt[r]) NC(nc->Recv(st->exkey[l].p + roff[r], rcnt[r], kNcclUint32, r, st->comm, s));
    }
    if (scnt[r]) NC(nc->Send(st->buflet[0].p + soff[r], scnt[r], kNcclUint8, r, st->comm, s));
    if (rcnt[r]) NC(nc->Recv(st->exlet.p + roff[r], rcnt[r], kNcclUint8, r, st->comm, s));
  }
  NC(nc->GroupEnd());
  return LTL4C_OK;
}

// Multi-GPU step 2: every node below the root lives on exactly one rank, so the
// per-level histograms (and the root's child histogram hist[1]) are sums over
// ranks: one all-reduce, then every rank applies the root rule.
ltl4c_status reduce_and_finalize(ltl4c_state *st, cudaStream_t s, const Launcher &L) {
  Nccl *nc = nccl();
  const size_t nsum = (sizeof(((DevAcc *)0)->hist) / sizeof(unsigned long long)) + 2;  // + events_seen, bound
  unsigned long long seen = st->events_seen;
  CU(cudaMemcpyAsync(&st->d_acc.p->events_seen, &seen, sizeof seen, cudaMemcpyHostToDevice, s));
  NC(nc->AllReduce(st->d_acc.p, st->d_gacc.p, nsum, kNcclUint64, kNcclSum, st->comm, s));
  CU(cudaMemcpyAsync(&st->d_gacc.p->medium_buckets, &st->d_acc.p->medium_buckets,
                     sizeof(DevAcc) - offsetof(DevAcc, medium_buckets), cudaMemcpyDeviceToDevice, s));
  CU(launch_finalize(st->d_prog.p, st->d_gacc.p, st->d_out.p, L));
  CU(cudaMemcpyAsync(st->h_out, st->d_out.p, sizeof(DevOut), cudaMemcpyDeviceToHost, s));
  CU(cudaStreamSynchronize(s));
  return LTL4C_OK;
}

void drop_graph(ltl4c_state *st) {
  if (st->graph_exec) cudaGraphExecDestroy(st->graph_exec);
  st->graph_exec = nullptr;
  st->graph_key.clear();
}

void fill_results(const ltl4c_state *st, const DevOut &o, uint64_t events_seen, bool comm, ltl4c_result *out) {
  for (uint32_t f = 0; f < st->prog->n_formulas; ++f) {
    const DevResult &r = o.res[f];
    ltl4c_result &x = out[f];
    std::memset(&x, 0, sizeof x);
    x.verdict = r.verdict;
    x.n_levels = r.n_levels;
    for (int l = 0; l <= kMaxLevels; ++l)
      for (int v = 0; v < 6; ++v) x.hist[l][v] = r.hist[l][v];
    x.events_seen = comm ? r.events_seen : events_seen;
    x.events_bound = r.events_bound;
  }
}

// Test-only virtual shards (LTL4C_VIRTUAL_SHARDS = G, a power of two <= 256): the
// multi-GPU owner partition with G owners on this GPU, then each owner's events
// through the local pipeline in turn with the per-level histograms summed in the
// accumulators, and the root rule once on the summed depth-1 histogram -- the
// sharded path of SURVEY §8(e) without the NCCL transport.
ltl4c_status run_virtual(ltl4c_state *st, const uint32_t *const *keys, const uint8_t *letters, uint64_t N,
                         cudaStream_t s, const Launcher &L) {
  const int K = (int)st->prog->n_levels, G = st->vshards;
  const bool online = st->flags & LTL4C_STATE_ONLINE;
  int bits = 0;
  while ((1 << bits) < G) ++bits;
  for (int l = 0; l < K; ++l) CU(st->exkey[l].ensure(N + 16));
  CU(st->exlet.ensure(N + 16));
  uint32_t *ok[kMaxLevels] = {st->exkey[0].p, K > 1 ? st->exkey[1].p : nullptr, K > 2 ? st->exkey[2].p : nullptr};
  {
    ltl4c_status r = owner_partition(st, keys, letters, N, bits, ok, st->exlet.p, s, L);
    if (r) return r;
  }
  if (!st->hc_cnt && cudaMallocHost((void **)&st->hc_cnt, sizeof(unsigned long long) * (256 + 256 * 256)) != cudaSuccess)
    return fail(LTL4C_E_OOM, "pinned allocation failed");
  uint32_t *cnt = reinterpret_cast<uint32_t *>(st->hc_cnt);
  if (N > 0) CU(cudaMemcpyAsync(cnt, st->totals.p, sizeof(uint32_t) * G, cudaMemcpyDeviceToHost, s));
  else std::memset(cnt, 0, sizeof(uint32_t) * G);
  CU(cudaStreamSynchronize(s));
  if (!online) CU(cudaMemsetAsync(st->d_acc.p, 0, sizeof(DevAcc), s));
  uint64_t off = 0;
  for (int g = 0; g < G; ++g) {
    const uint64_t ng = cnt[g];
    const uint32_t *gk[kMaxLevels] = {nullptr, nullptr, nullptr};
    for (int l = 0; l < K; ++l) gk[l] = st->exkey[l].p + off;
    const uint8_t *gl = st->exlet.p + off;
    off += ng;
    if (online) {
      ltl4c_status r = ensure_online_tables(st, ng, s, L);
      if (r) return r;
      for (int l = 1; l < K; ++l) CU(st->tlist[l].ensure(st->tab.d.node_cap[l]));
      CU(st->tcnt.ensure(kMaxLevels));
      if (++st->batch_id == 0) st->batch_id = 1;
      st->enq_events += ng;
      CU(st->d_bid.ensure(1));
      CU(launch_set_u32(st->d_bid.p, st->batch_id, L));
    }
    Plan plan;
    {
      ltl4c_status r = plan_batch(st, ng, &plan);
      if (r) return r;
    }
    // the spill-list lengths of this owner's pass start at zero
    CU(cudaMemsetAsync(&st->d_acc.p->medium_buckets, 0, 4 * sizeof(unsigned long long), s));
    ltl4c_status r = enqueue_main(st, plan, gk, gl, s, L, false, nullptr, false);
    if (r) return r;
    if (!online && ng > 0) {
      CU(cudaMemcpyAsync(&st->h_out->oversize_buckets, &st->d_acc.p->oversize_buckets, 2 * sizeof(unsigned long long),
                         cudaMemcpyDeviceToHost, s));
      CU(cudaStreamSynchronize(s));
      if (st->h_out->oversize_buckets) {
        ltl4c_status r2 = run_heavy(st, heavy_params(st, plan), K, s, L);
        if (r2) return r2;
      }
    }
  }
  CU(launch_finalize(st->d_prog.p, st->d_acc.p, st->d_out.p, L));
  CU(cudaMemcpyAsync(st->h_out, st->d_out.p, sizeof(DevOut), cudaMemcpyDeviceToHost, s));
  CU(cudaStreamSynchronize(s));
  return LTL4C_OK;
}

// async_dst: pipelined online batch -- the result is copied to this pinned slot
// and the call returns without waiting (ltl4c_result_get reads it)
ltl4c_status run_verify(ltl4c_state *st, const ltl4c_batch *b, cudaStream_t s, ltl4c_result *out,
                        const uint32_t *const *keys, const uint8_t *letters, DevOut *async_dst = nullptr) {
  const ltl4c_program *prog = st->prog;
  const int K = (int)prog->n_levels;
  const bool online = st->flags & LTL4C_STATE_ONLINE;
  const uint64_t N = b->n_events;
  st->cur_stream = s;
  Launcher L{s, before_launch, after_launch, st};
  if (!online) st->events_seen = 0;
  st->events_seen += N;
  const bool comm = st->comm && (st->n_ranks > 1 || st->force_exchange);
  if (st->vshards > 1 && !comm && !async_dst) {
    ltl4c_status r = run_virtual(st, keys, letters, N, s, L);
    if (r) return r;
    if (st->h_out->table_overflow) return fail(LTL4C_E_OOM, "carried table overflow");
    if (online) {
      st->known_leaves = st->h_out->leaves;
      for (int l = 0; l < kMaxLevels; ++l) st->known_nodes[l] = st->h_out->nodes[l];
      st->known_cum = st->enq_events;
    }
    fill_results(st, *st->h_out, st->events_seen, false, out);
    st->verifies++;
    return LTL4C_OK;
  }
  uint64_t Nloc = N;
  const uint32_t *lkeys[kMaxLevels] = {keys[0], K > 1 ? keys[1] : nullptr, K > 2 ? keys[2] : nullptr};
  const uint8_t *llet = letters;
  if (comm) {
    // route first: this rank then verifies the Nloc events it owns (up to G x N
    // when level-0 keys are skewed), and the carried tables are sized for those
    ltl4c_status r = exchange(st, keys, letters, N, s, L, &Nloc);
    if (r) return r;
    for (int l = 0; l < K; ++l) lkeys[l] = st->exkey[l].p;
    llet = st->exlet.p;
  }
  if (online) {
    ltl4c_status r = ensure_online_tables(st, Nloc, s, L);
    if (r) return r;
    for (int l = 1; l < K; ++l) CU(st->tlist[l].ensure(st->tab.d.node_cap[l]));
    CU(st->tcnt.ensure(kMaxLevels));
    if (++st->batch_id == 0) st->batch_id = 1;  // wrap: marks of batch 0 never exist
    CU(st->d_bid.ensure(1));
    st->enq_events += Nloc;
  }
  Plan plan;
  {
    ltl4c_status r = plan_batch(st, Nloc, &plan);
    if (r) return r;
  }
  if (comm) {
    if (online) CU(launch_set_u32(st->d_bid.p, st->batch_id, L));
    ltl4c_status r = enqueue_main(st, plan, lkeys, llet, s, L, false);
    if (r) return r;
    if (!online && Nloc > 0) {
      unsigned long long ov = 0;
      CU(cudaMemcpyAsync(&ov, &st->d_acc.p->oversize_buckets, sizeof ov, cudaMemcpyDeviceToHost, s));
      CU(cudaStreamSynchronize(s));
      if (ov) {
        st->h_out->oversize_buckets = ov;
        CU(cudaMemcpyAsync(&st->h_out->oversize_events, &st->d_acc.p->oversize_events, sizeof(unsigned long long),
                           cudaMemcpyDeviceToHost, s));
        CU(cudaStreamSynchronize(s));
        ltl4c_status r2 = run_heavy(st, heavy_params(st, plan), K, s, L);
        if (r2) return r2;
      }
    }
    ltl4c_status r3 = reduce_and_finalize(st, s, L);
    if (r3) return r3;
  } else {
  // Batches replay a captured CUDA graph of the launch sequence (one graph per
  // input pointers / size; online: per carried-table layout too, the batch id is
  // read from device memory); profiling runs the sequence directly so every kernel
  // can be bracketed by events; pipelined online batches copy their result to a
  // per-ticket slot and run the sequence directly.
  const bool use_graph = (!online || !async_dst) && !st->profiling && st->graphs && N > 0;  // (online: see below)
  if (online) CU(launch_set_u32(st->d_bid.p, st->batch_id, L));
  if (use_graph) {
    std::vector<uintptr_t> key = {(uintptr_t)N, (uintptr_t)letters, (uintptr_t)online};
    if (online) {
      const DevTables &T = st->tab.d;
      for (uintptr_t v : {(uintptr_t)T.epoch, (uintptr_t)T.leaf_cap, (uintptr_t)T.leaf_slot, (uintptr_t)T.leaf_state,
                          (uintptr_t)T.leaf_aux, (uintptr_t)st->tcnt.p, (uintptr_t)st->d_bid.p})
        key.push_back(v);
      for (int l = 0; l < kMaxLevels; ++l)
        for (uintptr_t v : {(uintptr_t)T.node_cap[l], (uintptr_t)T.node_slot[l], (uintptr_t)T.node_hist[l],
                            (uintptr_t)T.node_verdict[l], (uintptr_t)T.node_aux[l], (uintptr_t)st->tlist[l].p})
          key.push_back(v);
    }
    for (int l = 0; l < K; ++l) key.push_back((uintptr_t)keys[l]);
    // the captured launches bake in every buffer pointer: a buffer reallocated by an
    // ungraphed verify in between (profiling, another size) must not be replayed
    for (int i = 0; i < 2; ++i) {
      for (int l = 0; l < K; ++l) key.push_back((uintptr_t)st->bufkey[i][l].p);
      key.push_back((uintptr_t)st->buflet[i].p);
    }
    for (const void *b : {(const void *)st->counts.p, (const void *)st->totals.p, (const void *)st->bucket_off.p,
                          (const void *)st->oversize_list.p, (const void *)st->medium_list.p,
                          (const void *)st->large_list.p, (const void *)st->unit_start.p,
                          (const void *)st->d_acc.p, (const void *)st->d_out.p, (const void *)st->d_nvalid.p,
                          (const void *)st->d_prog.p, (const void *)st->h_out, (const void *)st->hot_cnt.p,
                          (const void *)st->hot_tab.p, (const void *)st->hot_partial.p,
                          (const void *)st->hot_chunk.p, (const void *)st->hot_n.p, (const void *)st->unit_start2.p,
                          (const void *)st->coarse_off.p})
      key.push_back((uintptr_t)b);
    // online: a stream of batches at new device addresses every call (slices) would be
    // captured every time; a layout is captured the second time in a row it is seen
    const bool known = !online || (st->graph_key == key && st->graph_exec) || st->graph_pending == key;
    if (!known) {
      st->graph_pending = key;
      ltl4c_status r = enqueue_main(st, plan, keys, letters, s, L, true, async_dst);
      if (r) return r;
    } else {
    if (st->graph_key != key || !st->graph_exec) {
      drop_graph(st);
      if (!st->cap_stream) CU(cudaStreamCreateWithFlags(&st->cap_stream, cudaStreamNonBlocking));
      const uint64_t before = st->launches;
      Launcher LC{st->cap_stream, nullptr, after_launch, st};
      st->cur_stream = st->cap_stream;
      CU(cudaStreamBeginCapture(st->cap_stream, cudaStreamCaptureModeThreadLocal));
      ltl4c_status r = enqueue_main(st, plan, keys, letters, st->cap_stream, LC);
      cudaGraph_t g = nullptr;
      cudaError_t ec = cudaStreamEndCapture(st->cap_stream, &g);
      st->cur_stream = s;
      if (r) { if (g) cudaGraphDestroy(g); return r; }
      CU(ec);
      cudaError_t ei = cudaGraphInstantiate(&st->graph_exec, g, 0);
      cudaGraphDestroy(g);
      CU(ei);
      st->graph_kernels = st->launches - before;
      st->launches = before;  // counted per replay below
      for (int k = 0; k < kKNumKernels; ++k) st->k_launches[k] = st->k_launches_saved[k];
      st->graph_key = key;
    }
    CU(cudaGraphLaunch(st->graph_exec, s));
    st->launches += st->graph_kernels;
    }
  } else {
    ltl4c_status r = enqueue_main(st, plan, keys, letters, s, L, true, async_dst);
    if (r) return r;
  }
  if (async_dst) {
    for (int k = 0; k < kKNumKernels; ++k) st->k_launches_saved[k] = st->k_launches[k];
    st->verifies++;
    return LTL4C_OK;
  }
  CU(cudaStreamSynchronize(s));
  if (!online && N > 0 && st->h_out->oversize_buckets > 0) {
    // buckets larger than one shared-memory chunk: segmented heavy path
    ltl4c_status r = run_heavy(st, heavy_params(st, plan), K, s, L);
    if (r) return r;
    CU(launch_finalize(st->d_prog.p, st->d_acc.p, st->d_out.p, L));
    CU(cudaMemcpyAsync(st->h_out, st->d_out.p, sizeof(DevOut), cudaMemcpyDeviceToHost, s));
    CU(cudaStreamSynchronize(s));
  }
  }
  for (int k = 0; k < kKNumKernels; ++k) st->k_launches_saved[k] = st->k_launches[k];
  if (st->h_out->table_overflow)
    return fail(LTL4C_E_OOM, "carried table overflow");
  if (online) {
    st->known_leaves = st->h_out->leaves;
    for (int l = 0; l < kMaxLevels; ++l) st->known_nodes[l] = st->h_out->nodes[l];
    st->known_cum = st->enq_events;
  }
  fill_results(st, *st->h_out, st->events_seen, comm, out);
  st->verifies++;
  return LTL4C_OK;
}

constexpr uint64_t kPackEvents = 1u << 16;  // host batches up to this size take the packed copy
constexpr size_t kPackBytes = kMaxLevels * 4 * kPackEvents + kPackEvents + 64;
ltl4c_status verify_common(ltl4c_state *st, const ltl4c_batch *b, void *stream, ltl4c_result *out,
                           bool host, DevOut *async_dst = nullptr) {
  if (!st || !b || (!out && !async_dst)) return fail(LTL4C_E_INVALID, "null argument");
  if (st->poisoned) return fail(LTL4C_E_POISONED, "state poisoned by an earlier failure; reset it");
  const int K = (int)st->prog->n_levels;
  if (b->n_events > (1ull << 32) - (1ull << 20))
    return fail(LTL4C_E_INVALID, "batch too large (max ~4.29e9 events)");
  if (b->n_events > 0) {
    for (int l = 0; l < K; ++l)
      if (!b->keys[l]) return fail(LTL4C_E_INVALID, "null key pointer");
    if (!b->letters) return fail(LTL4C_E_INVALID, "null letters pointer");
  }
  const bool online = st->flags & LTL4C_STATE_ONLINE;
  if (online && st->have_index && b->first_index != st->next_index)
    return fail(LTL4C_E_INVALID, "online batch is not contiguous with the previous batch");
  cudaStream_t s = (cudaStream_t)stream;
  int prev = 0;
  cudaGetDevice(&prev);
  if (prev != st->device) CU(cudaSetDevice(st->device));
  const uint32_t *keys[kMaxLevels] = {nullptr, nullptr, nullptr};
  const uint8_t *letters = b->letters;
  for (int l = 0; l < K; ++l) keys[l] = b->keys[l];
  ltl4c_status r = LTL4C_OK;
  const uint64_t n = b->n_events;
  if (host && n > 0 && n <= kPackEvents) {
    // a small batch from host memory (e.g. one event of a verdict stream): packed into
    // one pinned block and copied with one H2D copy into a buffer of fixed address, so
    // successive calls have the same layout (online: the sequence replays as a graph).
    const size_t kb = (4 * n + 15) & ~size_t(15), total = K * kb + n;
    if (!st->h_pack && cudaMallocHost((void **)&st->h_pack, kPackBytes) != cudaSuccess) r = fail(LTL4C_E_OOM, "pinned alloc");
    else if (st->d_pack.ensure(kPackBytes) != cudaSuccess) r = fail(LTL4C_E_OOM, "staging alloc");
    else if (!st->pack_done && cudaEventCreateWithFlags(&st->pack_done, cudaEventDisableTiming) != cudaSuccess)
      r = fail(LTL4C_E_CUDA, "event create failed");
    else {
      cudaEventSynchronize(st->pack_done);  // (the previous copy out of the block has completed)
      for (int l = 0; l < K; ++l) std::memcpy(st->h_pack + l * kb, b->keys[l], 4 * n);
      std::memcpy(st->h_pack + K * kb, b->letters, n);
      if (cudaMemcpyAsync(st->d_pack.p, st->h_pack, total, cudaMemcpyHostToDevice, s) != cudaSuccess ||
          cudaEventRecord(st->pack_done, s) != cudaSuccess)
        r = fail(LTL4C_E_CUDA, "H2D copy of the batch failed");
      for (int l = 0; l < K; ++l) keys[l] = reinterpret_cast<const uint32_t *>(st->d_pack.p + l * kb);
      letters = st->d_pack.p + K * kb;
    }
  } else if (host && n > 0) {
    for (int l = 0; l < K && !r; ++l) {
      if (st->hkeys[l].ensure(b->n_events) != cudaSuccess) r = fail(LTL4C_E_OOM, "staging alloc");
      else if (cudaMemcpyAsync(st->hkeys[l].p, b->keys[l], 4 * b->n_events, cudaMemcpyHostToDevice, s) != cudaSuccess)
        r = fail(LTL4C_E_CUDA, "H2D copy of keys failed");
      keys[l] = st->hkeys[l].p;
    }
    if (!r) {
      if (st->hlet.ensure(b->n_events) != cudaSuccess) r = fail(LTL4C_E_OOM, "staging alloc");
      else if (cudaMemcpyAsync(st->hlet.p, b->letters, b->n_events, cudaMemcpyHostToDevice, s) != cudaSuccess)
        r = fail(LTL4C_E_CUDA, "H2D copy of letters failed");
      letters = st->hlet.p;
    }
  }
  if (!r) r = run_verify(st, b, s, out, keys, letters, async_dst);
  if (prev != st->device) cudaSetDevice(prev);
  if (r) {
    if (online) st->poisoned = true;
    return r;
  }
  if (online) {
    st->next_index = b->first_index + b->n_events;
    st->have_index = true;
  }
  return LTL4C_OK;
}

}  // namespace

extern "C" {

const char *ltl4c_last_error(void) { return g_err.c_str(); }

const char *ltl4c_version(void) { return "ltl4c 0.1 sm_100a"; }

ltl4c_status ltl4c_state_create(const ltl4c_program *prog, int device, uint64_t capacity_hint,
                                uint32_t flags, ltl4c_state **out) {
  if (!prog || !out) return fail(LTL4C_E_INVALID, "null argument");
  *out = nullptr;
  if (flags & ~LTL4C_STATE_ONLINE) return fail(LTL4C_E_INVALID, "unknown flags");
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
    return fail(LTL4C_E_CUDA, "no CUDA device visible (this library has no CPU fallback)");
  if (device < 0 || device >= ndev) return fail(LTL4C_E_INVALID, "bad device ordinal");
  int prev = 0;
  cudaGetDevice(&prev);
  CU(cudaSetDevice(device));
  cudaDeviceProp dp{};
  CU(cudaGetDeviceProperties(&dp, device));
  if (dp.major != 10) {
    cudaSetDevice(prev);
    return fail(LTL4C_E_CUDA, "library is built for sm_100a (B200); device is sm_" +
                                  std::to_string(dp.major) + std::to_string(dp.minor));
  }
  auto st = new ltl4c_state();
  st->prog = prog;
  st->device = device;
  st->flags = flags;
  st->graphs = std::getenv("LTL4C_NO_GRAPH") == nullptr;
  st->force_exchange = std::getenv("LTL4C_FORCE_EXCHANGE") != nullptr;
  if (const char *e = std::getenv("LTL4C_BUCKET_MUL")) st->bucket_mul = std::max(1, std::atoi(e));
  if (const char *e = std::getenv("LTL4C_MAX_BITS")) {
    st->max_bits = std::max(1, std::min(kMaxPasses * kMaxDigitBits, std::atoi(e)));
    st->max_bits_set = true;
  }
  if (const char *e = std::getenv("LTL4C_WARP_GRID")) st->warp_grid = (uint32_t)std::max(0, std::atoi(e));
  if (const char *e = std::getenv("LTL4C_RANK_BALLOT")) st->rank_ballot = std::atoi(e);
  st->hot = std::getenv("LTL4C_NO_HOT") == nullptr;
  st->seg = std::getenv("LTL4C_NO_SEG") == nullptr;
  if (const char *e = std::getenv("LTL4C_SEG_UNIT")) st->seg_unit = std::max(32, std::atoi(e));
  st->coarse = std::getenv("LTL4C_NO_COARSE") == nullptr;
  st->force_onepass = std::getenv("LTL4C_FORCE_ONEPASS") != nullptr;
  if (const char *e = std::getenv("LTL4C_VIRTUAL_SHARDS")) {
    const int g = std::atoi(e);
    if (g > 1 && g <= 256 && !(g & (g - 1))) st->vshards = g;
  }
  DevProg &h = st->hprog;
  h.nf = prog->n_formulas;
  h.nl = prog->n_levels;
  h.na = prog->letter_bits;
  h.nq = prog->n_states;
  h.q0 = prog->initial;
  const int A = 1 << prog->letter_bits;
  for (uint32_t q = 0; q < prog->n_states; ++q)
    for (int a = 0; a < A; ++a) h.delta[q][a] = prog->delta[q * A + a];
  for (int a = 0; a < A; ++a) {
    unsigned long long m = 0;
    for (uint32_t q = 0; q < prog->n_states; ++q) m |= (unsigned long long)h.delta[q][a] << (4 * q);
    h.map[a] = m;
  }
  for (uint32_t f = 0; f < prog->n_formulas; ++f) {
    for (uint32_t q = 0; q < prog->n_states; ++q) h.lab[f][q] = prog->label[f * prog->n_states + q];
    for (uint32_t l = 0; l < prog->n_levels; ++l) {
      const ltl4c_quantifier &qq = prog->quant[f * prog->n_levels + l];
      h.qkind[f][l] = qq.kind;
      h.qcmp[f][l] = qq.cmp;
      h.qnum[f][l] = qq.num;
      h.qden[f][l] = qq.den;
    }
  }
  auto cleanup = [&](ltl4c_status r) {
    ltl4c_state_free(st);
    cudaSetDevice(prev);
    return r;
  };
  if (st->d_prog.ensure(1) || st->d_acc.ensure(1) || st->d_out.ensure(1) || st->d_nvalid.ensure(1))
    return cleanup(fail(LTL4C_E_OOM, "device allocation failed"));
  if (cudaMallocHost((void **)&st->h_out, sizeof(DevOut)) != cudaSuccess)
    return cleanup(fail(LTL4C_E_OOM, "pinned allocation failed"));
  std::memset(st->h_out, 0, sizeof(DevOut));
  if (cudaMemcpy(st->d_prog.p, &h, sizeof(DevProg), cudaMemcpyHostToDevice) != cudaSuccess ||
      cudaMemset(st->d_acc.p, 0, sizeof(DevAcc)) != cudaSuccess)
    return cleanup(fail(LTL4C_E_CUDA, "initialisation copy failed"));
  if (capacity_hint) {
    const int K = (int)prog->n_levels;
    for (int i = 0; i < 2; ++i) {
      for (int l = 0; l < K; ++l)
        if (st->bufkey[i][l].ensure(capacity_hint + 16)) return cleanup(fail(LTL4C_E_OOM, "buffer allocation failed"));
      if (st->buflet[i].ensure(capacity_hint + 16)) return cleanup(fail(LTL4C_E_OOM, "buffer allocation failed"));
    }
  }
  st->n_sms = dp.multiProcessorCount;
  {
    // warp-per-unit kernel: the (warps per CTA, CTAs per SM) pair that keeps the
    // most warps resident for this program's (K, F) shared-memory plan
    cudaError_t e = bucket_warp_config((int)prog->n_levels, (int)prog->n_formulas, (int)prog->n_states,
                                       (int)prog->letter_bits, st->warp_cfg);
    if (e == cudaSuccess)
      e = online_leaf_config((int)prog->n_levels, (int)prog->n_formulas, (int)prog->n_states, (int)prog->letter_bits,
                             st->online_cfg);
    if (e != cudaSuccess) return cleanup(fail(LTL4C_E_CUDA, std::string("bucket_warp_config: ") + cudaGetErrorString(e)));
    if (prog->n_levels == 1) {
      st->hot_mapk = prog->n_states <= 4 && prog->letter_bits <= 4 ? 0 : prog->n_states <= 8 ? 1 : -1;
      if (st->hot_mapk >= 0) st->hot_per_sm = hot_ctas_per_sm(st->hot_mapk);
      st->seg_per_sm = bucket_seg_ctas_per_sm((int)prog->n_states);
      if (st->hot_mapk == 0) st->coarse_per_sm = bucket_coarse_ctas_per_sm();
    }
  }
  cudaSetDevice(prev);
  *out = st;
  return LTL4C_OK;
}

ltl4c_status ltl4c_nccl_unique_id(void *out128) {
  if (!out128) return fail(LTL4C_E_INVALID, "null argument");
  Nccl *nc = nccl();
  if (!nc) return fail(LTL4C_E_NCCL, "NCCL library not found");
  NcclId id;
  NC(nc->GetUniqueId(&id));
  std::memcpy(out128, &id, sizeof id);
  return LTL4C_OK;
}

ltl4c_status ltl4c_state_comm(ltl4c_state *st, const void *nccl_id, int n_ranks, int rank) {
  if (!st) return fail(LTL4C_E_INVALID, "null state");
  if (n_ranks < 1 || rank < 0 || rank >= n_ranks) return fail(LTL4C_E_INVALID, "bad rank / size");
  if (n_ranks > 256 || (n_ranks & (n_ranks - 1)))
    return fail(LTL4C_E_INVALID, "the number of ranks must be a power of two <= 256");
  if (n_ranks > 1 && !nccl_id) return fail(LTL4C_E_INVALID, "null NCCL id");
  if (st->verifies) return fail(LTL4C_E_INVALID, "join the communicator before the first verify");
  Nccl *nc = nccl();
  if (!nc) return fail(LTL4C_E_NCCL, "NCCL library not found");
  int prev = 0;
  cudaGetDevice(&prev);
  CU(cudaSetDevice(st->device));
  NcclId id;
  if (n_ranks > 1) std::memcpy(&id, nccl_id, sizeof id);
  else NC(nc->GetUniqueId(&id));
  void *comm = nullptr;
  const int rc = nc->CommInitRank(&comm, n_ranks, id, rank);
  if (rc != 0) {
    cudaSetDevice(prev);
    return fail(LTL4C_E_NCCL, std::string("ncclCommInitRank: ") + (nc->ErrStr ? nc->ErrStr(rc) : "error"));
  }
  st->comm = comm;
  st->n_ranks = n_ranks;
  st->rank = rank;
  st->owner_bits = 0;
  while ((1 << st->owner_bits) < n_ranks) ++st->owner_bits;
  if (st->d_gacc.ensure(1) || st->d_sacc.ensure(1) ||
      (!st->hc_cnt && cudaMallocHost((void **)&st->hc_cnt, sizeof(unsigned long long) * (256 + 256 * 256)) != cudaSuccess)) {
    cudaSetDevice(prev);
    return fail(LTL4C_E_OOM, "allocation failed");
  }
  cudaSetDevice(prev);
  return LTL4C_OK;
}

ltl4c_status ltl4c_verify(ltl4c_state *st, const ltl4c_batch *batch, void *cuda_stream, ltl4c_result *out) {
  return verify_common(st, batch, cuda_stream, out, false);
}

ltl4c_status ltl4c_verify_host(ltl4c_state *st, const ltl4c_batch *batch, void *cuda_stream,
                               ltl4c_result *out) {
  return verify_common(st, batch, cuda_stream, out, true);
}

ltl4c_status ltl4c_verify_async(ltl4c_state *st, const ltl4c_batch *batch, void *cuda_stream, uint64_t *ticket) {
  if (!st || !batch || !ticket) return fail(LTL4C_E_INVALID, "null argument");
  if (!(st->flags & LTL4C_STATE_ONLINE)) return fail(LTL4C_E_INVALID, "ltl4c_verify_async needs an online state");
  if (st->comm) return fail(LTL4C_E_INVALID, "ltl4c_verify_async is single-GPU (no communicator)");
  const uint64_t t = st->next_ticket;
  const int slot = (int)(t % ltl4c_state::kRing);
  if (st->ring_ticket[slot]) return fail(LTL4C_E_INVALID, "too many results outstanding (read them with ltl4c_result_get)");
  int prev = 0;
  cudaGetDevice(&prev);
  if (prev != st->device) CU(cudaSetDevice(st->device));
  if (!st->ring_out) {
    if (cudaMallocHost((void **)&st->ring_out, sizeof(DevOut) * ltl4c_state::kRing) != cudaSuccess) {
      cudaSetDevice(prev);
      return fail(LTL4C_E_OOM, "pinned allocation failed");
    }
    for (int i = 0; i < ltl4c_state::kRing; ++i) CU(cudaEventCreateWithFlags(&st->ring_ev[i], cudaEventDisableTiming));
  }
  ltl4c_status r = verify_common(st, batch, cuda_stream, nullptr, false, &st->ring_out[slot]);
  if (!r) {
    if (cudaEventRecord(st->ring_ev[slot], (cudaStream_t)cuda_stream) != cudaSuccess) r = fail(LTL4C_E_CUDA, "event record");
  }
  if (prev != st->device) cudaSetDevice(prev);
  if (r) return r;
  st->ring_ticket[slot] = t;
  st->ring_seen[slot] = st->events_seen;
  st->ring_cum[slot] = st->enq_events;
  st->next_ticket = t + 1;
  st->outstanding++;
  *ticket = t;
  return LTL4C_OK;
}

ltl4c_status ltl4c_result_get(ltl4c_state *st, uint64_t ticket, ltl4c_result *out) {
  if (!st || !out) return fail(LTL4C_E_INVALID, "null argument");
  const int slot = (int)(ticket % ltl4c_state::kRing);
  if (ticket == 0 || st->ring_ticket[slot] != ticket) return fail(LTL4C_E_INVALID, "unknown or already read ticket");
  CU(cudaEventSynchronize(st->ring_ev[slot]));
  const DevOut &o = st->ring_out[slot];
  st->ring_ticket[slot] = 0;
  st->outstanding--;
  if (o.table_overflow) {
    st->poisoned = true;
    return fail(LTL4C_E_OOM, "carried table overflow");
  }
  if (st->ring_cum[slot] >= st->known_cum) {
    st->known_leaves = o.leaves;
    for (int l = 0; l < kMaxLevels; ++l) st->known_nodes[l] = o.nodes[l];
    st->known_cum = st->ring_cum[slot];
  }
  fill_results(st, o, st->ring_seen[slot], false, out);
  return LTL4C_OK;
}

ltl4c_status ltl4c_state_reset(ltl4c_state *st) {
  if (!st) return fail(LTL4C_E_INVALID, "null state");
  int prev = 0;
  cudaGetDevice(&prev);
  CU(cudaSetDevice(st->device));
  // drain every batch still in flight (pipelined batches may run on a non-blocking
  // stream) before the accumulators are cleared on that stream
  for (int i = 0; i < ltl4c_state::kRing; ++i)
    if (st->ring_ticket[i]) { cudaEventSynchronize(st->ring_ev[i]); st->ring_ticket[i] = 0; }
  CU(cudaStreamSynchronize(st->cur_stream));
  CU(cudaMemsetAsync(st->d_acc.p, 0, sizeof(DevAcc), st->cur_stream));
  CU(cudaStreamSynchronize(st->cur_stream));
  std::memset(st->h_out, 0, sizeof(DevOut));
  st->outstanding = 0;
  st->known_leaves = st->known_cum = st->enq_events = 0;
  for (int l = 0; l < kMaxLevels; ++l) st->known_nodes[l] = 0;
  st->epoch++;  // every carried table slot becomes stale
  st->tab.d.epoch = st->epoch;
  st->poisoned = false;
  st->have_index = false;
  st->next_index = 0;
  st->events_seen = 0;
  cudaSetDevice(prev);
  return LTL4C_OK;
}

// ------------------------------------------------------------ checkpoint / restore
namespace {
struct CkptHeader {
  char magic[8];
  uint64_t prog_hash;
  uint32_t n_levels, n_formulas, have_index, epoch, batch_id, pad;
  uint64_t next_index, events_seen, known_leaves, known_nodes[kMaxLevels], known_cum;
  uint64_t leaf_cap, node_cap;
};
constexpr char kCkptMagic[8] = {'L', 'T', 'L', '4', 'C', 'K', '0', '1'};

uint64_t prog_hash(const DevProg &p) {  // FNV-1a over the program tables
  const unsigned char *b = reinterpret_cast<const unsigned char *>(&p);
  uint64_t h = 1469598103934665603ull;
  for (size_t i = 0; i < sizeof p; ++i) h = (h ^ b[i]) * 1099511628211ull;
  return h;
}

// (buffer, bytes) of every carried table, in blob order
std::vector<std::pair<void *, size_t>> carried_buffers(ltl4c_state *st, uint64_t leaf_cap, uint64_t node_cap) {
  std::vector<std::pair<void *, size_t>> v;
  Tables &t = st->tab;
  v.push_back({t.leaf_slot.p, sizeof(uint4) * leaf_cap});
  v.push_back({t.leaf_state.p, leaf_cap});
  for (int l = 1; l < (int)st->prog->n_levels; ++l) {
    v.push_back({t.node_slot[l].p, sizeof(uint4) * node_cap});
    v.push_back({t.node_verdict[l].p, sizeof(uint32_t) * node_cap});
    v.push_back({t.node_hist[l].p, sizeof(uint32_t) * node_cap * kMaxFormulas * 6});
    v.push_back({t.node_aux[l].p, sizeof(uint32_t) * node_cap});
  }
  return v;
}

ltl4c_status drain(ltl4c_state *st) {
  for (int i = 0; i < ltl4c_state::kRing; ++i)
    if (st->ring_ticket[i]) CU(cudaEventSynchronize(st->ring_ev[i]));
  if (st->cur_stream) CU(cudaStreamSynchronize(st->cur_stream));
  CU(cudaDeviceSynchronize());
  return LTL4C_OK;
}
}  // namespace

ltl4c_status ltl4c_state_checkpoint_size(ltl4c_state *st, uint64_t *bytes) {
  if (!st || !bytes) return fail(LTL4C_E_INVALID, "null argument");
  if (!(st->flags & LTL4C_STATE_ONLINE)) return fail(LTL4C_E_INVALID, "checkpoint of an offline state");
  const uint64_t lc = st->tab.d.leaf_cap, nc = st->prog->n_levels > 1 ? st->tab.d.node_cap[1] : 0;
  uint64_t n = sizeof(CkptHeader) + sizeof(DevAcc) + (sizeof(uint4) + 1) * lc;
  for (int l = 1; l < (int)st->prog->n_levels; ++l) n += (sizeof(uint4) + 4 + 4 * kMaxFormulas * 6 + 4) * nc;
  *bytes = n;
  return LTL4C_OK;
}

ltl4c_status ltl4c_state_checkpoint(ltl4c_state *st, void *buf, uint64_t cap, uint64_t *written) {
  if (!st || !buf || !written) return fail(LTL4C_E_INVALID, "null argument");
  uint64_t need = 0;
  if (ltl4c_status r = ltl4c_state_checkpoint_size(st, &need)) return r;
  if (cap < need) return fail(LTL4C_E_INVALID, "checkpoint buffer too small");
  int prev = 0;
  cudaGetDevice(&prev);
  CU(cudaSetDevice(st->device));
  if (ltl4c_status r = drain(st)) return r;
  // the stream position and counters as of the last batch (results in flight included)
  for (int i = 0; i < ltl4c_state::kRing; ++i) st->ring_ticket[i] = 0;
  st->outstanding = 0;
  unsigned long long cnt[1 + kMaxLevels];
  CU(cudaMemcpy(cnt, &st->d_acc.p->leaves, sizeof cnt, cudaMemcpyDeviceToHost));
  st->known_leaves = cnt[0];
  for (int l = 0; l < kMaxLevels; ++l) st->known_nodes[l] = cnt[1 + l];
  st->known_cum = st->enq_events;
  CkptHeader h{};
  std::memcpy(h.magic, kCkptMagic, 8);
  h.prog_hash = prog_hash(st->hprog);
  h.n_levels = st->prog->n_levels;
  h.n_formulas = st->prog->n_formulas;
  h.have_index = st->have_index;
  h.epoch = st->tab.d.leaf_cap ? st->tab.d.epoch : st->epoch;
  h.batch_id = st->batch_id;
  h.next_index = st->next_index;
  h.events_seen = st->events_seen;
  h.known_leaves = st->known_leaves;
  for (int l = 0; l < kMaxLevels; ++l) h.known_nodes[l] = st->known_nodes[l];
  h.known_cum = 0;
  h.leaf_cap = st->tab.d.leaf_cap;
  h.node_cap = st->prog->n_levels > 1 ? st->tab.d.node_cap[1] : 0;
  unsigned char *o = static_cast<unsigned char *>(buf);
  std::memcpy(o, &h, sizeof h);
  o += sizeof h;
  CU(cudaMemcpy(o, st->d_acc.p, sizeof(DevAcc), cudaMemcpyDeviceToHost));
  o += sizeof(DevAcc);
  if (h.leaf_cap)
    for (auto &b : carried_buffers(st, h.leaf_cap, h.node_cap)) {
      CU(cudaMemcpy(o, b.first, b.second, cudaMemcpyDeviceToHost));
      o += b.second;
    }
  *written = (uint64_t)(o - static_cast<unsigned char *>(buf));
  cudaSetDevice(prev);
  return LTL4C_OK;
}

ltl4c_status ltl4c_state_restore(ltl4c_state *st, const void *buf, uint64_t len) {
  if (!st || !buf) return fail(LTL4C_E_INVALID, "null argument");
  if (!(st->flags & LTL4C_STATE_ONLINE)) return fail(LTL4C_E_INVALID, "restore into an offline state");
  CkptHeader h;
  if (len < sizeof h) return fail(LTL4C_E_INVALID, "not a checkpoint");
  std::memcpy(&h, buf, sizeof h);
  if (std::memcmp(h.magic, kCkptMagic, 8) != 0) return fail(LTL4C_E_INVALID, "not a checkpoint");
  if (h.prog_hash != prog_hash(st->hprog) || h.n_levels != st->prog->n_levels || h.n_formulas != st->prog->n_formulas)
    return fail(LTL4C_E_INVALID, "checkpoint of another program");
  uint64_t need = sizeof h + sizeof(DevAcc);
  if (h.leaf_cap) {
    need += (sizeof(uint4) + 1) * h.leaf_cap;
    for (uint32_t l = 1; l < h.n_levels; ++l) need += (sizeof(uint4) + 4 + 4 * kMaxFormulas * 6 + 4) * h.node_cap;
  }
  if (len < need) return fail(LTL4C_E_INVALID, "truncated checkpoint");
  int prev = 0;
  cudaGetDevice(&prev);
  CU(cudaSetDevice(st->device));
  if (ltl4c_status r = drain(st)) return r;
  for (int i = 0; i < ltl4c_state::kRing; ++i) st->ring_ticket[i] = 0;
  st->outstanding = 0;
  st->tab.release();
  const unsigned char *in = static_cast<const unsigned char *>(buf) + sizeof h;
  CU(cudaMemcpy(st->d_acc.p, in, sizeof(DevAcc), cudaMemcpyHostToDevice));
  in += sizeof(DevAcc);
  if (h.leaf_cap) {
    if (ltl4c_status r = alloc_tables(st, st->tab, h.leaf_cap, std::max<uint64_t>(h.node_cap, 1), 0, false, true)) return r;
    CU(cudaDeviceSynchronize());
    for (auto &b : carried_buffers(st, h.leaf_cap, h.node_cap)) {
      CU(cudaMemcpy(b.first, in, b.second, cudaMemcpyHostToDevice));
      in += b.second;
    }
    st->tab.d.epoch = h.epoch;
  }
  st->epoch = h.epoch;
  st->batch_id = h.batch_id;
  st->have_index = h.have_index != 0;
  st->next_index = h.next_index;
  st->events_seen = h.events_seen;
  st->known_leaves = h.known_leaves;
  for (int l = 0; l < kMaxLevels; ++l) st->known_nodes[l] = h.known_nodes[l];
  st->enq_events = st->known_cum = 0;
  st->poisoned = false;
  std::memset(st->h_out, 0, sizeof(DevOut));
  cudaSetDevice(prev);
  return LTL4C_OK;
}

ltl4c_status ltl4c_state_compact(ltl4c_state *st) {
  if (!st) return fail(LTL4C_E_INVALID, "null state");
  if (!(st->flags & LTL4C_STATE_ONLINE)) return fail(LTL4C_E_INVALID, "compact of an offline state");
  if (st->tab.d.leaf_cap == 0) return LTL4C_OK;
  int prev = 0;
  cudaGetDevice(&prev);
  CU(cudaSetDevice(st->device));
  if (ltl4c_status r = drain(st)) return r;
  for (int i = 0; i < ltl4c_state::kRing; ++i) st->ring_ticket[i] = 0;
  st->outstanding = 0;
  unsigned long long cnt[1 + kMaxLevels];
  CU(cudaMemcpy(cnt, &st->d_acc.p->leaves, sizeof cnt, cudaMemcpyDeviceToHost));
  st->known_leaves = cnt[0];
  uint64_t nodes = 0;
  for (int l = 0; l < kMaxLevels; ++l) {
    st->known_nodes[l] = cnt[1 + l];
    if (l >= 1 && l < (int)st->prog->n_levels) nodes = std::max<uint64_t>(nodes, cnt[1 + l]);
  }
  st->known_cum = st->enq_events = 0;
  // the smallest power-of-two capacities holding the live entries at load <= 1/2
  const uint64_t want_leaf = 1ull << std::max(12, ceil_log2(2 * st->known_leaves + 1));
  const uint64_t want_node = 1ull << std::max(12, ceil_log2(2 * nodes + 1));
  const bool smaller = want_leaf < st->tab.d.leaf_cap ||
                       (st->prog->n_levels > 1 && want_node < st->tab.d.node_cap[1]);
  if (smaller) {
    Tables nt;
    Launcher L{0, nullptr, nullptr, nullptr};
    if (ltl4c_status r = alloc_tables(st, nt, want_leaf, want_node, 0, false, true)) return r;
    nt.d.epoch = st->tab.d.epoch;
    CU(launch_rehash(st->tab.d, nt.d, (int)st->prog->n_levels, (int)st->prog->n_formulas,
                     &st->d_acc.p->table_overflow, L));
    CU(cudaDeviceSynchronize());
    st->tab.release();
    st->tab = nt;
    nt = Tables{};
  }
  cudaSetDevice(prev);
  return LTL4C_OK;
}

ltl4c_status ltl4c_state_nodes(ltl4c_state *st, uint32_t level, uint32_t formula, uint32_t *const *keys,
                               uint8_t *verdicts, uint64_t cap, uint64_t *count) {
  if (!st || !count) return fail(LTL4C_E_INVALID, "null argument");
  if (!(st->flags & LTL4C_STATE_ONLINE)) return fail(LTL4C_E_INVALID, "node dump of an offline state");
  const uint32_t K = st->prog->n_levels;
  if (level < 1 || level > K || formula >= st->prog->n_formulas) return fail(LTL4C_E_INVALID, "level or formula out of range");
  if (cap && (!verdicts || !keys)) return fail(LTL4C_E_INVALID, "null output buffer");
  *count = 0;
  const bool leaf = level == K;
  const uint64_t n = leaf ? st->tab.d.leaf_cap : st->tab.d.node_cap[level];
  if (n == 0) return LTL4C_OK;
  int prev = 0;
  cudaGetDevice(&prev);
  CU(cudaSetDevice(st->device));
  if (ltl4c_status r = drain(st)) return r;
  std::vector<uint4> slots(n);
  std::vector<uint8_t> state;
  std::vector<uint32_t> packed;
  CU(cudaMemcpy(slots.data(), leaf ? (const void *)st->tab.d.leaf_slot : (const void *)st->tab.d.node_slot[level],
                sizeof(uint4) * n, cudaMemcpyDeviceToHost));
  if (leaf) {
    state.resize(n);
    CU(cudaMemcpy(state.data(), st->tab.d.leaf_state, n, cudaMemcpyDeviceToHost));
  } else {
    packed.resize(n);
    CU(cudaMemcpy(packed.data(), st->tab.d.node_verdict[level], sizeof(uint32_t) * n, cudaMemcpyDeviceToHost));
  }
  const uint32_t ready = (st->tab.d.epoch << 1) | 1u;  // table tag of a live slot of this epoch
  uint64_t c = 0;
  for (uint64_t i = 0; i < n; ++i) {
    if (slots[i].x != ready) continue;
    if (c < cap) {
      const uint32_t kv[3] = {slots[i].y, slots[i].z, slots[i].w};
      for (uint32_t l = 0; l < level; ++l) keys[l][c] = kv[l];
      verdicts[c] = leaf ? st->hprog.lab[formula][state[i] & 0x7Fu] : (uint8_t)((packed[i] >> (8 * formula)) & 0xFFu);
    }
    ++c;
  }
  *count = c;
  cudaSetDevice(prev);
  return LTL4C_OK;
}

void ltl4c_state_free(ltl4c_state *st) {
  if (!st) return;
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(st->device);
  st->d_prog.release();
  st->d_acc.release();
  st->d_out.release();
  st->d_nvalid.release();
  for (int i = 0; i < 2; ++i) {
    for (int l = 0; l < kMaxLevels; ++l) st->bufkey[i][l].release();
    st->buflet[i].release();
  }
  st->counts.release();
  st->totals.release();
  st->bucket_off.release();
  st->oversize_list.release();
  st->medium_list.release();
  st->large_list.release();
  st->unit_start.release();
  st->sched.release();
  for (int l = 0; l < kMaxLevels; ++l) st->hkeys[l].release();
  st->hlet.release();
  st->tab.release();
  for (int l = 0; l < kMaxLevels; ++l) st->tlist[l].release();
  st->tcnt.release();
  st->h_part.release();
  st->h_lists.release();
  st->h_u32.release();
  st->h_cnt.release();
  st->hot_cnt.release();
  st->hot_tab.release();
  st->d_bid.release();
  st->hot_partial.release();
  st->hot_chunk.release();
  st->unit_start2.release();
  st->coarse_off.release();
  st->hot_n.release();
  for (auto &t : st->pending) {
    cudaEventDestroy(t.a);
    cudaEventDestroy(t.b);
  }
  for (auto e : st->event_pool) cudaEventDestroy(e);
  drop_graph(st);
  if (st->cap_stream) cudaStreamDestroy(st->cap_stream);
  if (st->comm && nccl() && nccl()->CommDestroy) nccl()->CommDestroy(st->comm);
  st->d_gacc.release();
  st->d_sacc.release();
  for (int l = 0; l < kMaxLevels; ++l) st->exkey[l].release();
  st->exlet.release();
  st->dc_cnt.release();
  if (st->hc_cnt) cudaFreeHost(st->hc_cnt);
  for (int i = 0; i < ltl4c_state::kRing; ++i)
    if (st->ring_ev[i]) cudaEventDestroy(st->ring_ev[i]);
  if (st->ring_out) cudaFreeHost(st->ring_out);
  if (st->h_out) cudaFreeHost(st->h_out);
  if (st->h_pack) cudaFreeHost(st->h_pack);
  if (st->pack_done) cudaEventDestroy(st->pack_done);
  st->d_pack.release();
  cudaSetDevice(prev);
  delete st;
}

ltl4c_status ltl4c_state_profile(ltl4c_state *st, int enable) {
  if (!st) return fail(LTL4C_E_INVALID, "null state");
  st->profiling = enable != 0;
  return LTL4C_OK;
}

ltl4c_status ltl4c_state_stats(ltl4c_state *st, ltl4c_stats *out) {
  if (!st || !out) return fail(LTL4C_E_INVALID, "null argument");
  drain_timings(st);
  std::memset(out, 0, sizeof *out);
  out->verifies = st->verifies;
  out->launches = st->launches;
  out->n_kernels = kKNumKernels;
  for (int k = 0; k < kKNumKernels; ++k) {
    std::snprintf(out->kernel_name[k], sizeof out->kernel_name[k], "%s", kKernelNames[k]);
    out->kernel_launches[k] = st->k_launches[k];
    out->kernel_ms[k] = st->k_ms[k];
  }
  return LTL4C_OK;
}

ltl4c_status ltl4c_state_stats_reset(ltl4c_state *st) {
  if (!st) return fail(LTL4C_E_INVALID, "null state");
  drain_timings(st);
  st->verifies = st->launches = 0;
  for (int k = 0; k < kKNumKernels; ++k) {
    st->k_launches[k] = 0;
    st->k_launches_saved[k] = 0;
    st->k_ms[k] = 0.0;
  }
  return LTL4C_OK;
}

}  // extern "C"
