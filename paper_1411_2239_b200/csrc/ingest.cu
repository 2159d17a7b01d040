// ingest.cu -- device-side trace ingest: JSON-lines key ->
// value records in device memory to the encoded batch layout of ltl4c_batch, on the
// GPU.  The paper's measured cost upstream of the monitor is its strace parsing
// module; here the records are structured logs.
//
// Semantics are those of the host encoder (encoder.cpp, include/ltl4c.h): §4.1
// "Valuation Extraction" ("the trace event is a key-value structure",
// epsilon(u_i, K)); guard key p_l -> the event's value for x_l if it is a JSON
// string or number, values identified by their canonical string (strings as
// written after unescaping, numbers as canonical decimals: 12 == 12.0 == 1.2e1 ==
// "12"); atoms per reading A12; the last occurrence of a repeated key wins;
// blank lines are skipped.  Dictionary ids are dense per level and persist across
// calls (an online stream shares them), but their ORDER is the order in which
// concurrent threads claim them, not first appearance: verdicts and counts are
// invariant to relabelling values (tests/test_oracle_pins.py), so only the
// partition of values into ids matters, and it is the host encoder's.
//
//   ingest_count   per 64 KB segment: newlines (one 256-thread CTA, 256 B a thread)
//   ingest_scan    exclusive scan of the segment counts (one CTA)
//   ingest_lines   line start offsets
//   ingest_parse   thread per line: a flat JSON object parsed in one pass; each
//                  value of interest hashed (64-bit, over its canonical bytes, never
//                  materialised); guard values -> dictionary ids (per-level table
//                  keyed by the hash: CAS claim, id from a counter, published once);
//                  atoms per A12; blank lines flagged
//   ingest_compact the events of non-blank lines packed in line order
// Values are identified by a 64-bit hash of their canonical bytes (reading A28:
// two distinct values of one key merge with probability ~ n^2 / 2^65).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <string>
#include <vector>

#include "kernels.cuh"
#include "program.h"
#include "util.cuh"

namespace ltl4c {

constexpr int kSegBytes = 1 << 16;       // bytes per ingest segment (256 threads x 256 B)
constexpr int kMaxAtomsB = LTL4C_MAX_BATCH_ATOMS;
constexpr int kMaxNames = kMaxLevels + kMaxAtomsB;

struct IngestParams {
  const char *text;
  unsigned long long len;
  uint32_t n_seg;
  uint32_t *seg_cnt;                    // [n_seg + 1] newlines per segment -> exclusive scan
  unsigned long long *line_start;       // [n_lines + 1]
  unsigned long long n_lines;           // (host upper bound for the grids)
  const unsigned long long *d_n_lines;  // (device)
  int K, A;
  unsigned long long name_hash[kMaxNames];  // K guard keys, then A atom predicates
  int atom_nargs[kMaxAtomsB];
  int atom_lv[kMaxAtomsB][kMaxLevels];
  const uint8_t *letter_class;               // [1 << A] letter code of each valuation, or null (code = valuation)
  unsigned long long *dict_key[kMaxLevels];  // per level: 64-bit value hash (0 = empty)
  uint32_t *dict_id[kMaxLevels];             // dense id (ABSENT until published)
  unsigned long long dict_cap;               // power of two
  uint32_t *dict_count;                      // [K] ids handed out
  uint32_t *tmp_keys[kMaxLevels];            // per line
  uint8_t *tmp_let;
  uint32_t *valid;                           // per line: 1 = an event
  uint32_t *pos;                             // exclusive scan of valid (blocks of 1024 lines)
  uint32_t *blk;                             // block sums
  uint32_t *keys_out[kMaxLevels];
  uint8_t *let_out;
  unsigned long long *n_out;
  unsigned long long *err_line;              // smallest malformed line + 1 (0: none)
  unsigned long long *overflow;              // dictionary full
};

namespace {

__device__ __forceinline__ unsigned long long fmix64(unsigned long long k) {
  k ^= k >> 33;
  k *= 0xff51afd7ed558ccdull;
  k ^= k >> 33;
  k *= 0xc4ceb9fe1a85ec53ull;
  k ^= k >> 33;
  return k;
}
struct Hash {  // FNV-1a over the canonical bytes, finalised by fmix64
  unsigned long long h = 1469598103934665603ull;
  __device__ void put(uint32_t c) { h = (h ^ (c & 0xFFu)) * 1099511628211ull; }
  __device__ unsigned long long done() const {
    const unsigned long long r = fmix64(h);
    return r ? r : 1ull;
  }
};

__device__ __forceinline__ bool is_ws(char c) { return c == ' ' || c == '\t' || c == '\r'; }

struct Cursor {
  const char *p, *end;
  bool bad = false;
  __device__ void ws() {
    while (p < end && is_ws(*p)) ++p;
  }
  __device__ char peek() const { return p < end ? *p : '\0'; }
};

__device__ bool hex4(Cursor &c, uint32_t *v) {
  if (c.end - c.p < 4) return false;
  *v = 0;
  for (int i = 0; i < 4; ++i) {
    const char x = c.p[i];
    *v <<= 4;
    if (x >= '0' && x <= '9') *v |= (uint32_t)(x - '0');
    else if (x >= 'a' && x <= 'f') *v |= (uint32_t)(x - 'a' + 10);
    else if (x >= 'A' && x <= 'F') *v |= (uint32_t)(x - 'A' + 10);
    else return false;
  }
  c.p += 4;
  return true;
}
__device__ void put_utf8(Hash &h, uint32_t c) {
  if (c < 0x80) h.put(c);
  else if (c < 0x800) { h.put(0xC0 | (c >> 6)); h.put(0x80 | (c & 63)); }
  else if (c < 0x10000) { h.put(0xE0 | (c >> 12)); h.put(0x80 | ((c >> 6) & 63)); h.put(0x80 | (c & 63)); }
  else { h.put(0xF0 | (c >> 18)); h.put(0x80 | ((c >> 12) & 63)); h.put(0x80 | ((c >> 6) & 63)); h.put(0x80 | (c & 63)); }
}
// string at '"': its unescaped bytes hashed
__device__ bool str(Cursor &c, Hash &h) {
  ++c.p;
  while (c.p < c.end && *c.p != '"') {
    if (*c.p != '\\') { h.put((uint8_t)*c.p++); continue; }
    if (++c.p >= c.end) return false;
    const char e = *c.p++;
    switch (e) {
      case '"': h.put('"'); break;
      case '\\': h.put('\\'); break;
      case '/': h.put('/'); break;
      case 'b': h.put('\b'); break;
      case 'f': h.put('\f'); break;
      case 'n': h.put('\n'); break;
      case 'r': h.put('\r'); break;
      case 't': h.put('\t'); break;
      case 'u': {
        uint32_t u;
        if (!hex4(c, &u)) return false;
        if (u >= 0xD800 && u < 0xDC00 && c.end - c.p >= 6 && c.p[0] == '\\' && c.p[1] == 'u') {
          c.p += 2;
          uint32_t lo;
          if (!hex4(c, &lo)) return false;
          if (lo >= 0xDC00 && lo < 0xE000) u = 0x10000 + ((u - 0xD800) << 10) + (lo - 0xDC00);
          else { put_utf8(h, u); u = lo; }
        }
        put_utf8(h, u);
        break;
      }
      default: return false;
    }
  }
  if (c.p >= c.end) return false;
  ++c.p;
  return true;
}
// number: its canonical decimal (leading / trailing zeros dropped, the point placed
// by the exponent; "0" for zero) hashed
__device__ bool num(Cursor &c, Hash &h) {
  bool neg = false;
  if (c.peek() == '-') { neg = true; ++c.p; }
  const char *ip = c.p;
  if (!(c.peek() >= '0' && c.peek() <= '9')) return false;
  while (c.peek() >= '0' && c.peek() <= '9') ++c.p;
  const char *ie = c.p, *fp = c.p, *fe = c.p;
  if (c.peek() == '.') {
    ++c.p;
    fp = c.p;
    if (!(c.peek() >= '0' && c.peek() <= '9')) return false;
    while (c.peek() >= '0' && c.peek() <= '9') ++c.p;
    fe = c.p;
  }
  long long e = 0;
  if (c.peek() == 'e' || c.peek() == 'E') {
    ++c.p;
    bool en = false;
    if (c.peek() == '+' || c.peek() == '-') en = *c.p++ == '-';
    if (!(c.peek() >= '0' && c.peek() <= '9')) return false;
    while (c.peek() >= '0' && c.peek() <= '9') {
      e = e * 10 + (*c.p++ - '0');
      if (e > 4096) return false;
    }
    if (en) e = -e;
  }
  // digit string D = integer digits . fraction digits; point = #integer digits + e
  const long long ni = ie - ip, nf = fe - fp;
  auto dig = [&](long long i) { return i < ni ? ip[i] : fp[i - ni]; };
  long long a = 0, b = ni + nf;  // [a, b) = D without leading / trailing zeros
  while (a < b && dig(a) == '0') ++a;
  while (b > a && dig(b - 1) == '0') --b;
  if (a == b) { h.put('0'); return true; }
  const long long point = ni + e - a, nd = b - a;
  if (neg) h.put('-');
  if (point <= 0) {
    h.put('0');
    h.put('.');
    for (long long i = 0; i < -point; ++i) h.put('0');
    for (long long i = a; i < b; ++i) h.put(dig(i));
  } else if (point >= nd) {
    for (long long i = a; i < b; ++i) h.put(dig(i));
    for (long long i = 0; i < point - nd; ++i) h.put('0');
  } else {
    for (long long i = 0; i < point; ++i) h.put(dig(a + i));
    h.put('.');
    for (long long i = a + point; i < b; ++i) h.put(dig(i));
  }
  return true;
}
__device__ bool lit(Cursor &c, const char *w, int n) {
  if (c.end - c.p < n) return false;
  for (int i = 0; i < n; ++i)
    if (c.p[i] != w[i]) return false;
  c.p += n;
  return true;
}
// a value we do not keep (nested array / object): skipped with its strings
__device__ bool skip_nested(Cursor &c) {
  int depth = 0;
  do {
    const char x = c.peek();
    if (x == '\0' && c.p >= c.end) return false;
    if (x == '"') {
      Hash d;
      if (!str(c, d)) return false;
      continue;
    }
    if (x == '[' || x == '{') ++depth;
    else if (x == ']' || x == '}') --depth;
    ++c.p;
    if (depth > 64) return false;
  } while (depth > 0);
  return true;
}

enum : uint8_t { kVNone = 0, kVTrue, kVOther, kVScalar, kVArray };
struct Val {
  uint8_t kind = kVNone;
  uint8_t n_items = 0;       // kVArray: items kept (scalars), 0xFF = a non-scalar item
  unsigned long long h = 0;  // kVScalar
  unsigned long long item[kMaxLevels];
};

// one value (at c.p, after whitespace)
__device__ bool value(Cursor &c, Val &v) {
  const char x = c.peek();
  v = Val{};
  if (x == '"') { Hash h; if (!str(c, h)) return false; v.kind = kVScalar; v.h = h.done(); return true; }
  if (x == '-' || (x >= '0' && x <= '9')) { Hash h; if (!num(c, h)) return false; v.kind = kVScalar; v.h = h.done(); return true; }
  if (x == 't') { v.kind = kVTrue; return lit(c, "true", 4); }
  if (x == 'f') { v.kind = kVOther; return lit(c, "false", 5); }
  if (x == 'n') { v.kind = kVOther; return lit(c, "null", 4); }
  if (x == '{') { v.kind = kVOther; return skip_nested(c); }
  if (x == '[') {
    ++c.p;
    v.kind = kVArray;
    c.ws();
    if (c.peek() == ']') { ++c.p; return true; }
    while (true) {
      c.ws();
      const char y = c.peek();
      if (y == '"' || y == '-' || (y >= '0' && y <= '9')) {
        Hash h;
        if (!(y == '"' ? str(c, h) : num(c, h))) return false;
        if (v.n_items != 0xFF) {
          if (v.n_items < kMaxLevels) v.item[v.n_items] = h.done();
          v.n_items = v.n_items < kMaxLevels ? v.n_items + 1 : 0xFF;  // (longer than any atom)
        }
      } else if (y == '[' || y == '{') {
        if (!skip_nested(c)) return false;
        v.n_items = 0xFF;
      } else if (y == 't' || y == 'f' || y == 'n') {
        if (!(lit(c, "true", 4) || lit(c, "false", 5) || lit(c, "null", 4))) return false;
        v.n_items = 0xFF;
      } else {
        return false;
      }
      c.ws();
      if (c.peek() == ',') { ++c.p; continue; }
      if (c.peek() == ']') { ++c.p; return true; }
      return false;
    }
  }
  return false;
}

__device__ uint32_t dict_id(const IngestParams &p, int l, unsigned long long h) {
  unsigned long long s = fmix64(h ^ 0x9e3779b97f4a7c15ull) & (p.dict_cap - 1);
  for (unsigned long long probes = 0; probes < p.dict_cap; ++probes) {
    unsigned long long k = *(volatile unsigned long long *)&p.dict_key[l][s];
    if (k == 0) {
      k = atomicCAS(&p.dict_key[l][s], 0ull, h);
      if (k == 0) {  // claimed: a new value
        const uint32_t id = atomicAdd(&p.dict_count[l], 1u);
        *(volatile uint32_t *)&p.dict_id[l][s] = id;
        return id;
      }
    }
    if (k == h) {  // published by its claimer (a thread that already passed its CAS)
      uint32_t id;
      while ((id = *(volatile uint32_t *)&p.dict_id[l][s]) == kAbsent) {
      }
      return id;
    }
    s = (s + 1) & (p.dict_cap - 1);
  }
  atomicAdd(p.overflow, 1ull);
  return kAbsent;
}

__global__ void __launch_bounds__(256) ingest_count_kernel(IngestParams p) {
  __shared__ uint32_t wsum[8];
  const unsigned long long b0 = (unsigned long long)blockIdx.x * kSegBytes + threadIdx.x * (kSegBytes / 256);
  uint32_t c = 0;
  for (int i = 0; i < kSegBytes / 256; i += 16) {
    const unsigned long long at = b0 + i;
    if (at + 16 <= p.len) {
      const uint4 v = __ldg(reinterpret_cast<const uint4 *>(p.text + at));
      const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int q = 0; q < 4; ++q)
#pragma unroll
        for (int y = 0; y < 4; ++y) c += ((w[q] >> (8 * y)) & 0xFFu) == '\n';
    } else {
      for (unsigned long long j = at; j < at + 16 && j < p.len; ++j) c += p.text[j] == '\n';
    }
  }
  c = __reduce_add_sync(0xffffffffu, c);
  if ((threadIdx.x & 31) == 0) wsum[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t t = 0;
    for (int w = 0; w < 8; ++w) t += wsum[w];
    p.seg_cnt[blockIdx.x] = t;
  }
}

// exclusive scan of a u32 array in place (one CTA of 1024 threads, any length);
// *total = the sum
__global__ void __launch_bounds__(1024) scan_u32_kernel(uint32_t *a, uint32_t n, unsigned long long *total,
                                                        unsigned long long add) {
  __shared__ uint32_t wsum[32];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const uint32_t per = (n + 1023) / 1024;
  const uint32_t lo = min(n, tid * per), hi = min(n, lo + per);
  uint32_t s = 0;
  for (uint32_t i = lo; i < hi; ++i) s += a[i];
  uint32_t inc = s;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, inc, d);
    if (lane >= d) inc += y;
  }
  if (lane == 31) wsum[wid] = inc;
  __syncthreads();
  if (wid == 0) {
    uint32_t t = wsum[lane];
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, t, d);
      if (lane >= d) t += y;
    }
    wsum[lane] = t;
  }
  __syncthreads();
  uint32_t run = inc - s + (wid ? wsum[wid - 1] : 0u);
  for (uint32_t i = lo; i < hi; ++i) {
    const uint32_t v = a[i];
    a[i] = run;
    run += v;
  }
  if (tid == 1023 && total) *total = (unsigned long long)run + add;
}

// line start offsets: line 0 starts at 0, line i + 1 after the i-th newline; the
// line after a final newline is the end of the text (a blank line)
__global__ void __launch_bounds__(256) ingest_lines_kernel(IngestParams p) {
  __shared__ uint32_t wsum[8];
  const unsigned long long b0 = (unsigned long long)blockIdx.x * kSegBytes + threadIdx.x * (kSegBytes / 256);
  uint32_t c = 0;
  for (int i = 0; i < kSegBytes / 256; ++i) c += b0 + i < p.len && p.text[b0 + i] == '\n';
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  uint32_t inc = c;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, inc, d);
    if (lane >= d) inc += y;
  }
  if (lane == 31) wsum[wid] = inc;
  __syncthreads();
  uint32_t before = 0;
  for (int w = 0; w < wid; ++w) before += wsum[w];
  unsigned long long line = (unsigned long long)p.seg_cnt[blockIdx.x] + before + inc - c;  // newlines before b0
  for (int i = 0; i < kSegBytes / 256; ++i) {
    const unsigned long long at = b0 + i;
    if (at < p.len && p.text[at] == '\n') p.line_start[++line] = at + 1;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) p.line_start[0] = 0;
}

__global__ void __launch_bounds__(128) ingest_parse_kernel(IngestParams p) {
  const unsigned long long n_lines = *p.d_n_lines;
  for (unsigned long long ln = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; ln < n_lines;
       ln += (unsigned long long)gridDim.x * blockDim.x) {
    const unsigned long long s0 = p.line_start[ln];
    unsigned long long s1 = ln + 1 < n_lines ? p.line_start[ln + 1] - 1 : p.len;  // (without its '\n')
    if (s1 > p.len) s1 = p.len;
    Cursor c{p.text + s0, p.text + s1};
    c.ws();
    uint32_t ok = 0;
    if (c.p < c.end) {  // (blank lines are no event)
      Val guard[kMaxLevels];
      Val atom[kMaxAtomsB];
      bool good = c.peek() == '{';
      if (good) {
        ++c.p;
        c.ws();
        if (c.peek() == '}') ++c.p;
        else
          while (good) {
            c.ws();
            if (c.peek() != '"') { good = false; break; }
            Hash kh;
            if (!str(c, kh)) { good = false; break; }
            const unsigned long long k = kh.done();
            c.ws();
            if (c.peek() != ':') { good = false; break; }
            ++c.p;
            c.ws();
            Val v;
            if (!value(c, v)) { good = false; break; }
            for (int l = 0; l < p.K; ++l)
              if (k == p.name_hash[l]) guard[l] = v;  // (the last occurrence wins)
            for (int j = 0; j < p.A; ++j)
              if (k == p.name_hash[p.K + j]) atom[j] = v;
            c.ws();
            if (c.peek() == ',') { ++c.p; continue; }
            if (c.peek() == '}') { ++c.p; break; }
            good = false;
          }
        c.ws();
        if (good && c.p != c.end) good = false;  // trailing characters
      }
      if (!good) {
        atomicMin(p.err_line, ln + 1);
      } else {
        ok = 1;
        for (int l = 0; l < p.K; ++l)
          p.tmp_keys[l][ln] = guard[l].kind == kVScalar ? dict_id(p, l, guard[l].h) : kAbsent;
        uint32_t let = 0;
        for (int j = 0; j < p.A; ++j) {
          const Val &v = atom[j];
          bool holds = v.kind == kVTrue;
          const int na = p.atom_nargs[j];
          if (!holds && na == 1 && v.kind == kVScalar) {
            const Val &g = guard[p.atom_lv[j][0]];
            holds = g.kind == kVScalar && g.h == v.h;
          } else if (!holds && na >= 1 && v.kind == kVArray && v.n_items == na) {
            holds = true;
            for (int i = 0; i < na && holds; ++i) {
              const Val &g = guard[p.atom_lv[j][i]];
              holds = g.kind == kVScalar && g.h == v.item[i];
            }
          }
          if (holds) let |= 1u << j;
        }
        p.tmp_let[ln] = p.letter_class ? p.letter_class[let] : (uint8_t)let;
      }
    }
    p.valid[ln] = ok;
  }
}

// per block of 1024 lines: the count of events (block sums) / their packing
__global__ void __launch_bounds__(1024) ingest_blocks_kernel(IngestParams p) {
  const unsigned long long n_lines = *p.d_n_lines;
  const unsigned long long ln = (unsigned long long)blockIdx.x * 1024 + threadIdx.x;
  const uint32_t v = ln < n_lines ? p.valid[ln] : 0u;
  const uint32_t s = __syncthreads_count(v);
  if (threadIdx.x == 0) p.blk[blockIdx.x] = s;
}

__global__ void __launch_bounds__(1024) ingest_compact_kernel(IngestParams p) {
  __shared__ uint32_t wsum[32];
  const unsigned long long n_lines = *p.d_n_lines;
  const unsigned long long ln = (unsigned long long)blockIdx.x * 1024 + threadIdx.x;
  const uint32_t v = ln < n_lines ? p.valid[ln] : 0u;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const uint32_t b = __ballot_sync(0xffffffffu, v);
  if (lane == 0) wsum[wid] = __popc(b);
  __syncthreads();
  uint32_t before = 0;
  for (int w = 0; w < wid; ++w) before += wsum[w];
  if (v) {
    const unsigned long long at = (unsigned long long)p.blk[blockIdx.x] + before + __popc(b & lanemask_lt());
    for (int l = 0; l < p.K; ++l) p.keys_out[l][at] = p.tmp_keys[l][ln];
    p.let_out[at] = p.tmp_let[ln];
  }
}

}  // namespace

// host side ---------------------------------------------------------------------
struct DevIngest {
  int device = 0;
  const ltl4c_program *prog = nullptr;
  IngestParams base{};
  unsigned long long dict_cap = 0;
  void *scratch = nullptr;      // line tables + per-line outputs (grown on demand)
  size_t scratch_bytes = 0;
  unsigned long long *small = nullptr;  // [0] n_lines, [1] n_out, [2] err_line, [3] overflow
};

static unsigned long long host_name_hash(const std::string &s) {
  unsigned long long h = 1469598103934665603ull;
  for (unsigned char c : s) h = (h ^ c) * 1099511628211ull;
  h ^= h >> 33;
  h *= 0xff51afd7ed558ccdull;
  h ^= h >> 33;
  h *= 0xc4ceb9fe1a85ec53ull;
  h ^= h >> 33;
  return h ? h : 1ull;
}

cudaError_t ingest_create(DevIngest *e, const ltl4c_program *prog, int device, unsigned long long max_values) {
  e->device = device;
  e->prog = prog;
  IngestParams &b = e->base;
  b.K = (int)prog->n_levels;
  b.A = (int)prog->n_atoms;
  for (int l = 0; l < b.K; ++l) b.name_hash[l] = host_name_hash(prog->key_names[l]);
  for (int j = 0; j < b.A; ++j) {
    const std::string &nm = prog->atom_names[j];
    b.name_hash[b.K + j] = host_name_hash(nm.substr(0, nm.find('(')));
    const auto &lv = j < (int)prog->atom_levels.size() ? prog->atom_levels[j] : std::vector<int>();
    b.atom_nargs[j] = (int)lv.size();
    for (size_t i = 0; i < lv.size() && i < (size_t)kMaxLevels; ++i) b.atom_lv[j][i] = lv[i];
  }
  cudaError_t r;
  if (!prog->letter_class.empty()) {
    uint8_t *lc = nullptr;
    if ((r = cudaMalloc((void **)&lc, prog->letter_class.size()))) return r;
    if ((r = cudaMemcpy(lc, prog->letter_class.data(), prog->letter_class.size(), cudaMemcpyHostToDevice))) return r;
    b.letter_class = lc;
  }
  unsigned long long cap = 1024;
  while (cap < 2 * max_values + 1) cap <<= 1;
  e->dict_cap = cap;
  b.dict_cap = cap;
  for (int l = 0; l < b.K; ++l) {
    if ((r = cudaMalloc((void **)&b.dict_key[l], sizeof(unsigned long long) * cap))) return r;
    if ((r = cudaMalloc((void **)&b.dict_id[l], sizeof(uint32_t) * cap))) return r;
    if ((r = cudaMemset(b.dict_key[l], 0, sizeof(unsigned long long) * cap))) return r;
    if ((r = cudaMemset(b.dict_id[l], 0xFF, sizeof(uint32_t) * cap))) return r;
  }
  if ((r = cudaMalloc((void **)&b.dict_count, sizeof(uint32_t) * kMaxLevels))) return r;
  if ((r = cudaMemset(b.dict_count, 0, sizeof(uint32_t) * kMaxLevels))) return r;
  if ((r = cudaMalloc((void **)&e->small, sizeof(unsigned long long) * 8))) return r;
  return cudaDeviceSynchronize();
}

void ingest_free(DevIngest *e) {
  for (int l = 0; l < e->base.K; ++l) {
    cudaFree(e->base.dict_key[l]);
    cudaFree(e->base.dict_id[l]);
  }
  cudaFree(e->base.dict_count);
  cudaFree(const_cast<uint8_t *>(e->base.letter_class));
  cudaFree(e->small);
  cudaFree(e->scratch);
}

// encode text[0, len) (device) into keys / letters (device, capacity events)
cudaError_t ingest_run(DevIngest *e, const char *text, unsigned long long len, uint32_t *const *keys,
                       uint8_t *letters, unsigned long long capacity, cudaStream_t s, unsigned long long *n_events,
                       unsigned long long *err_line, unsigned long long *overflow, unsigned long long *n_lines_out) {
  IngestParams p = e->base;
  p.text = text;
  p.len = len;
  p.n_seg = (uint32_t)((len + kSegBytes - 1) / kSegBytes);
  // lines <= newlines + 1; count them first (one small D2H to size the line tables)
  const size_t seg_b = sizeof(uint32_t) * (p.n_seg + 2);
  auto align = [](size_t x) { return (x + 255) & ~(size_t)255; };
  size_t need = align(seg_b);
  if (need > e->scratch_bytes) {
    cudaFree(e->scratch);
    e->scratch = nullptr;
    e->scratch_bytes = 0;
    cudaError_t r = cudaMalloc(&e->scratch, need);
    if (r) return r;
    e->scratch_bytes = need;
  }
  p.seg_cnt = reinterpret_cast<uint32_t *>(e->scratch);
  cudaMemsetAsync(e->small, 0, sizeof(unsigned long long) * 8, s);
  cudaMemsetAsync(p.seg_cnt, 0, seg_b, s);
  if (p.n_seg) ingest_count_kernel<<<p.n_seg, 256, 0, s>>>(p);
  scan_u32_kernel<<<1, 1024, 0, s>>>(p.seg_cnt, p.n_seg + 1, e->small, 1);  // lines = newlines + 1
  unsigned long long n_lines = 0;
  cudaMemcpyAsync(&n_lines, e->small, sizeof n_lines, cudaMemcpyDeviceToHost, s);
  cudaError_t r = cudaStreamSynchronize(s);
  if (r) return r;
  if (len == 0) n_lines = 0;
  const unsigned long long nblk = (n_lines + 1023) / 1024;
  need = align(seg_b) + align(sizeof(unsigned long long) * (n_lines + 1)) +
         align((sizeof(uint32_t) * p.K + 1 + 2 * sizeof(uint32_t)) * (n_lines + 1)) + align(sizeof(uint32_t) * (nblk + 1));
  if (need > e->scratch_bytes) {
    // keep the segment scan: copy it out of the old scratch
    void *ns = nullptr;
    if ((r = cudaMalloc(&ns, need))) return r;
    cudaMemcpyAsync(ns, e->scratch, seg_b, cudaMemcpyDeviceToDevice, s);
    if ((r = cudaStreamSynchronize(s))) return r;
    cudaFree(e->scratch);
    e->scratch = ns;
    e->scratch_bytes = need;
    p.seg_cnt = reinterpret_cast<uint32_t *>(ns);
  }
  char *q = reinterpret_cast<char *>(e->scratch) + align(seg_b);
  p.line_start = reinterpret_cast<unsigned long long *>(q);
  q += align(sizeof(unsigned long long) * (n_lines + 1));
  for (int l = 0; l < p.K; ++l) {
    p.tmp_keys[l] = reinterpret_cast<uint32_t *>(q);
    q += sizeof(uint32_t) * (n_lines + 1);
  }
  p.valid = reinterpret_cast<uint32_t *>(q);
  q += sizeof(uint32_t) * (n_lines + 1);
  p.tmp_let = reinterpret_cast<uint8_t *>(q);
  q = reinterpret_cast<char *>(align(reinterpret_cast<size_t>(q + n_lines + 1)));
  p.blk = reinterpret_cast<uint32_t *>(q);
  p.n_lines = n_lines;
  p.d_n_lines = e->small;
  p.n_out = e->small + 1;
  p.err_line = e->small + 2;
  p.overflow = e->small + 3;
  cudaMemsetAsync(p.err_line, 0xFF, sizeof(unsigned long long), s);  // (atomicMin)
  for (int l = 0; l < p.K; ++l) p.keys_out[l] = keys[l];
  p.let_out = letters;
  if (n_lines) {
    ingest_lines_kernel<<<p.n_seg, 256, 0, s>>>(p);
    const unsigned grid = (unsigned)std::min<unsigned long long>((n_lines + 127) / 128, 148ull * 16);
    ingest_parse_kernel<<<grid, 128, 0, s>>>(p);
    ingest_blocks_kernel<<<(unsigned)nblk, 1024, 0, s>>>(p);
    scan_u32_kernel<<<1, 1024, 0, s>>>(p.blk, (uint32_t)nblk, p.n_out, 0);
  }
  unsigned long long small[4] = {0, 0, 0, 0};
  cudaMemcpyAsync(small, e->small, sizeof small, cudaMemcpyDeviceToHost, s);
  if ((r = cudaStreamSynchronize(s))) return r;
  *n_events = n_lines ? small[1] : 0;
  *err_line = small[2] == ~0ull ? 0 : small[2];
  *overflow = small[3];
  *n_lines_out = n_lines;
  if (*err_line || *overflow || *n_events > capacity) return cudaSuccess;  // (the caller reports it)
  if (n_lines) ingest_compact_kernel<<<(unsigned)nblk, 1024, 0, s>>>(p);
  if ((r = cudaGetLastError())) return r;
  return cudaStreamSynchronize(s);
}

}  // namespace ltl4c

using namespace ltl4c;

struct ltl4c_dencoder {
  DevIngest e;
};

extern "C" {

ltl4c_status ltl4c_dencoder_create(const ltl4c_program *prog, int device, uint64_t max_values, ltl4c_dencoder **out) {
  if (!prog || !out) return fail(LTL4C_E_INVALID, "null argument");
  int prev = 0;
  cudaGetDevice(&prev);
  if (cudaSetDevice(device) != cudaSuccess) return fail(LTL4C_E_CUDA, "cudaSetDevice failed");
  auto *d = new ltl4c_dencoder();
  const cudaError_t r = ingest_create(&d->e, prog, device, std::max<uint64_t>(max_values, 1));
  cudaSetDevice(prev);
  if (r != cudaSuccess) {
    ingest_free(&d->e);
    delete d;
    return fail(r == cudaErrorMemoryAllocation ? LTL4C_E_OOM : LTL4C_E_CUDA,
                std::string("ltl4c_dencoder_create: ") + cudaGetErrorString(r));
  }
  *out = d;
  return LTL4C_OK;
}

void ltl4c_dencoder_free(ltl4c_dencoder *d) {
  if (!d) return;
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(d->e.device);
  ingest_free(&d->e);
  cudaSetDevice(prev);
  delete d;
}

ltl4c_status ltl4c_dencode_jsonl(ltl4c_dencoder *d, const char *text, uint64_t len, uint32_t *const *keys,
                                 uint8_t *letters, uint64_t capacity, uint64_t *n_events, void *cuda_stream) {
  if (!d || !n_events || (len && !text)) return fail(LTL4C_E_INVALID, "null argument");
  if (capacity && (!keys || !letters)) return fail(LTL4C_E_INVALID, "null output buffer");
  for (uint32_t l = 0; l < d->e.prog->n_levels && capacity; ++l)
    if (!keys[l]) return fail(LTL4C_E_INVALID, "null key buffer");
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(d->e.device);
  unsigned long long n = 0, err = 0, ovf = 0, lines = 0;
  const cudaError_t r = ingest_run(&d->e, text, len, keys, letters, capacity, (cudaStream_t)cuda_stream, &n, &err,
                                   &ovf, &lines);
  cudaSetDevice(prev);
  *n_events = n;
  if (r != cudaSuccess)
    return fail(r == cudaErrorMemoryAllocation ? LTL4C_E_OOM : LTL4C_E_CUDA,
                std::string("ltl4c_dencode_jsonl: ") + cudaGetErrorString(r));
  if (err) return fail(LTL4C_E_SYNTAX, "line " + std::to_string(err) + ": malformed record");
  if (ovf) return fail(LTL4C_E_BUDGET, "more distinct values than the dictionary capacity");
  if (n > capacity) return fail(LTL4C_E_INVALID, std::to_string(n) + " records exceed the capacity");
  return LTL4C_OK;
}

ltl4c_status ltl4c_dencoder_values(const ltl4c_dencoder *d, uint32_t level, uint64_t *count) {
  if (!d || !count) return fail(LTL4C_E_INVALID, "null argument");
  if (level >= d->e.prog->n_levels) return fail(LTL4C_E_INVALID, "level out of range");
  uint32_t c = 0;
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(d->e.device);
  const cudaError_t r = cudaMemcpy(&c, d->e.base.dict_count + level, sizeof c, cudaMemcpyDeviceToHost);
  cudaSetDevice(prev);
  if (r != cudaSuccess) return fail(LTL4C_E_CUDA, cudaGetErrorString(r));
  *count = c;
  return LTL4C_OK;
}

}  // extern "C"
