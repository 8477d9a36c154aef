// K4 (top-k merge), K3 (gather-rerank with dedup) and K5 (row normalisation + bf16 cast).
//
// K4 is the device-side counterpart of the point where Teola joins pipelined search stages
// (reference: pkg/src/teola_sim/optimizer.py:620-661 `_insert_aggregates`; executed
// instantly on the orchestrator at pkg/src/teola_sim/runtime.py:544-549) and of the
// cross-shard merge after the all-gather in sharded mode.
// K3 executes a Reranking primitive (reference: optimizer.py:199-218 decomposition; executed by
// runtime.py:653-655 from the `rerank0` table, profiles/default.json:71-94).
//
// Ordering everywhere: (score desc, id asc); padding entries are (-inf, -1).
#include "tsv_kernels.cuh"

#include <cuda_bf16.h>
#include <algorithm>
#include <cfloat>
#include <cstdlib>

namespace tsv {
namespace {

// 64-bit sort key: high word = order-preserving image of the fp32 score, low word = bitwise
// complement of the id so that smaller ids sort first among equal scores when the keys are
// sorted descending. Padding (id == -1) maps to low word 0, i.e. last among equal scores.
__device__ __forceinline__ uint64_t make_key(float s, int32_t id) {
  uint32_t u = __float_as_uint(s);
  u = (u & 0x80000000u) ? ~u : (u | 0x80000000u);
  return (static_cast<uint64_t>(u) << 32) | static_cast<uint32_t>(~static_cast<uint32_t>(id));
}
__device__ __forceinline__ float key_score(uint64_t k) {
  uint32_t u = static_cast<uint32_t>(k >> 32);
  u = (u & 0x80000000u) ? (u & 0x7FFFFFFFu) : ~u;
  return __uint_as_float(u);
}
__device__ __forceinline__ int32_t key_id(uint64_t k) {
  return static_cast<int32_t>(~static_cast<uint32_t>(k & 0xFFFFFFFFu));
}
__device__ __forceinline__ uint64_t pad_key() { return make_key(-INFINITY, -1); }

// In-place descending bitonic sort of n (power of two) keys in shared memory.
__device__ void bitonic_sort_desc(uint64_t* keys, int n) {
  for (int size = 2; size <= n; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      __syncthreads();
      for (int i = threadIdx.x; i < (n >> 1); i += blockDim.x) {
        const int lo = 2 * i - (i & (stride - 1));
        const int hi = lo + stride;
        const bool desc = ((lo & size) == 0);
        const uint64_t a = keys[lo], b = keys[hi];
        if ((a < b) == desc) {
          keys[lo] = b;
          keys[hi] = a;
        }
      }
    }
  }
  __syncthreads();
}

// Register-resident bitonic stages: a warp holds a 64-key chunk as a (index lane) and b (index
// lane + 32); strides below 32 exchange through shuffles, stride 32 is in-lane.
__device__ __forceinline__ void cas_shfl(uint64_t& v, int lane, int s, bool desc) {
  const uint64_t o = __shfl_xor_sync(0xffffffffu, v, s);
  const bool take_max = ((lane & s) == 0) == desc;
  v = take_max ? (v > o ? v : o) : (v < o ? v : o);
}
// All stages of merge size `size` with stride <= 32, on the chunk starting at index g0.
__device__ __forceinline__ void chunk_stages(uint64_t& a, uint64_t& b, int g0, int lane, int size) {
  const bool da = ((g0 + lane) & size) == 0;
  const bool db = ((g0 + lane + 32) & size) == 0;
  if (size >= 64) {
    const uint64_t hi = a > b ? a : b, lo = a > b ? b : a;
    a = da ? hi : lo;
    b = da ? lo : hi;
  }
  for (int st = min(size >> 1, 16); st > 0; st >>= 1) {
    cas_shfl(a, lane, st, da);
    cas_shfl(b, lane, st, db);
  }
}

// Descending bitonic sort of n (power of two) keys in shared memory with the short-stride
// stages in registers: 2 + log2(n / 64) block barriers per merge size instead of log2(size).
__device__ void bitonic_sort_desc_fast(uint64_t* keys, int n) {
  if (n < 64) {
    bitonic_sort_desc(keys, n);
    return;
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  __syncthreads();
  for (int c = warp; c < (n >> 6); c += nw) {
    uint64_t a = keys[c * 64 + lane], b = keys[c * 64 + 32 + lane];
    for (int size = 2; size <= 64; size <<= 1) chunk_stages(a, b, c * 64, lane, size);
    keys[c * 64 + lane] = a;
    keys[c * 64 + 32 + lane] = b;
  }
  for (int size = 128; size <= n; size <<= 1) {
    for (int stride = size >> 1; stride >= 64; stride >>= 1) {
      __syncthreads();
      for (int i = threadIdx.x; i < (n >> 1); i += blockDim.x) {
        const int lo = 2 * i - (i & (stride - 1));
        const int hi = lo + stride;
        const bool desc = ((lo & size) == 0);
        const uint64_t x = keys[lo], y = keys[hi];
        if ((x < y) == desc) {
          keys[lo] = y;
          keys[hi] = x;
        }
      }
    }
    __syncthreads();
    for (int c = warp; c < (n >> 6); c += nw) {
      uint64_t a = keys[c * 64 + lane], b = keys[c * 64 + 32 + lane];
      chunk_stages(a, b, c * 64, lane, size);
      keys[c * 64 + lane] = a;
      keys[c * 64 + 32 + lane] = b;
    }
  }
  __syncthreads();
}

// Warp-wide maximum of a 64-bit key in two redux.sync steps: the largest high word, then the
// largest low word among the lanes holding it (a lane without it offers 0, the low word of
// padding, which never beats a real key's). Five u64 shuffle + compare steps before.
__device__ __forceinline__ uint64_t warp_max_key(uint64_t v) {
  const uint32_t hi = static_cast<uint32_t>(v >> 32), lo = static_cast<uint32_t>(v);
  const uint32_t mh = __reduce_max_sync(0xffffffffu, hi);
  const uint32_t ml = __reduce_max_sync(0xffffffffu, hi == mh ? lo : 0u);
  return (static_cast<uint64_t>(mh) << 32) | ml;
}

// The k best of keys[0, n) with duplicates dropped, by ONE warp, written to out_s / out_id
// (padded with -inf / -1): lane l holds keys l + 32 i in registers, sorted descending once
// (odd-even transposition network), so its best key is always r[0]; each round takes the warp
// maximum of the heads (warp_max_key) and every lane whose head equals it pops it (a shift,
// no compares on the round's critical path). Duplicate candidate ids carry identical keys
// (same row, same arithmetic) and sit together at a lane's head, so popping equal heads is
// the dedup. Replaces a block-wide bitonic sort + serial scan (2.3 + 0.8 us at C = 200) for
// n <= 32 KPL. A round costs ~0.13 us (k = 10 vs k = 1: +1.2 us at C = 16 or 200); a one-redux
// fast path for rounds whose best score sits on one lane, and results kept in registers with a
// predicated pop, measured the same or slower.
template <int KPL>
__device__ void warp_select_dedup(const uint64_t* keys, int n, int k, float* out_s,
                                  int32_t* out_id) {
  const int lane = threadIdx.x & 31;
  const uint64_t pad = pad_key();
  uint64_t r[KPL];
#pragma unroll
  for (int i = 0; i < KPL; ++i) {
    const int c = lane + 32 * i;
    r[i] = c < n ? keys[c] : pad;
  }
#pragma unroll
  for (int p = 0; p < KPL; ++p) {
#pragma unroll
    for (int i = p & 1; i + 1 < KPL; i += 2) {
      const uint64_t a = r[i], b = r[i + 1];
      r[i] = a > b ? a : b;
      r[i + 1] = a > b ? b : a;
    }
  }
  int w = 0;
  for (; w < k; ++w) {
    const uint64_t m = warp_max_key(r[0]);
    if (key_id(m) < 0) break;  // only padding / invalid candidates left
    if (lane == 0) {
      out_s[w] = key_score(m);
      out_id[w] = key_id(m);
    }
    while (r[0] == m) {  // this lane's copies of m (at most a few; usually none)
#pragma unroll
      for (int i = 0; i + 1 < KPL; ++i) r[i] = r[i + 1];
      r[KPL - 1] = pad;
    }
  }
  for (int j = w + lane; j < k; j += 32) {
    out_s[j] = -INFINITY;
    out_id[j] = -1;
  }
}

// The same selection without k serial rounds, for 16 <= k <= 32: the KPL columns (key l + 32 i
// in lane l) are each bitonic-sorted across the warp (descending), then merged pairwise keeping
// the top 32 (max of a column and its partner reversed is bitonic; five more stages sort it),
// so lane l ends with the l-th largest key of all n. Duplicates are adjacent there: a lane
// keeps its key when it differs from lane l-1's, and a ballot gives each kept key its output
// position. Returns false (nothing written) when the 32 largest hold fewer than k distinct
// keys while more valid keys exist below them; the caller then runs warp_select_dedup.
// Below k = 16 the k serial rounds are cheaper (C3's k = 10: 17.6 vs 18.1 us with the network;
// k = 20: 19.1 vs 18.2, k = 32 at 148 x 200: 16.3 vs 13.8; profiles/r02/rerank_probe_topk_net.txt).
constexpr int kNetMinK = 16;
__device__ __forceinline__ uint64_t u64_max(uint64_t a, uint64_t b) { return a > b ? a : b; }
__device__ __forceinline__ uint64_t u64_min(uint64_t a, uint64_t b) { return a > b ? b : a; }

template <int N>
__device__ __forceinline__ void warp_bitonic_stages_desc(uint64_t (&v)[N], int lane, int size) {
  // the merge stages of one bitonic level: blocks of `size` lanes, descending where
  // (lane & size) == 0 (size = 64: the whole warp descending)
  const bool desc = (lane & size) == 0;
#pragma unroll
  for (int stride = 16; stride > 0; stride >>= 1) {
    if (stride >= size) continue;
    const bool keep_max = ((lane & stride) == 0) == desc;
#pragma unroll
    for (int i = 0; i < N; ++i) {
      const uint64_t o = __shfl_xor_sync(0xffffffffu, v[i], stride);
      v[i] = keep_max ? u64_max(v[i], o) : u64_min(v[i], o);
    }
  }
}

template <int KPL>
__device__ bool warp_topk_net(const uint64_t* keys, int n, int k, float* out_s, int32_t* out_id) {
  const int lane = threadIdx.x & 31;
  const uint64_t pad = pad_key();
  uint64_t r[KPL];
#pragma unroll
  for (int i = 0; i < KPL; ++i) {
    const int c = lane + 32 * i;
    r[i] = c < n ? keys[c] : pad;
  }
#pragma unroll
  for (int size = 2; size <= 32; size <<= 1) warp_bitonic_stages_desc<KPL>(r, lane, size == 32 ? 64 : size);
#pragma unroll
  for (int w = KPL / 2; w >= 1; w >>= 1) {
#pragma unroll
    for (int i = 0; i < w; ++i) r[i] = u64_max(r[i], __shfl_sync(0xffffffffu, r[i + w], 31 - lane));
#pragma unroll
    for (int stride = 16; stride > 0; stride >>= 1) {
      const bool keep_max = (lane & stride) == 0;
#pragma unroll
      for (int i = 0; i < w; ++i) {
        const uint64_t o = __shfl_xor_sync(0xffffffffu, r[i], stride);
        r[i] = keep_max ? u64_max(r[i], o) : u64_min(r[i], o);
      }
    }
  }
  const uint64_t v = r[0];
  const uint64_t prev = __shfl_up_sync(0xffffffffu, v, 1);
  const bool keep = key_id(v) >= 0 && (lane == 0 || v != prev);
  const uint32_t mask = __ballot_sync(0xffffffffu, keep);
  const int distinct = __popc(mask);
  const bool more_below = key_id(__shfl_sync(0xffffffffu, v, 31)) >= 0 && n > 32;
  if (distinct < k && more_below) return false;
  const int pos = __popc(mask & ((1u << lane) - 1u));
  if (keep && pos < k) {
    out_s[pos] = key_score(v);
    out_id[pos] = key_id(v);
  }
  for (int j = distinct + lane; j < k; j += 32) {
    out_s[j] = -INFINITY;
    out_id[j] = -1;
  }
  return true;
}

__device__ __forceinline__ int pow2_ceil(int n) {
  int p = 1;
  while (p < n) p <<= 1;
  return p;
}

// Copy the `need` largest of keys[0, m) into sel (capacity cap >= need) in any order, with an
// MSB-first 8-bit radix select: each pass histograms the digit below the fixed prefix and
// keeps the bin that holds the need-th largest key; it stops once that bin is taken whole.
// Returns the number of keys written. Keys are unique except for exact duplicates, which are
// interchangeable.
__device__ int radix_select_top(const uint64_t* keys, int m, int need, uint64_t* sel, int cap) {
  __shared__ int hist[256];
  __shared__ int sel_d, sel_above, sel_cnt, nsel;
  uint64_t prefix = 0, pmask = 0;
  for (int shift = 56; shift >= 0; shift -= 8) {
    for (int i = threadIdx.x; i < 256; i += blockDim.x) hist[i] = 0;
    __syncthreads();
    for (int i = threadIdx.x; i < m; i += blockDim.x) {
      const uint64_t k = keys[i];
      if ((k & pmask) == prefix) atomicAdd(&hist[(k >> shift) & 255], 1);
    }
    __syncthreads();
    if (threadIdx.x < 32) {  // digit holding the need-th largest (bins scanned high to low)
      const int lane = threadIdx.x;
      int c[8], tot = 0;
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        c[t] = hist[255 - (lane * 8 + t)];
        tot += c[t];
      }
      int incl = tot;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, incl, off);
        if (lane >= off) incl += v;
      }
      const int excl = incl - tot;
      if (excl < need && need <= incl) {
        int run = excl;
#pragma unroll
        for (int t = 0; t < 8; ++t) {
          if (run + c[t] >= need) {
            sel_d = 255 - (lane * 8 + t);
            sel_above = run;
            sel_cnt = c[t];
            break;
          }
          run += c[t];
        }
      }
    }
    __syncthreads();
    need -= sel_above;
    prefix |= static_cast<uint64_t>(sel_d) << shift;
    pmask |= 255ull << shift;
    const bool whole = sel_cnt == need;
    __syncthreads();  // sel_* are rewritten by the next pass
    if (whole) break;
  }
  if (threadIdx.x == 0) nsel = 0;
  __syncthreads();
  for (int i = threadIdx.x; i < m; i += blockDim.x) {  // strictly above the prefix: all in
    const uint64_t k = keys[i];
    if ((k & pmask) > prefix) sel[atomicAdd(&nsel, 1)] = k;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < m; i += blockDim.x) {  // on the prefix: as many as fit
    const uint64_t k = keys[i];
    if ((k & pmask) == prefix) {
      const int slot = atomicAdd(&nsel, 1);
      if (slot < cap) sel[slot] = k;
    }
  }
  __syncthreads();
  return nsel < cap ? nsel : cap;
}

// The kout best of the m keys in keys[0, m) (any order), written sorted (score desc, id asc)
// with (-inf, -1) padding to os / oi. keys has room for n_alloc >= pow2_ceil(m) keys plus
// pow2_ceil(kout) selection slots behind them. Block-wide.
__device__ void write_topk_of_keys(uint64_t* keys, int m, int n_alloc, int kout,
                                   float* __restrict__ os, int32_t* __restrict__ oi) {
  const int kp = pow2_ceil(kout);
  if (m > 2 * kp && m > 256) {
    // Many more candidates than outputs: radix-select the kout best keys, sort only those.
    uint64_t* sel = keys + n_alloc;
    const int got = radix_select_top(keys, m, kout, sel, kp);
    for (int i = got + threadIdx.x; i < kp; i += blockDim.x) sel[i] = pad_key();
    bitonic_sort_desc_fast(sel, kp);
    for (int j = threadIdx.x; j < kout; j += blockDim.x) {
      const uint64_t key = sel[j];
      const int32_t id = key_id(key);
      os[j] = id < 0 ? -INFINITY : key_score(key);
      oi[j] = id;
    }
    return;
  }
  const int np = pow2_ceil(m > 0 ? m : 1);
  for (int i = m + threadIdx.x; i < np; i += blockDim.x) keys[i] = pad_key();
  bitonic_sort_desc_fast(keys, np);
  for (int j = threadIdx.x; j < kout; j += blockDim.x) {
    const uint64_t key = j < np ? keys[j] : pad_key();
    const int32_t id = key_id(key);
    os[j] = id < 0 ? -INFINITY : key_score(key);
    oi[j] = id;
  }
}

// One block per query: gather lists * kin candidates, sort, keep kout.
__global__ void merge_topk_kernel(const float* __restrict__ in_s, const int32_t* __restrict__ in_id,
                                  int lists, int B, int kin, int64_t list_stride_rows, int kout,
                                  float* __restrict__ out_s, int32_t* __restrict__ out_id,
                                  int dedup, const int32_t* __restrict__ gate) {
  extern __shared__ uint64_t keys[];
  __shared__ int count;
  pdl_wait();
  if (gate != nullptr && *gate == 0) return;
  const int b = blockIdx.x;
  const int n = lists * kin;
  // Compact the real entries first: seeded / floored scans leave most partial lists mostly
  // padding, and the sort cost follows the compacted size (the key order makes the result
  // independent of the compaction order).
  if (threadIdx.x == 0) count = 0;
  __syncthreads();
  // eight independent loads in flight per thread (the lists are L2-resident, latency-bound)
  constexpr int kBatch = 8;
  for (int base = 0; base < n; base += kBatch * blockDim.x) {
    int32_t id[kBatch];
    float sc[kBatch];
#pragma unroll
    for (int u = 0; u < kBatch; ++u) {
      const int i = base + u * blockDim.x + threadIdx.x;
      id[u] = -1;
      if (i < n) {
        const int r = i / kin;
        const int64_t off = (static_cast<int64_t>(r) * list_stride_rows + b) * kin + (i - r * kin);
        id[u] = __ldg(in_id + off);
        sc[u] = __ldg(in_s + off);
      }
    }
#pragma unroll
    for (int u = 0; u < kBatch; ++u)
      if (id[u] >= 0) keys[atomicAdd(&count, 1)] = make_key(sc[u], id[u]);
  }
  __syncthreads();
  const int m = count;
  if (!dedup) {
    write_topk_of_keys(keys, m, pow2_ceil(n), kout, out_s + static_cast<int64_t>(b) * kout,
                       out_id + static_cast<int64_t>(b) * kout);
    return;
  }
  const int np = pow2_ceil(m > 0 ? m : 1);
  for (int i = m + threadIdx.x; i < np; i += blockDim.x) keys[i] = pad_key();
  bitonic_sort_desc_fast(keys, np);
  // Copies of one id carry identical scores, so they are adjacent after the sort.
  if (threadIdx.x == 0) {
    int w = 0;
    int32_t last = -2;
    for (int i = 0; i < np && w < kout; ++i) {
      const int32_t id = key_id(keys[i]);
      if (id < 0) break;
      if (id == last) continue;
      last = id;
      out_s[static_cast<int64_t>(b) * kout + w] = key_score(keys[i]);
      out_id[static_cast<int64_t>(b) * kout + w] = id;
      ++w;
    }
    for (; w < kout; ++w) {
      out_s[static_cast<int64_t>(b) * kout + w] = -INFINITY;
      out_id[static_cast<int64_t>(b) * kout + w] = -1;
    }
  }
}

// Candidate select (append mode, k > 32): one block per query; the query's candidate row holds
// every corpus row that scored above its seeded floor, in arrival order. Exact top-k of those
// (the floor is a lower bound of the final k-th score, so they include the whole result), or,
// when the row overflowed, nothing but the overflow flag that gates the fallback pass.
__global__ void cand_select_kernel(const float* __restrict__ buf_s, const int32_t* __restrict__ buf_i,
                                   const int32_t* __restrict__ cnt, int cap, int kout,
                                   float* __restrict__ out_s, int32_t* __restrict__ out_id,
                                   int32_t* __restrict__ overflow) {
  extern __shared__ uint64_t keys[];
  pdl_wait();
  const int b = blockIdx.x;
  const int m = cnt[b];
  if (m > cap) {
    if (threadIdx.x == 0) atomicExch(overflow, 1);
    return;
  }
  const int64_t row = static_cast<int64_t>(b) * cap;
  for (int i = threadIdx.x; i < m; i += blockDim.x)
    keys[i] = make_key(__ldg(buf_s + row + i), __ldg(buf_i + row + i));
  __syncthreads();
  write_topk_of_keys(keys, m, pow2_ceil(cap), kout, out_s + static_cast<int64_t>(b) * kout,
                     out_id + static_cast<int64_t>(b) * kout);
}

// One block per question: score C candidate rows (gathered by id from the arena) against the
// question vector, drop duplicate ids, keep the best k.
template <int kThreads, int kPer, int kUnroll>
__global__ void __launch_bounds__(kThreads) rerank_kernel(
    const __nv_bfloat16* __restrict__ arena, const float* __restrict__ arena_hi,
    const float* __restrict__ arena_lo, int64_t nrows, int dim, const void* __restrict__ q,
    const float* __restrict__ q_lo, int q_is_f32, const int32_t* __restrict__ cand, int C, int k,
    float* __restrict__ out_s, int32_t* __restrict__ out_id, int tiled,
    const int32_t* __restrict__ offs) {
  extern __shared__ uint8_t sm[];
  float* qv = reinterpret_cast<float*>(sm);                       // dim floats
  uint64_t* keys = reinterpret_cast<uint64_t*>(sm + ((dim * 4 + 15) & ~15));
  const int np = pow2_ceil(C);
  int32_t* ids = reinterpret_cast<int32_t*>(keys + np);           // C candidate ids
  const int b = blockIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int kWarps = kThreads / 32;

  // the question vector and the candidate ids are staged once, so the gather loop below waits
  // on one memory round trip per batch of rows instead of two
  const int64_t base = offs != nullptr ? __ldg(offs + b) : 0;  // per-question segment start
  for (int c = threadIdx.x; c < C; c += kThreads) ids[c] = __ldg(cand + static_cast<int64_t>(b) * C + c);
  for (int d = threadIdx.x; d < dim; d += kThreads) {
    const int64_t o = static_cast<int64_t>(b) * dim + d;
    qv[d] = q_is_f32 ? reinterpret_cast<const float*>(q)[o] + (q_lo ? q_lo[o] : 0.f)
                     : __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(q)[o]);
  }
  for (int i = threadIdx.x; i < np; i += kThreads) keys[i] = pad_key();
  __syncthreads();

  const int chunks = dim >> 3;  // 8 bf16 (16 B) per chunk; dim % 8 == 0 enforced by the host
  const int64_t kb_per_row = (dim + 63) >> 6;
  // kPer candidates per warp iteration with independent loads and accumulators: the gather is
  // latency-bound (one row is only 1.5-2 KB), so every lane keeps kPer rows' chunks in flight.
  for (int c0 = kPer * warp; c0 < C; c0 += kPer * kWarps) {
    int32_t id[kPer];
    bool ok[kPer];
    float acc[kPer];
#pragma unroll
    for (int u = 0; u < kPer; ++u) {
      id[u] = c0 + u < C ? ids[c0 + u] : -1;
      ok[u] = id[u] >= 0 && base + id[u] < nrows;  // warp-uniform
      acc[u] = 0.f;
    }
    if (arena_hi != nullptr) {  // fp32 storage: row = hi + lo, fp32 FMA
#pragma unroll
      for (int u = 0; u < kPer; ++u) {
        if (!ok[u]) continue;
        const float4* hi = reinterpret_cast<const float4*>(arena_hi + (base + id[u]) * dim);
        const float4* lo = reinterpret_cast<const float4*>(arena_lo + (base + id[u]) * dim);
        for (int ch = lane; ch < (dim >> 2); ch += 32) {
          const float4 h = __ldg(hi + ch), l = __ldg(lo + ch);
          const float* qq = qv + ch * 4;
          acc[u] = fmaf(h.x + l.x, qq[0], acc[u]);
          acc[u] = fmaf(h.y + l.y, qq[1], acc[u]);
          acc[u] = fmaf(h.z + l.z, qq[2], acc[u]);
          acc[u] = fmaf(h.w + l.w, qq[3], acc[u]);
        }
      }
    } else {
      const uint4* row[kPer];
#pragma unroll
      for (int u = 0; u < kPer; ++u) {
        const int64_t r = ok[u] ? base + id[u] : 0;
        // tiled layout: 16-byte chunk ch of row r lives in k-block tile (r/128, ch/8)
        row[u] = tiled ? reinterpret_cast<const uint4*>(
                             arena + ((r >> 7) * kb_per_row * 128 + (r & 127)) * 64)
                       : reinterpret_cast<const uint4*>(arena + r * dim);
      }
#pragma unroll kUnroll
      for (int ch = lane; ch < chunks; ch += 32) {
        const int64_t off = tiled ? static_cast<int64_t>(ch >> 3) * 1024 + (ch & 7) : ch;
        uint4 raw[kPer];
#pragma unroll
        for (int u = 0; u < kPer; ++u) raw[u] = ok[u] ? __ldg(row[u] + off) : make_uint4(0, 0, 0, 0);
        const float* qq = qv + ch * 8;
#pragma unroll
        for (int u = 0; u < kPer; ++u) {
          const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&raw[u]);
#pragma unroll
          for (int t = 0; t < 4; ++t) {
            const float2 f = __bfloat1622float2(h[t]);
            acc[u] = fmaf(f.x, qq[2 * t], acc[u]);
            acc[u] = fmaf(f.y, qq[2 * t + 1], acc[u]);
          }
        }
      }
    }
#pragma unroll
    for (int u = 0; u < kPer; ++u) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) acc[u] += __shfl_xor_sync(0xffffffffu, acc[u], o);
      if (lane == 0 && ok[u]) keys[c0 + u] = make_key(acc[u], id[u]);
    }
  }
  bitonic_sort_desc_fast(keys, np);
  // Dedup: duplicates of one id carry identical scores, so they are adjacent after the sort.
  if (threadIdx.x == 0) {
    int w = 0;
    int32_t last = -2;
    for (int i = 0; i < np && w < k; ++i) {
      const int32_t id = key_id(keys[i]);
      if (id < 0) break;
      if (id == last) continue;
      last = id;
      out_s[static_cast<int64_t>(b) * k + w] = key_score(keys[i]);
      out_id[static_cast<int64_t>(b) * k + w] = id;
      ++w;
    }
    for (; w < k; ++w) {
      out_s[static_cast<int64_t>(b) * k + w] = -INFINITY;
      out_id[static_cast<int64_t>(b) * k + w] = -1;
    }
  }
}

// K3, bf16 arenas: the same computation as rerank_kernel with the gather pipelined through
// shared memory. Each warp owns a ring of `slots` row buffers and walks its candidates
// (c = warp, warp + kWarps, ...): it keeps `slots` rows in flight with cp.async (16-byte
// LDGSTS per lane, no registers held) and scores the oldest as soon as it lands, then refills
// that slot. A warp therefore never idles between a round trip and the next: the memory
// system sees ~slots rows per warp continuously instead of bursts of 2 rows per round trip
// (the register-gather kernel's 5 dependent rounds for C = 200).
__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gmem_src) {
  const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(smem_dst));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(gmem_src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// (a, b) -> bf16x2 word (a in the low half), round to nearest even
__device__ __forceinline__ uint32_t pack_bf16x2(float a, float b) {
  const __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<const uint32_t*>(&h);
}

// bf16x2 word -> (element 2t, element 2t+1) as fp32: a bf16 is the high half of an fp32
__device__ __forceinline__ float2 bf16x2_to_float2(uint32_t w) {
  return make_float2(__uint_as_float(w << 16), __uint_as_float(w & 0xFFFF0000u));
}

// Lane `lane` always owns chunks lane + 32 j (j < CPL) of every row, so the question's matching
// elements live in its registers for the whole kernel and a row chunk costs one shared-memory
// load, four bf16x2 -> fp32x2 conversions and four packed fp32x2 FMAs (FFMA2; even / odd
// elements in the two halves, summed at the end).
template <int kWarps, int kSlots, int CPL, bool kTiled>
__global__ void __launch_bounds__(kWarps * 32) rerank_ring_kernel(
    const __nv_bfloat16* __restrict__ arena, int64_t nrows, int dim, const void* __restrict__ q,
    int q_is_f32, const int32_t* __restrict__ cand, int C, int k, const int32_t* __restrict__ offs,
    float* __restrict__ out_s, int32_t* __restrict__ out_id, int use_sort) {
  extern __shared__ __align__(16) uint8_t sm[];
  // once every block has passed here the next launch on the stream may be scheduled (its blocks
  // take free SM slots and wait for this grid's completion in their own griddepcontrol.wait)
  if (threadIdx.x == 0) pdl_allow_dependents();
  pdl_wait();  // (programmatic launch: the question and the candidates are the previous kernels')
  const int row_bytes = dim * 2;
  uint8_t* ring = sm;                                                   // [kWarps][kSlots][row]
  uint64_t* keys = reinterpret_cast<uint64_t*>(sm + static_cast<size_t>(kWarps) * kSlots * row_bytes);
  const int np = pow2_ceil(C);
  int32_t* ids = reinterpret_cast<int32_t*>(keys + np);                 // segment-local ids
  const int b = blockIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int chunks = dim >> 3;  // 16-byte chunks per row
  // The question's elements of this lane's chunks go to registers first: their round trip
  // overlaps the candidate ids' (nothing below waits for them until the first row is scored).
  float2 qr[CPL][4];
#pragma unroll
  for (int j = 0; j < CPL; ++j) {
    const int ch = lane + 32 * j;
#pragma unroll
    for (int t = 0; t < 4; ++t) qr[j][t] = make_float2(0.f, 0.f);
    if (ch < chunks) {
      const int64_t o = static_cast<int64_t>(b) * dim + ch * 8;
      if (q_is_f32) {
        const float4 x0 = __ldg(reinterpret_cast<const float4*>(reinterpret_cast<const float*>(q) + o));
        const float4 x1 = __ldg(reinterpret_cast<const float4*>(reinterpret_cast<const float*>(q) + o + 4));
        qr[j][0] = make_float2(x0.x, x0.y);
        qr[j][1] = make_float2(x0.z, x0.w);
        qr[j][2] = make_float2(x1.x, x1.y);
        qr[j][3] = make_float2(x1.z, x1.w);
      } else {
        const uint4 w = __ldg(reinterpret_cast<const uint4*>(reinterpret_cast<const __nv_bfloat16*>(q) + o));
        qr[j][0] = bf16x2_to_float2(w.x);
        qr[j][1] = bf16x2_to_float2(w.y);
        qr[j][2] = bf16x2_to_float2(w.z);
        qr[j][3] = bf16x2_to_float2(w.w);
      }
    }
  }
  const int64_t base = offs != nullptr ? __ldg(offs + b) : 0;  // per-question segment start
  // Each warp stages only its own candidates' ids (c = warp + kWarps i): no block barrier
  // before the gather starts. The keys' padding tail is ordered before the sort by its barrier.
  for (int c = warp + kWarps * lane; c < C; c += kWarps * 32)
    ids[c] = __ldg(cand + static_cast<int64_t>(b) * C + c);
  for (int i = C + threadIdx.x; i < np; i += kWarps * 32) keys[i] = pad_key();
  __syncwarp();

  const int64_t kb_per_row = (dim + 63) >> 6;
  uint8_t* my_ring = ring + static_cast<size_t>(warp) * kSlots * row_bytes;
  auto valid = [&](int c) {
    if (c >= C) return false;
    const int32_t id = ids[c];
    return id >= 0 && base + id < nrows;
  };
  auto issue = [&](int c, int slot) {  // whole warp; always commits one group
    if (valid(c)) {
      const int64_t r = base + ids[c];
      const uint4* src = kTiled ? reinterpret_cast<const uint4*>(
                                      arena + ((r >> 7) * kb_per_row * 128 + (r & 127)) * 64)
                                : reinterpret_cast<const uint4*>(arena + r * dim);
      uint4* dst = reinterpret_cast<uint4*>(my_ring + static_cast<size_t>(slot) * row_bytes);
#pragma unroll
      for (int j = 0; j < CPL; ++j) {
        const int ch = lane + 32 * j;
        if (ch < chunks)
          cp_async16(dst + ch, src + (kTiled ? static_cast<int64_t>(ch >> 3) * 1024 + (ch & 7) : ch));
      }
    }
    cp_async_commit();
  };
#pragma unroll
  for (int s = 0; s < kSlots; ++s) issue(warp + s * kWarps, s);
  // R rows per step: with 4 slots a warp scores two landed rows at once (two independent FFMA2 /
  // butterfly chains interleaved, each row's operation order unchanged, so the scores are
  // bit-identical) while the other two are in flight.
  constexpr int R = kSlots == 4 ? 2 : 1;
  int slot = 0;
  for (int c = warp; c < C; c += R * kWarps) {
    cp_async_wait<kSlots - R>();  // the oldest R groups (candidates c, c + kWarps) have landed
    __syncwarp();
    float2 a2[R];
#pragma unroll
    for (int r = 0; r < R; ++r) a2[r] = make_float2(0.f, 0.f);
#pragma unroll
    for (int j = 0; j < CPL; ++j) {
      const int ch = lane + 32 * j;
      if (ch < chunks) {
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const uint4 raw = reinterpret_cast<const uint4*>(
              my_ring + static_cast<size_t>(slot + r) * row_bytes)[ch];
          a2[r] = __ffma2_rn(bf16x2_to_float2(raw.x), qr[j][0], a2[r]);
          a2[r] = __ffma2_rn(bf16x2_to_float2(raw.y), qr[j][1], a2[r]);
          a2[r] = __ffma2_rn(bf16x2_to_float2(raw.z), qr[j][2], a2[r]);
          a2[r] = __ffma2_rn(bf16x2_to_float2(raw.w), qr[j][3], a2[r]);
        }
      }
    }
    float acc[R];
#pragma unroll
    for (int r = 0; r < R; ++r) acc[r] = a2[r].x + a2[r].y;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
#pragma unroll
      for (int r = 0; r < R; ++r) acc[r] += __shfl_xor_sync(0xffffffffu, acc[r], o);
    }
    if (lane == 0) {
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int cr = c + r * kWarps;  // (a slot of an invalid candidate holds stale bytes)
        if (cr < C) keys[cr] = valid(cr) ? make_key(acc[r], ids[cr]) : pad_key();
      }
    }
    __syncwarp();  // every lane done reading the slots before they are refilled
#pragma unroll
    for (int r = 0; r < R; ++r) issue(c + r * kWarps + kSlots * kWarps, slot + r);
    slot += R;
    if (slot == kSlots) slot = 0;
  }
  cp_async_wait<0>();
  const bool net = !(use_sort & 2) && k >= kNetMinK && k <= 32;
  use_sort &= 1;
  if (C <= 256 && !use_sort) {  // one warp selects: no block-wide sort
    __syncthreads();
    if (warp == 0) {
      float* os = out_s + static_cast<int64_t>(b) * k;
      int32_t* oi = out_id + static_cast<int64_t>(b) * k;
      if (!(net && warp_topk_net<8>(keys, C, k, os, oi)))
        warp_select_dedup<8>(keys, C, k, os, oi);
    }
    return;
  }
  if (C <= 512 && !use_sort) {
    __syncthreads();
    if (warp == 0)
      warp_select_dedup<16>(keys, C, k, out_s + static_cast<int64_t>(b) * k,
                            out_id + static_cast<int64_t>(b) * k);
    return;
  }
  bitonic_sort_desc_fast(keys, np);
  // Dedup: duplicates of one id carry identical scores, so they are adjacent after the sort.
  if (threadIdx.x == 0) {
    int w = 0;
    int32_t last = INT32_MIN;
    for (int i = 0; i < np && w < k; ++i) {
      const int32_t id = key_id(keys[i]);
      if (id < 0) break;
      if (id == last) continue;
      last = id;
      out_s[static_cast<int64_t>(b) * k + w] = key_score(keys[i]);
      out_id[static_cast<int64_t>(b) * k + w] = id;
      ++w;
    }
    for (; w < k; ++w) {
      out_s[static_cast<int64_t>(b) * k + w] = -INFINITY;
      out_id[static_cast<int64_t>(b) * k + w] = -1;
    }
  }
}

// K3 for the common rerank shapes (C <= 32 * kWarps candidates, k <= 32): the gather and
// scoring of rerank_ring_kernel, with the per-row bookkeeping moved out of the loop and the
// block-wide sort replaced by per-warp top-k lists.
//  * each warp owns candidates c = warp + kWarps j (j < 32): lane j holds candidate j's id,
//    validity (one ballot) and row address, so a row's issue is two shuffles and CPL cp.async;
//  * after the butterfly reduction every lane holds the row's score; the warp keeps a sorted
//    top-k list in registers (lane r = rank r) and inserts with one ballot + one shuffle when
//    the key beats the list's k-th (a key already in the list is a duplicate candidate id:
//    same row, same score);
//  * warp 0 merges the kWarps lists with k rounds of a warp-wide max, dropping every copy of
//    the chosen key (duplicates across warps).
// k rounds of a warp-wide max over the keys in `mine` (pad-filled): round r yields the r-th key
// (score desc, id asc) and drops every copy of it (duplicate candidate ids). Lane 0 writes the
// result to out_key (as keys) or to out_s / out_id. Whole warp.
template <int kPer>
__device__ __forceinline__ void warp_topk_rounds(uint64_t (&mine)[kPer], int k, uint64_t* out_key,
                                                 float* out_s, int32_t* out_id) {
  const uint64_t pad = pad_key();
  const int lane = threadIdx.x & 31;
  for (int rk = 0; rk < k; ++rk) {
    uint64_t m = mine[0];
#pragma unroll
    for (int i = 1; i < kPer; ++i) m = mine[i] > m ? mine[i] : m;
    m = warp_max_key(m);
    if (lane == 0) {
      if (out_key != nullptr) {
        out_key[rk] = m;
      } else {
        const int32_t id = m == pad ? -1 : key_id(m);
        out_s[rk] = id < 0 ? -INFINITY : key_score(m);
        out_id[rk] = id;
      }
    }
#pragma unroll
    for (int i = 0; i < kPer; ++i)
      if (mine[i] == m) mine[i] = pad;
  }
}

// splits > 1: the candidates of question b are split over `splits` blocks (blockIdx.x =
// b * splits + s, candidates [C s / splits, C (s + 1) / splits)), so a batch of few questions
// or long candidate lists still fills the GPU with short per-warp chains; each block leaves its
// top k in part_keys, and the last block of the question to finish (arrivals[b], self-resetting)
// merges the splits' lists.
template <int kWarps, int kSlots, int CPL, bool kTiled>
__global__ void __launch_bounds__(kWarps * 32) rerank_lists_kernel(
    const __nv_bfloat16* __restrict__ arena, int64_t nrows, int dim, const void* __restrict__ q,
    int q_is_f32, const int32_t* __restrict__ cand, int C, int k, const int32_t* __restrict__ offs,
    float* __restrict__ out_s, int32_t* __restrict__ out_id, int splits,
    uint64_t* __restrict__ part_keys, int32_t* __restrict__ arrivals) {
  extern __shared__ __align__(16) uint8_t sm[];
  pdl_wait();  // (programmatic launch: the question and the candidates are the previous kernels')
  const int row_bytes = dim * 2;
  uint8_t* ring = sm;                                                   // [kWarps][kSlots][row]
  uint64_t* lists = reinterpret_cast<uint64_t*>(sm + static_cast<size_t>(kWarps) * kSlots * row_bytes);
  const int b = blockIdx.x / splits, split = blockIdx.x - b * splits;
  const int c_beg = static_cast<int>(static_cast<int64_t>(C) * split / splits);
  const int c_end = static_cast<int>(static_cast<int64_t>(C) * (split + 1) / splits);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int chunks = dim >> 3;
  float2 qr[CPL][4];
#pragma unroll
  for (int j = 0; j < CPL; ++j) {
    const int ch = lane + 32 * j;
#pragma unroll
    for (int t = 0; t < 4; ++t) qr[j][t] = make_float2(0.f, 0.f);
    if (ch < chunks) {
      const int64_t o = static_cast<int64_t>(b) * dim + ch * 8;
      if (q_is_f32) {
        const float4 x0 = __ldg(reinterpret_cast<const float4*>(reinterpret_cast<const float*>(q) + o));
        const float4 x1 = __ldg(reinterpret_cast<const float4*>(reinterpret_cast<const float*>(q) + o + 4));
        qr[j][0] = make_float2(x0.x, x0.y);
        qr[j][1] = make_float2(x0.z, x0.w);
        qr[j][2] = make_float2(x1.x, x1.y);
        qr[j][3] = make_float2(x1.z, x1.w);
      } else {
        const uint4 w = __ldg(reinterpret_cast<const uint4*>(reinterpret_cast<const __nv_bfloat16*>(q) + o));
        qr[j][0] = bf16x2_to_float2(w.x);
        qr[j][1] = bf16x2_to_float2(w.y);
        qr[j][2] = bf16x2_to_float2(w.z);
        qr[j][3] = bf16x2_to_float2(w.w);
      }
    }
  }
  const int64_t base = offs != nullptr ? __ldg(offs + b) : 0;  // per-question segment start
  const int cw = c_end - c_beg;  // this block's candidates
  const int nrow = warp < cw ? (cw - warp + kWarps - 1) / kWarps : 0;  // <= 32
  const int32_t my_id =
      lane < nrow ? __ldg(cand + static_cast<int64_t>(b) * C + c_beg + warp + kWarps * lane) : -1;
  const bool my_ok = my_id >= 0 && base + my_id < nrows;
  const uint32_t okmask = __ballot_sync(0xffffffffu, my_ok);
  const int64_t r = my_ok ? base + my_id : 0;
  const int64_t kb_per_row = (dim + 63) >> 6;
  const uint4* my_src = kTiled ? reinterpret_cast<const uint4*>(arena + ((r >> 7) * kb_per_row * 128 + (r & 127)) * 64)
                               : reinterpret_cast<const uint4*>(arena + r * dim);
  uint8_t* my_ring = ring + static_cast<size_t>(warp) * kSlots * row_bytes;
  auto issue = [&](int j, int slot) {  // whole warp; always commits one group
    const uint4* src = reinterpret_cast<const uint4*>(
        __shfl_sync(0xffffffffu, reinterpret_cast<uintptr_t>(my_src), j & 31));
    if (j < nrow && ((okmask >> j) & 1u)) {
      uint4* dst = reinterpret_cast<uint4*>(my_ring + static_cast<size_t>(slot) * row_bytes);
#pragma unroll
      for (int jj = 0; jj < CPL; ++jj) {
        const int ch = lane + 32 * jj;
        if (ch < chunks)
          cp_async16(dst + ch, src + (kTiled ? static_cast<int64_t>(ch >> 3) * 1024 + (ch & 7) : ch));
      }
    }
    cp_async_commit();
  };
#pragma unroll
  for (int s_ = 0; s_ < kSlots; ++s_) issue(s_, s_);
  uint64_t lk = pad_key();   // this warp's top-k list, rank = lane
  uint64_t thr = pad_key();  // its k-th key
  int slot = 0;
  for (int j = 0; j < nrow; ++j) {
    cp_async_wait<kSlots - 1>();  // the oldest group (row j) has landed
    __syncwarp();
    if ((okmask >> j) & 1u) {
      const uint4* row = reinterpret_cast<const uint4*>(my_ring + static_cast<size_t>(slot) * row_bytes);
      float2 a2 = make_float2(0.f, 0.f);
#pragma unroll
      for (int jj = 0; jj < CPL; ++jj) {
        const int ch = lane + 32 * jj;
        if (ch < chunks) {
          const uint4 raw = row[ch];
          a2 = __ffma2_rn(bf16x2_to_float2(raw.x), qr[jj][0], a2);
          a2 = __ffma2_rn(bf16x2_to_float2(raw.y), qr[jj][1], a2);
          a2 = __ffma2_rn(bf16x2_to_float2(raw.z), qr[jj][2], a2);
          a2 = __ffma2_rn(bf16x2_to_float2(raw.w), qr[jj][3], a2);
        }
      }
      float acc = a2.x + a2.y;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
      const uint64_t key = make_key(acc, __shfl_sync(0xffffffffu, my_id, j));
      if (key > thr && !__any_sync(0xffffffffu, lk == key)) {
        const int pos = __popc(__ballot_sync(0xffffffffu, lk > key));
        const uint64_t up = __shfl_up_sync(0xffffffffu, lk, 1);
        if (lane == pos) lk = key;
        else if (lane > pos) lk = up;
        thr = __shfl_sync(0xffffffffu, lk, k - 1);
      }
    }
    __syncwarp();  // every lane done reading the slot before it is refilled
    issue(j + kSlots, slot);
    if (++slot == kSlots) slot = 0;
  }
  cp_async_wait<0>();
  if (lane < k) lists[warp * k + lane] = lk;
  __syncthreads();
  if (warp != 0) return;
  constexpr int kPer = kWarps;  // kWarps * k <= kWarps * 32 keys, kWarps per lane
  uint64_t mine[kPer];
#pragma unroll
  for (int i = 0; i < kPer; ++i) {
    const int e = lane + 32 * i;
    mine[i] = e < kWarps * k ? lists[e] : pad_key();
  }
  if (splits == 1) {
    warp_topk_rounds<kPer>(mine, k, nullptr, out_s + static_cast<int64_t>(b) * k,
                           out_id + static_cast<int64_t>(b) * k);
    return;
  }
  warp_topk_rounds<kPer>(mine, k, part_keys + static_cast<int64_t>(blockIdx.x) * k, nullptr,
                         nullptr);
  // the last of the question's blocks merges the splits' lists (threadfence reduction)
  __shared__ int last;
  if (lane == 0) {
    __threadfence();
    last = atomicAdd(arrivals + b, 1) == splits - 1;
  }
  __syncwarp();
  if (!last) return;
  __threadfence();
  uint64_t all[8];  // splits * k <= 256 keys
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int e = lane + 32 * i;
    all[i] = e < splits * k ? __ldcg(reinterpret_cast<const unsigned long long*>(
                                  part_keys + static_cast<int64_t>(b) * splits * k + e))
                            : pad_key();
  }
  warp_topk_rounds<8>(all, k, nullptr, out_s + static_cast<int64_t>(b) * k,
                      out_id + static_cast<int64_t>(b) * k);
  if (lane == 0) arrivals[b] = 0;  // ready for the next launch on this workspace
}

// Contextual retrieval's chain in one launch (reference workloads.py:247-257:
// each query searches its own small index, then its hits are reranked): query b searches rows
// [q_rows[2b], q_rows[2b + 1]) of the arena (its own index segment, <= max_rows rows), keeps the
// top k_s (Searching), then scores those k_s rows against its rerank question and keeps the top
// k_r (Reranking). Unfused this is normalise + scan + merge + rerank: 4 launches, ~35 us as one
// CUDA graph, dominated by the scan's fixed costs on a 48-row segment. One block per query:
//  * warps 0 / 1 L2-normalise the search query / rerank question with the math of
//    normalize_kernel (so the bf16 vectors equal the unfused chain's staged ones) into shared
//    memory; every lane then keeps its 16-byte chunks of both as fp32 pairs in registers;
//  * each warp walks its rows (c = warp + kSegWarps j) through a cp.async ring, as
//    rerank_lists_kernel does, and scores every row against BOTH vectors from the one copy in
//    shared memory, with the lists kernel's exact arithmetic (packed FFMA2 over the chunks in
//    order, butterfly sum): a row's rerank score is bit-identical to K3's;
//  * selection by rank (count of larger keys; keys are unique: distinct ids): the k_s best
//    search keys land at their rank, then the k_r best of those by rerank score.
// The contraction is 2 x 48 rows x D per query: CUDA-core work, latency-bound either way.
constexpr int kSegWarps = 8;
constexpr int kSegSlots = 3;

template <int CPL, bool kTiled>
__global__ void __launch_bounds__(kSegWarps * 32) search_rerank_seg_kernel(
    const __nv_bfloat16* __restrict__ arena, int64_t nrows, int dim, const void* __restrict__ qs,
    const void* __restrict__ qr, int q_is_f32, int do_normalize, const int64_t* __restrict__ q_rows,
    int max_rows, int k_s, int k_r, int local_ids, float* __restrict__ os_s,
    int32_t* __restrict__ os_i, float* __restrict__ or_s, int32_t* __restrict__ or_i) {
  extern __shared__ __align__(16) uint8_t sm[];
  const int row_bytes = dim * 2;
  uint8_t* ring = sm;                                                   // [warps][slots][row]
  __nv_bfloat16* qv = reinterpret_cast<__nv_bfloat16*>(
      ring + static_cast<size_t>(kSegWarps) * kSegSlots * row_bytes);  // [2][dim]
  uint64_t* keys_s = reinterpret_cast<uint64_t*>(qv + 2 * dim);
  const int msel = min(k_s, max_rows);
  uint64_t* keys_r = keys_s + max_rows;
  float* score_r = reinterpret_cast<float*>(keys_r + msel);
  int32_t* sel = reinterpret_cast<int32_t*>(score_r + max_rows);
  const int b = blockIdx.x;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) pdl_allow_dependents();  // (see rerank_ring_kernel)
  pdl_wait();
  const int64_t rb = q_rows[2 * b];
  int64_t re = min(q_rows[2 * b + 1], nrows);
  if (re < rb) re = rb;
  const int n = static_cast<int>(min(re - rb, static_cast<int64_t>(max_rows)));
  auto id_of = [&](int c) { return static_cast<int32_t>(local_ids ? c : rb + c); };
  const int chunks = dim >> 3;
  const int64_t kb_per_row = (dim + 63) >> 6;
  const int nrow = warp < n ? (n - warp + kSegWarps - 1) / kSegWarps : 0;
  uint8_t* my_ring = ring + static_cast<size_t>(warp) * kSegSlots * row_bytes;
  auto issue = [&](int j, int slot) {  // whole warp; always commits one group
    if (j < nrow) {
      const int64_t r = rb + warp + static_cast<int64_t>(kSegWarps) * j;
      const uint4* src = kTiled ? reinterpret_cast<const uint4*>(
                                      arena + ((r >> 7) * kb_per_row * 128 + (r & 127)) * 64)
                                : reinterpret_cast<const uint4*>(arena + r * dim);
      uint4* dst = reinterpret_cast<uint4*>(my_ring + static_cast<size_t>(slot) * row_bytes);
#pragma unroll
      for (int jj = 0; jj < CPL; ++jj) {
        const int ch = lane + 32 * jj;
        if (ch < chunks)
          cp_async16(dst + ch, src + (kTiled ? static_cast<int64_t>(ch >> 3) * 1024 + (ch & 7) : ch));
      }
    }
    cp_async_commit();
  };
  // the rows' round trips start before the questions are normalised
#pragma unroll
  for (int s_ = 0; s_ < kSegSlots; ++s_) issue(s_, s_);
  if (warp < 2) {  // warp 0: search query, warp 1: rerank question (= the query when qr is null)
    const void* src = (warp == 1 && qr != nullptr) ? qr : qs;
    const float* sf = reinterpret_cast<const float*>(src) + static_cast<int64_t>(b) * dim;
    const __nv_bfloat16* sb = reinterpret_cast<const __nv_bfloat16*>(src) + static_cast<int64_t>(b) * dim;
    float ss = 0.f;
    if (do_normalize) {
      for (int d = lane; d < dim; d += 32) {
        const float x = q_is_f32 ? sf[d] : __bfloat162float(sb[d]);
        ss = fmaf(x, x, ss);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
    }
    const float scale = (do_normalize && ss > 0.f) ? rsqrtf(ss) : 1.f;
    __nv_bfloat16* out = qv + warp * dim;
    for (int d = lane; d < dim; d += 32) {
      const float x = q_is_f32 ? sf[d] : __bfloat162float(sb[d]);
      out[d] = __float2bfloat16_rn(x * scale);
    }
  }
  __syncthreads();
  float2 qa[CPL][4], qb[CPL][4];  // search query / rerank question, this lane's chunks
#pragma unroll
  for (int j = 0; j < CPL; ++j) {
    const int ch = lane + 32 * j;
    const uint4 wa = ch < chunks ? reinterpret_cast<const uint4*>(qv)[ch] : make_uint4(0, 0, 0, 0);
    const uint4 wb = ch < chunks ? reinterpret_cast<const uint4*>(qv + dim)[ch] : make_uint4(0, 0, 0, 0);
    qa[j][0] = bf16x2_to_float2(wa.x);
    qa[j][1] = bf16x2_to_float2(wa.y);
    qa[j][2] = bf16x2_to_float2(wa.z);
    qa[j][3] = bf16x2_to_float2(wa.w);
    qb[j][0] = bf16x2_to_float2(wb.x);
    qb[j][1] = bf16x2_to_float2(wb.y);
    qb[j][2] = bf16x2_to_float2(wb.z);
    qb[j][3] = bf16x2_to_float2(wb.w);
  }
  int slot = 0;
  for (int j = 0; j < nrow; ++j) {
    cp_async_wait<kSegSlots - 1>();
    __syncwarp();
    const uint4* row = reinterpret_cast<const uint4*>(my_ring + static_cast<size_t>(slot) * row_bytes);
    float2 a2 = make_float2(0.f, 0.f), b2 = make_float2(0.f, 0.f);
#pragma unroll
    for (int jj = 0; jj < CPL; ++jj) {
      const int ch = lane + 32 * jj;
      if (ch < chunks) {
        const uint4 raw = row[ch];
        const float2 x0 = bf16x2_to_float2(raw.x), x1 = bf16x2_to_float2(raw.y);
        const float2 x2 = bf16x2_to_float2(raw.z), x3 = bf16x2_to_float2(raw.w);
        a2 = __ffma2_rn(x0, qa[jj][0], a2);
        a2 = __ffma2_rn(x1, qa[jj][1], a2);
        a2 = __ffma2_rn(x2, qa[jj][2], a2);
        a2 = __ffma2_rn(x3, qa[jj][3], a2);
        b2 = __ffma2_rn(x0, qb[jj][0], b2);
        b2 = __ffma2_rn(x1, qb[jj][1], b2);
        b2 = __ffma2_rn(x2, qb[jj][2], b2);
        b2 = __ffma2_rn(x3, qb[jj][3], b2);
      }
    }
    float sa = a2.x + a2.y, sb2 = b2.x + b2.y;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      sa += __shfl_xor_sync(0xffffffffu, sa, o);
      sb2 += __shfl_xor_sync(0xffffffffu, sb2, o);
    }
    if (lane == 0) {
      const int c = warp + kSegWarps * j;
      keys_s[c] = make_key(sa, id_of(c));
      score_r[c] = sb2;
    }
    __syncwarp();  // every lane done reading the slot before it is refilled
    issue(j + kSegSlots, slot);
    if (++slot == kSegSlots) slot = 0;
  }
  cp_async_wait<0>();
  __syncthreads();
  // Searching: the k_s best rows by search score, at their rank
  for (int c = tid; c < n; c += kSegWarps * 32) {
    const uint64_t key = keys_s[c];
    int rank = 0;
    for (int j = 0; j < n; ++j) rank += keys_s[j] > key ? 1 : 0;
    if (rank < k_s) {
      os_s[static_cast<int64_t>(b) * k_s + rank] = key_score(key);
      os_i[static_cast<int64_t>(b) * k_s + rank] = key_id(key);
      sel[rank] = c;
    }
  }
  for (int r = n + tid; r < k_s; r += kSegWarps * 32) {
    os_s[static_cast<int64_t>(b) * k_s + r] = -INFINITY;
    os_i[static_cast<int64_t>(b) * k_s + r] = -1;
  }
  const int m = min(k_s, n);
  if (k_r <= 0) return;  // search-only mode (a batch of segmented Searching requests)
  __syncthreads();
  // Reranking of those rows against the question
  for (int r = tid; r < m; r += kSegWarps * 32) keys_r[r] = make_key(score_r[sel[r]], id_of(sel[r]));
  __syncthreads();
  for (int r = tid; r < m; r += kSegWarps * 32) {
    const uint64_t key = keys_r[r];
    int rank = 0;
    for (int j = 0; j < m; ++j) rank += keys_r[j] > key ? 1 : 0;
    if (rank < k_r) {
      or_s[static_cast<int64_t>(b) * k_r + rank] = key_score(key);
      or_i[static_cast<int64_t>(b) * k_r + rank] = key_id(key);
    }
  }
  for (int r = m + tid; r < k_r; r += kSegWarps * 32) {
    or_s[static_cast<int64_t>(b) * k_r + r] = -INFINITY;
    or_i[static_cast<int64_t>(b) * k_r + r] = -1;
  }
}

// K2s: latency-bound searches in ONE launch (BASELINE C1: 16 queries over a 10k x 384 corpus;
// reference: the naive-RAG Searching primitive, optimizer.py:178-198). The tensor-core scan
// costs ~27 us there as normalise + scan + merge (three launches; the scan's first-tile
// insertion chain and setup dominate a 40-tile corpus). Here a grid of (row blocks x query
// groups of QG) CTAs, 8 warps each:
//  * warps < QG L2-normalise one query each (normalize_kernel's math: the same bf16 query the
//    tensor-core path scans) into shared memory; every lane then holds its 16-byte chunks of
//    all QG queries as fp32 pairs in registers;
//  * each warp streams its rows (c = warp + 8 j) through a 6-slot cp.async ring; per row a lane
//    does CPL x QG x 4 packed FFMA2, and one "transposed" butterfly (QG-1 + 5 - log2 QG
//    shuffles instead of 5 QG) leaves lane l holding the full score of query l >> (5 - log2 QG);
//  * the owner lane of each query stores the row's score in shared memory ([QG][rows of the
//    block]); no per-row selection in the streaming loop (a per-row register-list insertion
//    was half of its instructions: with ~16 rows per warp most rows enter a k-list);
//  * then one warp per query selects the block's top k from those scores (lane-local sorted
//    key lists, k rounds of a warp max; keys (score, id) are unique, ties go to the smaller
//    id), writes them as keys to scratch, and the last block of the query group (arrival
//    counter, self-resetting) merges the row blocks' lists and writes the result.
constexpr int kSmallWarps = 8;
__device__ __forceinline__ unsigned long long global_ns_small() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
constexpr int kSmallSlots = 6;

// v[0..N) per lane -> full warp sum of v[q] in every lane whose (lane >> (5 - log2 N)) == q.
template <int N>
__device__ __forceinline__ float transpose_reduce(float (&v)[N], int lane) {
  int off = 16;
#pragma unroll
  for (int m = N; m > 1; m >>= 1) {
    const bool hi = (lane & off) != 0;
#pragma unroll
    for (int i = 0; i < m / 2; ++i) {
      const float send = hi ? v[i] : v[i + m / 2];
      const float keep = hi ? v[i + m / 2] : v[i];
      v[i] = keep + __shfl_xor_sync(0xffffffffu, send, off);
    }
    off >>= 1;
  }
  float r = v[0];
  for (; off > 0; off >>= 1) r += __shfl_xor_sync(0xffffffffu, r, off);
  return r;
}

// Insert key into a descending register list of K keys (precondition: key > l[K-1]).
template <int K>
__device__ __forceinline__ void key_list_insert(uint64_t (&l)[K], uint64_t key) {
#pragma unroll
  for (int i = K - 1; i > 0; --i) {
    const bool keep = l[i] > key;
    const bool prev_keep = l[i - 1] > key;
    l[i] = keep ? l[i] : (prev_keep ? key : l[i - 1]);
  }
  if (!(l[0] > key)) l[0] = key;
}

// Scores of one row against the QG queries, accumulated as packed fp32 pairs.
template <int QG, int CPL>
__device__ __forceinline__ void small_row_dot(const uint4* __restrict__ row, int lane, int chunks,
                                              const float2 (&qf)[QG][CPL][4], float2 (&acc)[QG]) {
#pragma unroll
  for (int qi = 0; qi < QG; ++qi) acc[qi] = make_float2(0.f, 0.f);
#pragma unroll
  for (int jj = 0; jj < CPL; ++jj) {
    const int ch = lane + 32 * jj;
    if (ch < chunks) {
      const uint4 raw = row[ch];
      const float2 x0 = bf16x2_to_float2(raw.x), x1 = bf16x2_to_float2(raw.y);
      const float2 x2 = bf16x2_to_float2(raw.z), x3 = bf16x2_to_float2(raw.w);
#pragma unroll
      for (int qi = 0; qi < QG; ++qi) {
        acc[qi] = __ffma2_rn(x0, qf[qi][jj][0], acc[qi]);
        acc[qi] = __ffma2_rn(x1, qf[qi][jj][1], acc[qi]);
        acc[qi] = __ffma2_rn(x2, qf[qi][jj][2], acc[qi]);
        acc[qi] = __ffma2_rn(x3, qf[qi][jj][3], acc[qi]);
      }
    }
  }
}

// k rounds of a warp-wide max over up to 32 * N keys held N per lane (pad-filled; keys unique):
// round r's key goes to out[r] (lane 0).
template <int N>
__device__ __forceinline__ void warp_select_rounds(uint64_t (&v)[N], int k, uint64_t* out, int lane) {
  const uint64_t pad = pad_key();
  for (int r = 0; r < k; ++r) {
    uint64_t m = v[0];
#pragma unroll
    for (int i = 1; i < N; ++i) m = v[i] > m ? v[i] : m;
    m = warp_max_key(m);
    if (lane == 0) out[r] = m;
    if (m == pad) {
      for (int rr = r + 1; rr < k && lane == 0; ++rr) out[rr] = pad;
      break;
    }
#pragma unroll
    for (int i = 0; i < N; ++i) v[i] = v[i] == m ? pad : v[i];
  }
}

template <int QG, int CPL, int KC, bool kTiled>
__global__ void __launch_bounds__(kSmallWarps * 32, 1) small_scan_kernel(
    const __nv_bfloat16* __restrict__ arena, int dim, const void* __restrict__ q, int q_is_f32,
    int do_normalize, int B, int64_t row_beg, int64_t row_end, int32_t id_offset, int k,
    int resident, uint64_t* __restrict__ part_keys, int32_t* __restrict__ arrive,
    float* __restrict__ out_s, int32_t* __restrict__ out_i, unsigned long long* __restrict__ trace) {
  // (trace: development timestamps per block and phase, TSV_SMALL_TRACE; null in production)
  auto stamp = [&](int ph) {
    if (trace != nullptr && threadIdx.x == 0)
      trace[(blockIdx.y * gridDim.x + blockIdx.x) * 8 + ph] = global_ns_small();
  };
  stamp(0);
  constexpr int kLog = QG == 16 ? 4 : (QG == 8 ? 3 : (QG == 4 ? 2 : (QG == 2 ? 1 : 0)));
  static_assert((1 << kLog) == QG, "QG must be a power of two <= 16");
  extern __shared__ __align__(16) uint8_t sm[];
  const int row_bytes = dim * 2;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = blockIdx.y, q0 = g * QG, nq = min(QG, B - q0);
  const int nblk = gridDim.x;
  const int64_t n = row_end - row_beg;
  const int64_t per = (n + nblk - 1) / nblk;
  const int64_t r0 = row_beg + blockIdx.x * per, r1 = min(row_end, r0 + per);
  const int nr = r1 > r0 ? static_cast<int>(r1 - r0) : 0;
  const int nrow = warp < nr ? (nr - warp + kSmallWarps - 1) / kSmallWarps : 0;
  // resident: every row of the warp has its own buffer (all loads issued at once, one round
  // trip); otherwise a kSmallSlots-deep ring
  const int slots = resident ? static_cast<int>((per + kSmallWarps - 1) / kSmallWarps) : kSmallSlots;
  uint8_t* ring = sm;                                                   // [warps][slots][row]
  __nv_bfloat16* qv = reinterpret_cast<__nv_bfloat16*>(
      ring + static_cast<size_t>(kSmallWarps) * slots * row_bytes);   // [QG][dim]
  float* sc = reinterpret_cast<float*>(qv + QG * dim);                  // [QG][per] scores
  __shared__ int last;
  __shared__ uint64_t sel_s[kSmallWarps][16];  // final selection, one row per warp
  const int chunks = dim >> 3;
  const int64_t kb_per_row = (dim + 63) >> 6;
  uint8_t* my_ring = ring + static_cast<size_t>(warp) * slots * row_bytes;
  pdl_wait();
  stamp(1);
  auto issue = [&](int j, int slot) {
    if (j < nrow) {
      const int64_t r = r0 + warp + static_cast<int64_t>(kSmallWarps) * j;
      const uint4* src = kTiled ? reinterpret_cast<const uint4*>(
                                      arena + ((r >> 7) * kb_per_row * 128 + (r & 127)) * 64)
                                : reinterpret_cast<const uint4*>(arena + r * dim);
      uint4* dst = reinterpret_cast<uint4*>(my_ring + static_cast<size_t>(slot) * row_bytes);
#pragma unroll
      for (int jj = 0; jj < CPL; ++jj) {
        const int ch = lane + 32 * jj;
        if (ch < chunks)
          cp_async16(dst + ch, src + (kTiled ? static_cast<int64_t>(ch >> 3) * 1024 + (ch & 7) : ch));
      }
    }
  };
  if (resident) {
    for (int j = 0; j < nrow; ++j) issue(j, j);
    cp_async_commit();
  } else {
#pragma unroll
    for (int s_ = 0; s_ < kSmallSlots; ++s_) {
      issue(s_, s_);
      cp_async_commit();
    }
  }
  // queries of this group -> shared memory, L2-normalised in fp32 and rounded to bf16 (K5's
  // arithmetic; each lane sums its 16-byte chunks, so the sum order is the chunk order): one
  // global round trip per query
  for (int qi = warp; qi < QG; qi += kSmallWarps) {
    uint4* out = reinterpret_cast<uint4*>(qv + qi * dim);
    float x[CPL][8];
#pragma unroll
    for (int j = 0; j < CPL; ++j) {
      const int ch = lane + 32 * j;
#pragma unroll
      for (int t = 0; t < 8; ++t) x[j][t] = 0.f;
      if (qi < nq && ch < chunks) {
        const int64_t o = static_cast<int64_t>(q0 + qi) * dim + ch * 8;
        if (q_is_f32) {
          const float4 a = __ldg(reinterpret_cast<const float4*>(reinterpret_cast<const float*>(q) + o));
          const float4 b = __ldg(reinterpret_cast<const float4*>(reinterpret_cast<const float*>(q) + o + 4));
          x[j][0] = a.x; x[j][1] = a.y; x[j][2] = a.z; x[j][3] = a.w;
          x[j][4] = b.x; x[j][5] = b.y; x[j][6] = b.z; x[j][7] = b.w;
        } else {
          const uint4 w = __ldg(reinterpret_cast<const uint4*>(reinterpret_cast<const __nv_bfloat16*>(q) + o));
          const float2 p0 = bf16x2_to_float2(w.x), p1 = bf16x2_to_float2(w.y);
          const float2 p2 = bf16x2_to_float2(w.z), p3 = bf16x2_to_float2(w.w);
          x[j][0] = p0.x; x[j][1] = p0.y; x[j][2] = p1.x; x[j][3] = p1.y;
          x[j][4] = p2.x; x[j][5] = p2.y; x[j][6] = p3.x; x[j][7] = p3.y;
        }
      }
    }
    float ss = 0.f;
    if (do_normalize) {
#pragma unroll
      for (int j = 0; j < CPL; ++j)
#pragma unroll
        for (int t = 0; t < 8; ++t) ss = fmaf(x[j][t], x[j][t], ss);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
    }
    const float scale = (do_normalize && ss > 0.f) ? rsqrtf(ss) : 1.f;
#pragma unroll
    for (int j = 0; j < CPL; ++j) {
      const int ch = lane + 32 * j;
      if (ch < chunks) {
        uint4 w;
        w.x = pack_bf16x2(x[j][0] * scale, x[j][1] * scale);
        w.y = pack_bf16x2(x[j][2] * scale, x[j][3] * scale);
        w.z = pack_bf16x2(x[j][4] * scale, x[j][5] * scale);
        w.w = pack_bf16x2(x[j][6] * scale, x[j][7] * scale);
        out[ch] = w;
      }
    }
  }
  __syncthreads();
  stamp(2);
  float2 qf[QG][CPL][4];
#pragma unroll
  for (int qi = 0; qi < QG; ++qi)
#pragma unroll
    for (int j = 0; j < CPL; ++j) {
      const int ch = lane + 32 * j;
      const uint4 w = ch < chunks ? reinterpret_cast<const uint4*>(qv + qi * dim)[ch]
                                  : make_uint4(0, 0, 0, 0);
      qf[qi][j][0] = bf16x2_to_float2(w.x);
      qf[qi][j][1] = bf16x2_to_float2(w.y);
      qf[qi][j][2] = bf16x2_to_float2(w.z);
      qf[qi][j][3] = bf16x2_to_float2(w.w);
    }
  const int my_q = lane >> (5 - kLog);
  const bool owner = (lane & ((1 << (5 - kLog)) - 1)) == 0;
  if (resident) {
    cp_async_wait<0>();
    __syncwarp();
    // two rows per step: their dot products and butterflies are independent (ILP)
    int j = 0;
    for (; j + 1 < nrow; j += 2) {
      float2 a0[QG], a1[QG];
      small_row_dot<QG, CPL>(reinterpret_cast<const uint4*>(my_ring + static_cast<size_t>(j) * row_bytes),
                             lane, chunks, qf, a0);
      small_row_dot<QG, CPL>(reinterpret_cast<const uint4*>(my_ring + static_cast<size_t>(j + 1) * row_bytes),
                             lane, chunks, qf, a1);
      float v0[QG], v1[QG];
#pragma unroll
      for (int qi = 0; qi < QG; ++qi) {
        v0[qi] = a0[qi].x + a0[qi].y;
        v1[qi] = a1[qi].x + a1[qi].y;
      }
      const float s0 = transpose_reduce<QG>(v0, lane);
      const float s1 = transpose_reduce<QG>(v1, lane);
      if (owner) {
        sc[my_q * per + warp + kSmallWarps * j] = s0;
        sc[my_q * per + warp + kSmallWarps * (j + 1)] = s1;
      }
    }
    if (j < nrow) {
      float2 a0[QG];
      small_row_dot<QG, CPL>(reinterpret_cast<const uint4*>(my_ring + static_cast<size_t>(j) * row_bytes),
                             lane, chunks, qf, a0);
      float v0[QG];
#pragma unroll
      for (int qi = 0; qi < QG; ++qi) v0[qi] = a0[qi].x + a0[qi].y;
      const float s0 = transpose_reduce<QG>(v0, lane);
      if (owner) sc[my_q * per + warp + kSmallWarps * j] = s0;
    }
  } else {
    int slot = 0;
    for (int j = 0; j < nrow; ++j) {
      cp_async_wait<kSmallSlots - 1>();
      __syncwarp();
      float2 acc[QG];
      small_row_dot<QG, CPL>(reinterpret_cast<const uint4*>(my_ring + static_cast<size_t>(slot) * row_bytes),
                             lane, chunks, qf, acc);
      __syncwarp();  // every lane done reading the slot before it is refilled
      issue(j + kSmallSlots, slot);
      cp_async_commit();
      if (++slot == kSmallSlots) slot = 0;
      float v[QG];
#pragma unroll
      for (int qi = 0; qi < QG; ++qi) v[qi] = acc[qi].x + acc[qi].y;
      const float score = transpose_reduce<QG>(v, lane);
      if (owner) sc[my_q * per + warp + kSmallWarps * j] = score;
    }
    cp_async_wait<0>();
  }
  __syncthreads();
  stamp(3);
  // block top-k per query (one warp per query: lane-local lists over the block's scores, then
  // k rounds of a warp max; (score, id) keys are unique, ties go to the smaller id) ->
  // scratch [groups][QG][nblk][k] (a query's lists contiguous for the final merge)
  const uint64_t pad = pad_key();
  for (int qi = warp; qi < nq; qi += kSmallWarps) {
    uint64_t l[KC];
#pragma unroll
    for (int i = 0; i < KC; ++i) l[i] = pad;
    for (int c = lane; c < nr; c += 32) {
      const uint64_t key = make_key(sc[qi * per + c], static_cast<int32_t>(r0 + c) + id_offset);
      if (key > l[KC - 1]) key_list_insert<KC>(l, key);
    }
    uint64_t* part = part_keys + ((static_cast<int64_t>(g) * QG + qi) * nblk + blockIdx.x) * k;
    for (int r = 0; r < k; ++r) {
      uint64_t m = l[0];
      m = warp_max_key(m);
      if (lane == 0) part[r] = m;
      if (l[0] == m && m != pad) {  // exactly one lane pops its head
#pragma unroll
        for (int i = 0; i < KC - 1; ++i) l[i] = l[i + 1];
        l[KC - 1] = pad;
      }
    }
  }
  __threadfence();
  __syncthreads();
  stamp(4);
  if (tid == 0) last = atomicAdd(arrive + g, 1) == nblk - 1;
  __syncthreads();
  stamp(5);
  if (!last) return;
  __threadfence();
  // last block of the group: one warp per query takes the top k of the row blocks' nblk * k
  // keys (contiguous: coalesced loads, all issued before any compare)
  for (int qi = warp; qi < nq; qi += kSmallWarps) {
    const uint64_t* src = part_keys + (static_cast<int64_t>(g) * QG + qi) * nblk * k;
    const int total = nblk * k;
    uint64_t* sel = sel_s[warp];
    if (total <= 32 * 16) {
      uint64_t v[16];
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        const int e = lane + 32 * u;
        v[u] = e < total ? static_cast<uint64_t>(__ldcg(reinterpret_cast<const unsigned long long*>(src + e)))
                         : pad;
      }
      warp_select_rounds<16>(v, k, sel, lane);
    } else {  // (many row blocks) lane-local lists first
      uint64_t l[KC];
#pragma unroll
      for (int i = 0; i < KC; ++i) l[i] = pad;
      for (int e = lane; e < total; e += 32) {
        const uint64_t key = static_cast<uint64_t>(__ldcg(reinterpret_cast<const unsigned long long*>(src + e)));
        if (key > l[KC - 1]) key_list_insert<KC>(l, key);
      }
      warp_select_rounds<KC>(l, k, sel, lane);
    }
    __syncwarp();
    if (lane == 0) {
      for (int r = 0; r < k; ++r) {
        const uint64_t m = sel[r];
        const int32_t id = m == pad ? -1 : key_id(m);
        out_s[static_cast<int64_t>(q0 + qi) * k + r] = id < 0 ? -INFINITY : key_score(m);
        out_i[static_cast<int64_t>(q0 + qi) * k + r] = id;
      }
    }
  }
  if (tid == 0) arrive[g] = 0;  // ready for the next launch on this scratch
  __syncthreads();
  stamp(6);
}

// One warp per row: optional L2 normalisation (fp32 math) and cast to bf16.
__global__ void normalize_kernel(const void* __restrict__ src, int src_is_f32, int64_t n, int dim,
                                 int do_normalize, __nv_bfloat16* __restrict__ dst) {
  pdl_allow_dependents();  // the scan after it sets up while the queries are normalised
  const int64_t row = static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= n) return;
  const float* sf = reinterpret_cast<const float*>(src) + row * dim;
  const __nv_bfloat16* sb = reinterpret_cast<const __nv_bfloat16*>(src) + row * dim;
  float ss = 0.f;
  if (do_normalize) {
    for (int d = lane; d < dim; d += 32) {
      const float x = src_is_f32 ? sf[d] : __bfloat162float(sb[d]);
      ss = fmaf(x, x, ss);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
  }
  const float scale = (do_normalize && ss > 0.f) ? rsqrtf(ss) : 1.f;
  __nv_bfloat16* out = dst + row * dim;
  for (int d = lane; d < dim; d += 32) {
    const float x = src_is_f32 ? sf[d] : __bfloat162float(sb[d]);
    out[d] = __float2bfloat16_rn(x * scale);
  }
}

// One warp per row: optional L2 normalisation (fp32) and split into a tf32 "hi" plane (low 13
// mantissa bits cleared) and the fp32 residual "lo" = x - hi, so hi*hi + hi*lo + lo*hi on the
// tf32 tensor cores reproduces fp32 products to ~2^-21 relative (fp32 mode, K1f).
__global__ void split_f32_kernel(const void* __restrict__ src, int src_is_f32, int64_t n, int dim,
                                 int do_normalize, float* __restrict__ hi, float* __restrict__ lo) {
  const int64_t row = static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= n) return;
  const float* sf = reinterpret_cast<const float*>(src) + row * dim;
  const __nv_bfloat16* sb = reinterpret_cast<const __nv_bfloat16*>(src) + row * dim;
  float ss = 0.f;
  if (do_normalize) {
    for (int d = lane; d < dim; d += 32) {
      const float x = src_is_f32 ? sf[d] : __bfloat162float(sb[d]);
      ss = fmaf(x, x, ss);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
  }
  const float scale = (do_normalize && ss > 0.f) ? 1.0f / sqrtf(ss) : 1.f;
  for (int d = lane; d < dim; d += 32) {
    const float x = (src_is_f32 ? sf[d] : __bfloat162float(sb[d])) * scale;
    const float h = __uint_as_float(__float_as_uint(x) & 0xFFFFE000u);
    hi[row * dim + d] = h;
    lo[row * dim + d] = x - h;
  }
}

// Tiled-layout ingest: one warp per row, optional L2 normalisation, bf16 cast, and scatter of
// the row's 64-element k-block pieces into their [128 x 64] tiles.
__global__ void scatter_tiled_kernel(const void* __restrict__ src, int src_is_f32, int64_t n,
                                     int dim, int do_normalize, __nv_bfloat16* __restrict__ arena,
                                     int64_t first_row) {
  const int64_t r = static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (r >= n) return;
  const float* sf = reinterpret_cast<const float*>(src) + r * dim;
  const __nv_bfloat16* sb = reinterpret_cast<const __nv_bfloat16*>(src) + r * dim;
  float ss = 0.f;
  if (do_normalize) {
    for (int d = lane; d < dim; d += 32) {
      const float x = src_is_f32 ? sf[d] : __bfloat162float(sb[d]);
      ss = fmaf(x, x, ss);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
  }
  const float scale = (do_normalize && ss > 0.f) ? rsqrtf(ss) : 1.f;
  const int64_t row = first_row + r;
  const int kbs = (dim + 63) >> 6;
  __nv_bfloat16* base = arena + ((row >> 7) * kbs * 128 + (row & 127)) * 64;
  for (int d = lane; d < dim; d += 32) {
    const float x = src_is_f32 ? sf[d] : __bfloat162float(sb[d]);
    base[static_cast<int64_t>(d >> 6) * 128 * 64 + (d & 63)] = __float2bfloat16_rn(x * scale);
  }
}

// Admission floor from a sample pass: one below the sample's k-th score (so ties at the final
// boundary stay admissible), or -FLT_MAX when the sample had fewer than k rows.
__global__ void seed_floor_kernel(const float* __restrict__ s, const int32_t* __restrict__ id,
                                  int B, int k, float* __restrict__ floor_out) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  const int64_t o = static_cast<int64_t>(b) * k + (k - 1);
  floor_out[b] = id[o] >= 0 ? nextafterf(s[o], -INFINITY) : -FLT_MAX;
}

// ---------------------------------------------------------------------------------------------
// Peer exchange fused with the cross-shard merge (sharded mode over NVLink / NVSwitch).
// Every rank owns a symmetric buffer:
//   header   word 0: abort flag (any rank that gave up waiting sets it in every buffer)
//   stamps   [world][max_b] u32: stamps[src][b] = epoch of the last call in which rank src
//            delivered query b's list into this buffer
//   recv_s / recv_i [2 parities][world][max_b][max_k]
// A call (epoch e, parity e & 1); CTA c owns a contiguous range of queries [b0, b1):
//   phase 1  push the range's local top-k lists into slot [parity][rank][b] of every peer's
//            buffer (stores through mapped peer memory, all threads), then ONE system-scope
//            fence by thread 0 and relaxed stores of stamp e into every peer's
//            stamps[rank][b], b in the range (fence + relaxed store = release). The first
//            version fenced per query and released every stamp separately: ~9 system fences
//            per query at G = 8, 0.2-0.5 ms per exchange (scripts/k6_probe.py);
//   phase 2  one thread per (source, query) of the range polls stamps[src][b] >= e (acquire),
//            then the range's queries are merged one by one by RANK: the world lists of a query
//            are each sorted (score desc, id asc), so the output position of entry j of list
//            r is j + (entries of every other list that order before it), a binary search per
//            list (ties broken by list index, so positions are unique), stopped as soon as the
//            position reaches k. Two block barriers per query instead of a bitonic sort.
// Stamps are per (source, query slot), so calls with different batch sizes interleave freely:
// a slot left untouched by a smaller batch is simply older, and the next call that covers it
// waits for that call's own stamp. A rank can be at most one call ahead of another (its next
// call waits for this call's stamps of every peer), so the two parities never alias.
// Every CTA sends everything before it waits and the grid is at most one CTA per SM, so no CTA
// waits on data that a non-resident CTA still has to send. A wait longer than timeout_ns (a
// peer that never arrives: dead rank, mismatched call sequence) aborts: the waiting CTA writes
// padding for its queries, raises the abort flag in every rank's buffer (their waits end at
// once) and in the caller-visible error word, and the host reports DeviceError.
struct PeerArgs {
  void* const* peers;  // device array: base of each rank's symmetric buffer
  int rank, world, B, k, max_b, max_k, parity;
  uint32_t epoch;
  uint64_t timeout_ns;
  const float* local_s;
  const int32_t* local_i;
  float* out_s;
  int32_t* out_i;
  uint32_t* err;  // host-mapped error word (1 = aborted)
};

constexpr size_t kPeerHeaderBytes = 256;

__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_relaxed_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.relaxed.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint64_t global_timer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__host__ __device__ __forceinline__ size_t peer_stamp_bytes(int world, int max_b) {
  return ((static_cast<size_t>(world) * max_b * 4 + 255) / 256) * 256;
}

constexpr int kPeerThreads = 256;

__global__ void __launch_bounds__(kPeerThreads) peer_exchange_merge_kernel(const PeerArgs a) {
  extern __shared__ uint64_t keys[];  // [world * k] keys of the query being merged
  __shared__ int nvalid;
  const size_t data_off = kPeerHeaderBytes + peer_stamp_bytes(a.world, a.max_b);
  const size_t plane = static_cast<size_t>(a.world) * a.max_b * a.max_k;  // entries per parity
  auto stamps = [&](void* base) {
    return reinterpret_cast<uint32_t*>(static_cast<uint8_t*>(base) + kPeerHeaderBytes);
  };
  auto recv_s = [&](void* base) {
    return reinterpret_cast<float*>(static_cast<uint8_t*>(base) + data_off);
  };
  auto recv_i = [&](void* base) {
    return reinterpret_cast<int32_t*>(static_cast<uint8_t*>(base) + data_off + 2 * plane * 4);
  };
  const int per = (a.B + gridDim.x - 1) / gridDim.x;
  const int b0 = blockIdx.x * per, b1 = min(a.B, b0 + per);
  if (b0 >= b1) return;
  const int nb = b1 - b0, tid = threadIdx.x;
  // phase 1: push this range's lists to every rank (own buffer included), one fence, stamps
  for (int p = 0; p < a.world; ++p) {
    void* base = a.peers[p];
    float* ds = recv_s(base);
    int32_t* di = recv_i(base);
    const size_t slot0 = ((static_cast<size_t>(a.parity) * a.world + a.rank) * a.max_b) * a.max_k;
    for (int e = tid; e < nb * a.k; e += blockDim.x) {
      const int bb = b0 + e / a.k, j = e - (e / a.k) * a.k;
      ds[slot0 + static_cast<size_t>(bb) * a.max_k + j] = a.local_s[static_cast<int64_t>(bb) * a.k + j];
      di[slot0 + static_cast<size_t>(bb) * a.max_k + j] = a.local_i[static_cast<int64_t>(bb) * a.k + j];
    }
  }
  __syncthreads();
  if (tid == 0) {
    __threadfence_system();
    for (int p = 0; p < a.world; ++p)
      for (int bb = b0; bb < b1; ++bb)
        st_relaxed_sys(stamps(a.peers[p]) + static_cast<size_t>(a.rank) * a.max_b + bb, a.epoch);
  }
  // phase 2: wait for every (source, query) of the range
  void* own = a.peers[a.rank];
  uint32_t* abort_word = static_cast<uint32_t*>(own);
  const uint32_t* st = stamps(own);
  const uint64_t t0 = global_timer_ns();
  int bad = 0;
  for (int w = tid; w < a.world * nb; w += blockDim.x) {
    const int src = w % a.world, bb = b0 + w / a.world;
    const uint32_t* sp = st + static_cast<size_t>(src) * a.max_b + bb;
    // (signed distance: stamps are a wrapping u32 epoch counter)
    while (static_cast<int32_t>(ld_acquire_sys(sp) - a.epoch) < 0) {
      if (ld_acquire_sys(abort_word) != 0 || global_timer_ns() - t0 > a.timeout_ns) {
        bad = 1;
        break;
      }
      __nanosleep(128);
    }
    if (bad) break;
  }
  if (__syncthreads_or(bad)) {
    if (tid == 0) {
      for (int p = 0; p < a.world; ++p) st_release_sys(static_cast<uint32_t*>(a.peers[p]), 1u);
      *reinterpret_cast<volatile uint32_t*>(a.err) = 1u;
      __threadfence_system();
    }
    for (int e = tid; e < nb * a.k; e += blockDim.x) {
      a.out_s[static_cast<int64_t>(b0) * a.k + e] = -INFINITY;
      a.out_i[static_cast<int64_t>(b0) * a.k + e] = -1;
    }
    return;
  }
  const volatile float* rs = recv_s(own);
  const volatile int32_t* ri = recv_i(own);
  const int n = a.world * a.k;
  const uint64_t pad = pad_key();
  for (int bb = b0; bb < b1; ++bb) {
    if (tid == 0) nvalid = 0;
    for (int i = tid; i < n; i += blockDim.x) {
      const int r = i / a.k, j = i - (i / a.k) * a.k;
      const size_t o = ((static_cast<size_t>(a.parity) * a.world + r) * a.max_b + bb) * a.max_k + j;
      const int32_t id = ri[o];
      keys[i] = id >= 0 ? make_key(rs[o], id) : pad;
    }
    __syncthreads();
    int mine = 0;
    for (int i = tid; i < n; i += blockDim.x) {
      const uint64_t key = keys[i];
      if (key == pad) continue;
      ++mine;
      const int r = i / a.k;
      int pos = i - r * a.k;
      for (int r2 = 0; r2 < a.world && pos < a.k; ++r2) {
        if (r2 == r) continue;
        const uint64_t* L = keys + r2 * a.k;
        int lo = 0, hi = a.k;  // entries of list r2 ordered before `key`
        while (lo < hi) {
          const int mid = (lo + hi) >> 1;
          const uint64_t x = L[mid];
          if (x > key || (r2 < r && x == key)) lo = mid + 1;
          else hi = mid;
        }
        pos += lo;
      }
      if (pos < a.k) {
        a.out_s[static_cast<int64_t>(bb) * a.k + pos] = key_score(key);
        a.out_i[static_cast<int64_t>(bb) * a.k + pos] = key_id(key);
      }
    }
    if (mine) atomicAdd(&nvalid, mine);
    __syncthreads();
    for (int pos = nvalid + tid; pos < a.k; pos += blockDim.x) {
      a.out_s[static_cast<int64_t>(bb) * a.k + pos] = -INFINITY;
      a.out_i[static_cast<int64_t>(bb) * a.k + pos] = -1;
    }
    __syncthreads();  // keys / nvalid reused by the next query
  }
}

// Launch with programmatic stream serialisation (see pdl_wait in tsv_kernels.cuh).
template <typename... KArgs, typename... Args>
int launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t stream,
               Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return static_cast<int>(cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...));
}

}  // namespace

size_t peer_buffer_bytes(int world, int max_b, int max_k) {
  return kPeerHeaderBytes + peer_stamp_bytes(world, max_b) +
         2 * 2 * static_cast<size_t>(world) * max_b * max_k * 4;
}

int launch_peer_exchange_merge(void* const* peers_dev, int rank, int world, int B, int k,
                               int max_b, int max_k, uint32_t epoch, uint64_t timeout_ns,
                               const float* local_s, const int32_t* local_i, float* out_s,
                               int32_t* out_i, uint32_t* err_word, int num_sms,
                               cudaStream_t stream) {
  PeerArgs a{peers_dev, rank, world, B, k, max_b, max_k, static_cast<int>(epoch & 1u), epoch,
             timeout_ns, local_s, local_i, out_s, out_i, err_word};
  const int grid = B < num_sms ? B : num_sms;
  const size_t smem = static_cast<size_t>(world) * k * sizeof(uint64_t);
  if (smem > 48 * 1024) {
    static std::atomic<uint64_t> configured{0};
    if (first_on_device(configured)) {
      cudaError_t e = cudaFuncSetAttribute(peer_exchange_merge_kernel,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      if (e != cudaSuccess) return static_cast<int>(e);
    }
  }
  peer_exchange_merge_kernel<<<grid, kPeerThreads, smem, stream>>>(a);
  return static_cast<int>(cudaGetLastError());
}

int launch_seed_floor(const float* s, const int32_t* id, int B, int k, float* floor_out,
                      cudaStream_t stream) {
  if (B <= 0) return 0;
  seed_floor_kernel<<<(B + 255) / 256, 256, 0, stream>>>(s, id, B, k, floor_out);
  return static_cast<int>(cudaGetLastError());
}

int launch_scatter_tiled(const void* src, int src_is_f32, int64_t n, int dim, int do_normalize,
                         void* arena, int64_t first_row, cudaStream_t stream) {
  if (n <= 0) return 0;
  constexpr int kWarps = 8;
  const int64_t blocks = (n + kWarps - 1) / kWarps;
  scatter_tiled_kernel<<<static_cast<unsigned>(blocks), kWarps * 32, 0, stream>>>(
      src, src_is_f32, n, dim, do_normalize, reinterpret_cast<__nv_bfloat16*>(arena), first_row);
  return static_cast<int>(cudaGetLastError());
}

int launch_split_f32(const void* src, int src_is_f32, int64_t n, int dim, int do_normalize,
                     float* hi, float* lo, cudaStream_t stream) {
  if (n <= 0) return 0;
  constexpr int kWarps = 8;
  const int64_t blocks = (n + kWarps - 1) / kWarps;
  split_f32_kernel<<<static_cast<unsigned>(blocks), kWarps * 32, 0, stream>>>(
      src, src_is_f32, n, dim, do_normalize, hi, lo);
  return static_cast<int>(cudaGetLastError());
}

int launch_cand_select(const float* buf_s, const int32_t* buf_i, const int32_t* cnt, int cap,
                       int B, int kout, float* out_s, int32_t* out_id, int32_t* overflow,
                       cudaStream_t stream) {
  if (B <= 0) return 0;
  int np = 1;
  while (np < cap) np <<= 1;
  int kp = 1;
  while (kp < kout) kp <<= 1;
  const size_t smem = static_cast<size_t>(np + kp) * sizeof(uint64_t);
  if (smem > 200 * 1024) return static_cast<int>(cudaErrorInvalidValue);
  static std::atomic<uint64_t> configured{0};
  if (smem > 48 * 1024 && first_on_device(configured)) {
    cudaError_t e = cudaFuncSetAttribute(cand_select_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    if (e != cudaSuccess) return static_cast<int>(e);
  }
  return launch_pdl(cand_select_kernel, dim3(B), dim3(256), smem, stream, buf_s, buf_i, cnt, cap,
                    kout, out_s, out_id, overflow);
}

int launch_merge_topk(const float* in_s, const int32_t* in_id, int lists, int B, int kin,
                      int64_t list_stride_rows, int kout, float* out_s, int32_t* out_id,
                      cudaStream_t stream, int dedup, const int32_t* gate) {
  if (B <= 0) return 0;
  int np = 1;
  while (np < lists * kin) np <<= 1;
  if (np > 16384) return static_cast<int>(cudaErrorInvalidValue);
  int kp = 1;
  while (kp < kout) kp <<= 1;
  const size_t smem = static_cast<size_t>(np + kp) * sizeof(uint64_t);  // keys + selection
  static std::atomic<uint64_t> configured{0};
  if (smem > 48 * 1024 && first_on_device(configured)) {
    cudaError_t e = cudaFuncSetAttribute(merge_topk_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, 132 * 1024);
    if (e != cudaSuccess) return static_cast<int>(e);
  }
  const int threads = np >= 1024 ? 256 : (np >= 256 ? 128 : 64);
  return launch_pdl(merge_topk_kernel, dim3(B), dim3(threads), smem, stream, in_s, in_id, lists,
                    B, kin, list_stride_rows, kout, out_s, out_id, dedup, gate);
}

template <int kThreads, int kPer, int kUnroll>
int launch_rerank_v(const void* arena, const float* arena_hi, const float* arena_lo, int64_t nrows,
                    int dim, const void* q, const float* q_lo, int q_is_f32, int B,
                    const int32_t* cand, int C, int k, float* out_s, int32_t* out_id,
                    cudaStream_t stream, int tiled, size_t smem, const int32_t* offs) {
  auto kern = rerank_kernel<kThreads, kPer, kUnroll>;
  static std::atomic<uint64_t> configured{0};
  if (smem > 48 * 1024 && first_on_device(configured)) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    if (e != cudaSuccess) return static_cast<int>(e);
  }
  kern<<<B, kThreads, smem, stream>>>(reinterpret_cast<const __nv_bfloat16*>(arena), arena_hi,
                                      arena_lo, nrows, dim, q, q_lo, q_is_f32, cand, C, k, out_s,
                                      out_id, tiled, offs);
  return static_cast<int>(cudaGetLastError());
}

int launch_rerank(const void* arena, const float* arena_hi, const float* arena_lo, int64_t nrows,
                  int dim, const void* q, const float* q_lo, int q_is_f32, int B,
                  const int32_t* cand, int C, int k, float* out_s, int32_t* out_id,
                  cudaStream_t stream, int tiled, const int32_t* offs) {
  if (B <= 0) return 0;
  int np = 1;
  while (np < C) np <<= 1;
  const size_t smem = ((static_cast<size_t>(dim) * 4 + 15) & ~size_t(15)) + np * sizeof(uint64_t) +
                      static_cast<size_t>(C) * sizeof(int32_t);
  if (smem > 200 * 1024) return static_cast<int>(cudaErrorInvalidValue);
  // 20 warps x 2 rows per iteration, chunk loop unrolled 4x (every load of a row pair in
  // flight at once for dim <= 1024), two blocks per SM: C=200 takes 5 iterations. Measured at
  // C3 (256 x 200 x 768, rows from HBM): 24.8 us vs 32.6 with 16 warps x 4 rows, unroll 2.
  return launch_rerank_v<640, 2, 4>(arena, arena_hi, arena_lo, nrows, dim, q, q_lo, q_is_f32, B,
                                    cand, C, k, out_s, out_id, stream, tiled, smem, offs);
}

// TSV_RERANK_BITONIC=1: the ring kernel's block-wide bitonic sort + serial dedup (the round-2
// middle version) instead of the one-warp selection, for A/B runs.
// TSV_RERANK_NO_NET=1: k serial selection rounds instead of the warp top-k network (bit 1).
static int rerank_use_sort() {
  auto on = [](const char* v) { return v != nullptr && v[0] != '\0' && v[0] != '0'; };
  return (on(getenv("TSV_RERANK_BITONIC")) ? 1 : 0) | (on(getenv("TSV_RERANK_NO_NET")) ? 2 : 0);
}

template <int kWarps, int kSlots, int CPL, bool kTiled>
int launch_rerank_ring_v(const void* arena, int64_t nrows, int dim, const void* q, int q_is_f32,
                         int B, const int32_t* cand, int C, int k, const int32_t* offs,
                         float* out_s, int32_t* out_id, cudaStream_t stream) {
  int np = 1;
  while (np < C) np <<= 1;
  const size_t smem = static_cast<size_t>(kWarps) * kSlots * dim * 2 + np * sizeof(uint64_t) +
                      static_cast<size_t>(C) * sizeof(int32_t);
  if (smem > 220 * 1024) return static_cast<int>(cudaErrorInvalidValue);
  auto kern = rerank_ring_kernel<kWarps, kSlots, CPL, kTiled>;
  static std::atomic<uint64_t> configured{0};
  if (smem > 48 * 1024 && first_on_device(configured)) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    if (e != cudaSuccess) return static_cast<int>(e);
  }
  return launch_pdl(kern, dim3(B), dim3(kWarps * 32), smem, stream,
                    reinterpret_cast<const __nv_bfloat16*>(arena), nrows, dim, q, q_is_f32, cand, C,
                    k, offs, out_s, out_id, rerank_use_sort());
}

struct RerankSplit {  // split mode scratch (see rerank_lists_kernel)
  int splits = 1;
  uint64_t* part_keys = nullptr;  // [B * splits * k]
  int32_t* arrivals = nullptr;    // [B], zero between launches
};

template <int kWarps, int kSlots, int CPL, bool kTiled>
int launch_rerank_lists_v(const void* arena, int64_t nrows, int dim, const void* q, int q_is_f32,
                          int B, const int32_t* cand, int C, int k, const int32_t* offs,
                          float* out_s, int32_t* out_id, cudaStream_t stream,
                          const RerankSplit& sp) {
  const size_t smem = static_cast<size_t>(kWarps) * kSlots * dim * 2 +
                      static_cast<size_t>(kWarps) * 32 * sizeof(uint64_t);
  if (smem > 220 * 1024) return static_cast<int>(cudaErrorInvalidValue);
  auto kern = rerank_lists_kernel<kWarps, kSlots, CPL, kTiled>;
  static std::atomic<uint64_t> configured{0};
  if (smem > 48 * 1024 && first_on_device(configured)) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    if (e != cudaSuccess) return static_cast<int>(e);
  }
  return launch_pdl(kern, dim3(B * sp.splits), dim3(kWarps * 32), smem, stream,
                    reinterpret_cast<const __nv_bfloat16*>(arena), nrows, dim, q, q_is_f32, cand, C,
                    k, offs, out_s, out_id, sp.splits, sp.part_keys, sp.arrivals);
}

template <int CPL, bool kTiled>
int launch_rerank_ring_s(int slots, const void* arena, int64_t nrows, int dim, const void* q,
                         int q_is_f32, int B, const int32_t* cand, int C, int k,
                         const int32_t* offs, float* out_s, int32_t* out_id, cudaStream_t stream,
                         const RerankSplit& sp) {
  // per-warp lists (no block-wide sort) for k <= 32 with at most 32 candidates per warp:
  // 8 warps per block by default (TSV_RERANK_WARPS=16 / 32 for A/B)
  const int per_block = (C + sp.splits - 1) / sp.splits;
  int nw = 8;
  if (const char* w = getenv("TSV_RERANK_WARPS")) nw = atoi(w);
  if (per_block > nw * 32) nw = per_block <= 16 * 32 ? 16 : 32;
  // The ring kernel (16 warps, one-warp selection) wherever its blocks fit one wave (B <= 2
  // per SM): C3 256 x 200 x 768 18.6 vs 20.2 us (lists), C5 16 x 32 x 1024 4.4 vs 4.9,
  // 64 x 100 x 1024 9.9 vs 11.9, 256 x 32 x 768 5.6 vs 6.1. Many questions with short lists
  // go to the per-warp lists (8-warp blocks, more resident per SM): 1024 x 50 x 768 23.1 vs
  // 34.1 us (scripts/rerank_probe.py with PROBE_SHAPES). TSV_RERANK_LISTS forces the lists.
  const bool lists_ok = sp.splits > 1 || (B > 296 && C < 128) || getenv("TSV_RERANK_LISTS");
  if (k <= 32 && per_block <= nw * 32 && lists_ok && !getenv("TSV_RERANK_SORT")) {
#define TSV_LISTS(W, S) launch_rerank_lists_v<W, S, CPL, kTiled>(arena, nrows, dim, q, q_is_f32, B, cand, C, k, offs, out_s, out_id, stream, sp)
    if (nw == 8) return slots == 2 ? TSV_LISTS(8, 2) : (slots == 3 ? TSV_LISTS(8, 3) : TSV_LISTS(8, 4));
    if (nw == 16) return slots == 2 ? TSV_LISTS(16, 2) : (slots == 3 ? TSV_LISTS(16, 3) : TSV_LISTS(16, 4));
    if (nw == 32 && 32 * 2 * dim * 2 <= 200 * 1024) return TSV_LISTS(32, 2);
#undef TSV_LISTS
  }
  if (sp.splits != 1) return static_cast<int>(cudaErrorInvalidValue);
  switch (slots) {
    case 2: return launch_rerank_ring_v<16, 2, CPL, kTiled>(arena, nrows, dim, q, q_is_f32, B, cand, C, k, offs, out_s, out_id, stream);
    case 3: return launch_rerank_ring_v<16, 3, CPL, kTiled>(arena, nrows, dim, q, q_is_f32, B, cand, C, k, offs, out_s, out_id, stream);
    default: return launch_rerank_ring_v<16, 4, CPL, kTiled>(arena, nrows, dim, q, q_is_f32, B, cand, C, k, offs, out_s, out_id, stream);
  }
}

template <bool kTiled>
int launch_rerank_ring_t(int slots, const void* arena, int64_t nrows, int dim, const void* q,
                         int q_is_f32, int B, const int32_t* cand, int C, int k,
                         const int32_t* offs, float* out_s, int32_t* out_id, cudaStream_t stream,
                         const RerankSplit& sp) {
  const int cpl = (dim / 8 + 31) / 32;  // 16-byte chunks per lane
#define TSV_RING(N) launch_rerank_ring_s<N, kTiled>(slots, arena, nrows, dim, q, q_is_f32, B, cand, C, k, offs, out_s, out_id, stream, sp)
  if (cpl <= 1) return TSV_RING(1);
  if (cpl <= 2) return TSV_RING(2);
  if (cpl <= 3) return TSV_RING(3);
  if (cpl <= 4) return TSV_RING(4);
  if (cpl <= 8) return TSV_RING(8);
#undef TSV_RING
  return static_cast<int>(cudaErrorInvalidValue);
}

int rerank_lists_splits(int B, int C, int k, int dim, int num_sms) {
  if (k > 32 || dim > 2048 || getenv("TSV_RERANK_SORT")) return 1;
  // Measured (C3, C5): spreading one question over several blocks is slower (more per-block
  // setup for a kernel that is bound by instruction issue), so splitting is opt-in.
  if (!getenv("TSV_RERANK_SPLITS")) return 1;
  int splits = (6 * num_sms + B - 1) / B;  // ~6 blocks of 8 warps per SM
  splits = std::min(splits, std::max(1, C / 16));  // >= 16 candidates per block
  splits = std::max(1, std::min(splits, std::min(8, 256 / k)));
  if (const char* e = getenv("TSV_RERANK_SPLITS")) splits = std::max(1, std::min(8, atoi(e)));
  while (splits < 8 && (C + splits - 1) / splits > 32 * 32) ++splits;
  return splits;
}

size_t search_rerank_seg_smem(int dim, int max_rows, int k_s) {
  const int msel = std::min(k_s, max_rows);
  return static_cast<size_t>(kSegWarps) * kSegSlots * dim * 2 + static_cast<size_t>(dim) * 4 +
         static_cast<size_t>(max_rows) * 12 + static_cast<size_t>(msel) * 12;
}

template <int CPL, bool kTiled>
int launch_search_rerank_seg_v(size_t smem, const void* arena, int64_t nrows, int dim,
                               const void* qs, const void* qr, int q_is_f32, int do_normalize,
                               const int64_t* q_rows, int B, int max_rows, int k_s, int k_r,
                               int local_ids, float* os_s, int32_t* os_i, float* or_s,
                               int32_t* or_i, cudaStream_t stream) {
  auto kern = search_rerank_seg_kernel<CPL, kTiled>;
  static std::atomic<uint64_t> configured{0};
  if (first_on_device(configured)) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    if (e != cudaSuccess) return static_cast<int>(e);
  }
  return launch_pdl(kern, dim3(B), dim3(kSegWarps * 32), smem, stream,
                    reinterpret_cast<const __nv_bfloat16*>(arena), nrows, dim, qs, qr, q_is_f32,
                    do_normalize, q_rows, max_rows, k_s, k_r, local_ids, os_s, os_i, or_s, or_i);
}

int launch_search_rerank_seg(const void* arena, int64_t nrows, int dim, int tiled, const void* qs,
                             const void* qr, int q_is_f32, int do_normalize,
                             const int64_t* q_rows, int B, int max_rows, int k_s, int k_r,
                             int local_ids, float* os_s, int32_t* os_i, float* or_s,
                             int32_t* or_i, cudaStream_t stream) {
  if (B <= 0) return 0;
  const size_t smem = search_rerank_seg_smem(dim, max_rows, k_s);
  if (smem > 220 * 1024 || dim % 8 != 0 || dim > 2048) return static_cast<int>(cudaErrorInvalidValue);
  const int cpl = (dim / 8 + 31) / 32;
#define TSV_SEG(C, T) launch_search_rerank_seg_v<C, T>(smem, arena, nrows, dim, qs, qr, q_is_f32, do_normalize, q_rows, B, max_rows, k_s, k_r, local_ids, os_s, os_i, or_s, or_i, stream)
#define TSV_SEG_T(C) (tiled ? TSV_SEG(C, true) : TSV_SEG(C, false))
  if (cpl <= 1) return TSV_SEG_T(1);
  if (cpl <= 2) return TSV_SEG_T(2);
  if (cpl <= 4) return TSV_SEG_T(4);
  return TSV_SEG_T(8);
#undef TSV_SEG_T
#undef TSV_SEG
}

int small_scan_qg(int dim) { return dim <= 256 ? 16 : (dim <= 512 ? 8 : 4); }

template <int QG, int CPL, int KC, bool kTiled>
int launch_small_scan_v(const void* arena, int dim, const void* q, int q_is_f32, int do_normalize,
                        int B, int64_t row_beg, int64_t row_end, int32_t id_offset, int k,
                        int nblk, uint64_t* part_keys, int32_t* arrive, float* out_s,
                        int32_t* out_i, cudaStream_t stream, unsigned long long* trace) {
  const int64_t n = row_end - row_beg;
  const int64_t per = (n + nblk - 1) / nblk;
  const size_t fixed = static_cast<size_t>(QG) * dim * 2 + static_cast<size_t>(QG) * per * 4;
  const int64_t rows_per_warp = (per + kSmallWarps - 1) / kSmallWarps;
  // every row of the block resident in shared memory when it fits (one load round trip)
  const size_t res_bytes = static_cast<size_t>(kSmallWarps) * rows_per_warp * dim * 2 + fixed;
  const int resident = res_bytes <= 200 * 1024 && !getenv("TSV_SMALL_RING") ? 1 : 0;
  const size_t smem = resident ? res_bytes
                               : static_cast<size_t>(kSmallWarps) * kSmallSlots * dim * 2 + fixed;
  if (smem > 200 * 1024) return static_cast<int>(cudaErrorInvalidValue);
  auto kern = small_scan_kernel<QG, CPL, KC, kTiled>;
  static std::atomic<uint64_t> configured{0};
  if (first_on_device(configured)) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    if (e != cudaSuccess) return static_cast<int>(e);
  }
  const int groups = (B + QG - 1) / QG;
  return launch_pdl(kern, dim3(nblk, groups), dim3(kSmallWarps * 32), smem, stream,
                    reinterpret_cast<const __nv_bfloat16*>(arena), dim, q, q_is_f32, do_normalize,
                    B, row_beg, row_end, id_offset, k, resident, part_keys, arrive, out_s, out_i,
                    trace);
}

int launch_small_scan(const void* arena, int dim, int tiled, const void* q, int q_is_f32,
                      int do_normalize, int B, int64_t row_beg, int64_t row_end, int32_t id_offset,
                      int k, int nblk, uint64_t* part_keys, int32_t* arrive, float* out_s,
                      int32_t* out_i, cudaStream_t stream, unsigned long long* trace) {
  if (dim % 8 != 0 || dim > 1024 || k > 16) return static_cast<int>(cudaErrorInvalidValue);
#define TSV_SMALL(QG, CPL, KC, T) launch_small_scan_v<QG, CPL, KC, T>(arena, dim, q, q_is_f32, do_normalize, B, row_beg, row_end, id_offset, k, nblk, part_keys, arrive, out_s, out_i, stream, trace)
#define TSV_SMALL_K(QG, CPL, T) (k <= 8 ? TSV_SMALL(QG, CPL, 8, T) : TSV_SMALL(QG, CPL, 16, T))
#define TSV_SMALL_D(T) (dim <= 256 ? TSV_SMALL_K(16, 1, T) : (dim <= 512 ? TSV_SMALL_K(8, 2, T) : TSV_SMALL_K(4, 4, T)))
  return tiled ? TSV_SMALL_D(true) : TSV_SMALL_D(false);
#undef TSV_SMALL_D
#undef TSV_SMALL_K
#undef TSV_SMALL
}

// Pipelined gather (bf16 arenas, dim <= 2048): cp.async rings of `slots` rows per warp, split
// over blocks per rerank_lists_splits. 2 slots where two blocks share an SM (C3, 256 x 200 x
// 768: 17.7 us vs 19.1 with 4); 4 slots scored two rows at a time where the grid leaves one
// block per SM and each warp has >= 4 rows (128 x 200 x 1024: 15.4 vs 16.8 us, 64 x 100 x
// 1024: 9.6 vs 10.2; C5's 16 x 32: 4.3 vs 4.2; profiles/r02/rerank_probe_paired.txt).
int launch_rerank_ring(const void* arena, int64_t nrows, int dim, const void* q, int q_is_f32,
                       int B, const int32_t* cand, int C, int k, const int32_t* offs,
                       float* out_s, int32_t* out_id, cudaStream_t stream, int tiled,
                       int splits, uint64_t* part_keys, int32_t* arrivals, int num_sms) {
  if (B <= 0) return 0;
  const int row_bytes = dim * 2;
  int slots = (B * splits <= num_sms && C >= 64) ? 4 : 2;
  if (const char* e = getenv("TSV_RERANK_SLOTS")) slots = atoi(e);
  slots = slots < 2 ? 2 : (slots > 4 ? 4 : slots);
  while (slots > 2 && 16 * slots * row_bytes > 200 * 1024) --slots;
  if (dim > 2048) return static_cast<int>(cudaErrorInvalidValue);
  RerankSplit sp{splits, part_keys, arrivals};
  return tiled ? launch_rerank_ring_t<true>(slots, arena, nrows, dim, q, q_is_f32, B, cand, C, k, offs, out_s, out_id, stream, sp)
               : launch_rerank_ring_t<false>(slots, arena, nrows, dim, q, q_is_f32, B, cand, C, k, offs, out_s, out_id, stream, sp);
}

int launch_normalize(const void* src, int src_is_f32, int64_t n, int dim, int do_normalize,
                     void* dst_bf16, cudaStream_t stream) {
  if (n <= 0) return 0;
  constexpr int kWarps = 8;
  const int64_t blocks = (n + kWarps - 1) / kWarps;
  normalize_kernel<<<static_cast<unsigned>(blocks), kWarps * 32, 0, stream>>>(
      src, src_is_f32, n, dim, do_normalize, reinterpret_cast<__nv_bfloat16*>(dst_bf16));
  return static_cast<int>(cudaGetLastError());
}

}  // namespace tsv
