// K1 / K2: fused inner-product scan + per-query top-k on sm_100a.
//
// Replaces the latency lookup that Teola's simulator performs for a Searching batch
// (reference: pkg/src/teola_sim/runtime.py:653-655 `_execute` PHASE_GENERAL branch, whose
// table lives in pkg/src/teola_sim/profiles/default.json:47-70 `vdb-search0`).
//
// Design (one persistent CTA per SM, warp-specialised):
//   warp 0      TMA producer: per k-block, MB query tiles [128 x 64] + one corpus tile
//               [128 x 64] bf16, SWIZZLE_128B, into a STAGES-deep smem ring.
//   warp 1      MMA issuer: tcgen05.mma.cta_group::1.kind::f16, M=128 (queries) x N=128
//               (corpus rows) x K=16, fp32 accumulators in TMEM, double-buffered
//               (2 x MB x 128 columns).
//   warps 4..   epilogue: one thread per query (= TMEM lane). tcgen05.ld 32 columns at a
//               time, max-reduce, and only if the chunk beats the running threshold insert
//               into a register-resident sorted list of KCAP (score, id) pairs.
// The score matrix never leaves TMEM. Each CTA emits one sorted partial list per query per
// work item; K4 (tsv_merge.cu) merges the partial lists of all corpus ranges.
#include "tsv_kernels.cuh"
#include "tsv_ptx.cuh"

#include <cuda_bf16.h>
#include <cfloat>
#include <cstdlib>
#include <utility>

namespace tsv {
namespace {

constexpr int kLockWindow = 2;  // 256-row tiles a worker may run ahead of its range partners

// Range lockstep is a cache optimisation, never a correctness requirement: the launch is not
// cooperative, so a partner CTA may not be resident (another kernel holds SMs: concurrent
// scans on two streams, MPS, green contexts). A wait that sees no progress for kLockSpinNs
// gives up and the waiter runs the rest of its item unlocked (it keeps publishing its own
// progress for partners that do wait). Co-resident partners are never more than a tile or two
// (~15-30 us at D=1024) behind, so the bound only fires when a partner cannot run.
constexpr uint64_t kLockSpinNs = 200 * 1000;
__device__ __forceinline__ uint64_t global_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// Wait until *progress >= target; false when it stalled for kLockSpinNs (partner not running).
__device__ __forceinline__ bool lock_wait(volatile int32_t* progress, int64_t target) {
  if (*progress >= target) return true;
  int32_t seen = *progress;
  uint64_t t0 = global_ns();
  while (true) {
    __nanosleep(256);
    const int32_t now = *progress;
    if (now >= target) return true;
    if (now != seen) {  // partner moving: restart the stall clock
      seen = now;
      t0 = global_ns();
    } else if (global_ns() - t0 > kLockSpinNs) {
      return false;
    }
  }
}

// Lists of more than kRegListMax entries live in shared memory (one column per query thread,
// entry j of thread t at [j * 128 + t], so lock-step accesses are bank-conflict free).
constexpr int kRegListMax = 32;

// TF32 = fp32 mode (K1f): operands are fp32 (hi, lo) splits, 32 elements per 128-byte k-block
// row, three kind::tf32 MMAs per k-step (hi*hi + hi*lo + lo*hi).
// NB = 2 (wide tile): M=128 queries x N=256 corpus rows per MMA, for 64 < B <= 128 on long
// scans: the query operand is re-read from L2 once per 256 corpus rows instead of per 128.
template <int MB, int KCAP = 1, bool TF32 = false, int NB = 1>
struct ScanCfg {
  static constexpr int kTileN = NB * kBlockN;                      // corpus rows per tile
  static constexpr bool kSmemList = KCAP > kRegListMax;
  static constexpr int kParts = TF32 ? 2 : 1;                      // hi (+ lo) planes
  static constexpr int kABytes = kBlockM * 128;                    // 16 KB per plane tile
  static constexpr int kBBytes = kTileN * 128;                     // 16 (32) KB per plane tile
  static constexpr int kStageBytes = kParts * (MB * kABytes + kBBytes);
  static constexpr int kListBytes = kSmemList ? kBlockM * KCAP * 8 : 0;
  static constexpr int kStages =
      (kSmemList || TF32 || NB > 1) ? (227 * 1024 - 2048 - kListBytes) / kStageBytes
                                    : (MB == 2 ? 4 : 7);
  // fp32 mode keeps three accumulators per tile (hi*hi of even k-blocks, of odd k-blocks, and
  // the small hi*lo + lo*hi terms): the tensor core accumulates with truncation, so fewer
  // additions per accumulator keep the sum within 1e-5; they are added (round-to-nearest) in
  // the epilogue. That needs 384 columns, so fp32 mode runs single-buffered.
  static constexpr int kAccBufs = TF32 ? 1 : 2;
  static constexpr int kAccCols = TF32 ? 3 * kBlockN : MB * kTileN;  // per accumulator buffer
  static constexpr int kTmemCols = TF32 ? 512 : 2 * kAccCols;
  static constexpr int kEpiWarps = MB * 4;
  static constexpr int kThreads = (kNumNonEpiWarps + kEpiWarps) * 32;
  static constexpr int kBarBytes = 256;
  static constexpr int kSmemBytes = kStages * kStageBytes + kListBytes + kBarBytes + 1024;
  static_assert(!kSmemList || MB == 1, "shared-memory lists need one query tile per CTA");
  static_assert(!TF32 || MB == 1, "fp32 mode uses one query tile per CTA");
  static_assert(NB == 1 || (MB == 1 && !TF32 && !kSmemList), "wide tiles: one query tile, bf16");
  static_assert(kStages >= 2, "not enough shared memory for the pipeline");
};

__device__ __forceinline__ void resolve_item(const ScanParams& p, int i, ScanItem& it, int qg_size,
                                             int tile_rows = kBlockN) {
  if (p.items != nullptr) {
    it = p.items[i];
    return;
  }
  int qg, r;
  if (p.flags & kFlagRangeMajor) {
    const int nqg = (p.B + qg_size - 1) / qg_size;
    r = i / nqg;
    qg = i - r * nqg;
  } else {
    qg = i / p.R;
    r = i - qg * p.R;
  }
  it.q_begin = qg * qg_size;
  it.q_count = min(qg_size, p.B - it.q_begin);
  const int64_t n = p.row_end - p.row_beg;
  const int64_t tiles = (n + tile_rows - 1) / tile_rows;
  const int64_t t0 = tiles * r / p.R;
  int64_t t1 = tiles * (r + 1) / p.R;
  if (p.sample_div > 1 && t1 > t0) t1 = t0 + (t1 - t0 + p.sample_div - 1) / p.sample_div;
  it.row_begin = p.row_beg + t0 * tile_rows;
  it.row_end = min(p.row_end, p.row_beg + t1 * tile_rows);
  if (it.row_end < it.row_begin) it.row_end = it.row_begin;
  it.out_row = static_cast<int64_t>(r) * p.B + it.q_begin;
  it.id_offset = p.id_offset;
}

// Order-preserving float <-> uint32 keys for the shared admission floor (atomicMax).
__device__ __forceinline__ uint32_t ord_key(float f) {
  const uint32_t u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
// Admission bound for a published k-th score f: admit x >= f, i.e. x > nextafter(f, -inf).
// Key 0 (nothing published yet) admits everything.
__device__ __forceinline__ float floor_admit(uint32_t key) {
  if (key == 0) return -FLT_MAX;
  const float f = __uint_as_float((key & 0x80000000u) ? (key & 0x7fffffffu) : ~key);
  return nextafterf(f, -INFINITY);
}
__device__ __forceinline__ uint32_t floor_load(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}

// Insert (x, xi) into a list sorted by (score desc, id asc). Precondition: x > s[K-1].
// Elements with score >= x keep their place (they were seen earlier, so their ids are
// smaller), the rest shift down one slot and the last one drops out.
template <int K>
__device__ __forceinline__ void list_insert(float (&s)[K], int32_t (&id)[K], float x, int32_t xi) {
#pragma unroll
  for (int i = K - 1; i > 0; --i) {
    const bool keep = s[i] >= x;
    const bool prev_keep = s[i - 1] >= x;
    const float ns = keep ? s[i] : (prev_keep ? x : s[i - 1]);
    const int32_t ni = keep ? id[i] : (prev_keep ? xi : id[i - 1]);
    s[i] = ns;
    id[i] = ni;
  }
  if (!(s[0] >= x)) {
    s[0] = x;
    id[0] = xi;
  }
}

// v[j] for a run-time j via a 5-level tree of constant-index selects: indexing the chunk
// dynamically would spill it to local memory.
__device__ __forceinline__ float pick32(const uint32_t (&v)[32], int j) {
  uint32_t a[16], b[8], c[4], d[2];
#pragma unroll
  for (int i = 0; i < 16; ++i) a[i] = (j & 1) ? v[2 * i + 1] : v[2 * i];
#pragma unroll
  for (int i = 0; i < 8; ++i) b[i] = (j & 2) ? a[2 * i + 1] : a[2 * i];
#pragma unroll
  for (int i = 0; i < 4; ++i) c[i] = (j & 4) ? b[2 * i + 1] : b[2 * i];
#pragma unroll
  for (int i = 0; i < 2; ++i) d[i] = (j & 8) ? c[2 * i + 1] : c[2 * i];
  return __uint_as_float((j & 16) ? d[1] : d[0]);
}

// Candidate bit mask of a 32-score chunk: bit j set iff v[j] > thr and j < valid.
__device__ __forceinline__ uint32_t chunk_mask(const uint32_t (&v)[32], float thr, int valid) {
  uint32_t mask = 0;
#pragma unroll
  for (int j = 0; j < 32; ++j) mask |= (__uint_as_float(v[j]) > thr ? 1u : 0u) << j;
  if (valid < 32) mask &= valid > 0 ? (0xffffffffu >> (32 - valid)) : 0u;
  return mask;
}

__device__ __forceinline__ float chunk_max(const uint32_t (&v)[32]) {
  float m0 = fmaxf(__uint_as_float(v[0]), __uint_as_float(v[1]));
  float m1 = fmaxf(__uint_as_float(v[2]), __uint_as_float(v[3]));
#pragma unroll
  for (int j = 4; j < 32; j += 4) {
    m0 = fmaxf(m0, fmaxf(__uint_as_float(v[j]), __uint_as_float(v[j + 1])));
    m1 = fmaxf(m1, fmaxf(__uint_as_float(v[j + 2]), __uint_as_float(v[j + 3])));
  }
  return fmaxf(m0, m1);
}

// Filter one 32-score chunk (this thread's query x 32 corpus rows) into its register list.
// Common case: one max-reduce and a compare. Rare case (the chunk beats the admission bound
// max(k-th, fl)): a candidate bit mask, then a rolled loop over its set bits in ascending
// row order (so equal scores keep the smaller id first). The rare path is deliberately small:
// a fully unrolled 32-way insertion body per chunk overflows the instruction cache, and with
// 32 queries per warp the "rare" path runs for most chunks of a short scan.
template <int K>
__device__ __forceinline__ void scan_chunk(const uint32_t (&v)[32], float (&s)[K], int32_t (&id)[K],
                                           int32_t id0, int valid, float fl) {
  const float thr = fmaxf(s[K - 1], fl);
  if (chunk_max(v) > thr) {
    uint32_t mask = chunk_mask(v, thr, valid);
    while (mask) {
      const int j = __ffs(mask) - 1;
      mask &= mask - 1;
      const float x = pick32(v, j);
      if (x > fmaxf(s[K - 1], fl)) list_insert<K>(s, id, x, id0 + j);
    }
  }
}

// Candidate (append) mode: every score of the chunk above thr goes to the query's candidate
// row; one atomic per chunk reserves the slots. Same cheap common path as scan_chunk.
__device__ __forceinline__ void scan_chunk_append(const uint32_t (&v)[32], float thr, int32_t id0,
                                                  int valid, int32_t* cnt, float* cs, int32_t* ci,
                                                  int cap) {
  if (chunk_max(v) > thr) {
    uint32_t mask = chunk_mask(v, thr, valid);
    if (mask == 0) return;
    int pos = atomicAdd(cnt, __popc(mask));
    while (mask) {
      const int j = __ffs(mask) - 1;
      mask &= mask - 1;
      if (pos < cap) {
        cs[pos] = pick32(v, j);
        ci[pos] = id0 + j;
      }
      ++pos;
    }
  }
}

// Shared-memory list variant (KCAP > 32), warp-cooperative: the list of query row q is
// ls/li[q * K .. q * K + K) sorted by (score desc, id asc); every lane of a warp holds K/32
// consecutive entries of the list being updated. One candidate is inserted by the whole warp:
// its rank comes from a warp reduction, the tail shifts one slot via a shuffle, and the
// admission threshold of the owner lane (`tau`, the last entry) is refreshed. This replaces a
// K-long dependent chain of shared-memory moves with ~40 warp instructions.
template <int K>
__device__ __forceinline__ float coop_list_insert(float* ls, int32_t* li, int qrow, float x,
                                                  int32_t xi, int lane) {
  constexpr int kPer = K / 32;
  float* rs = ls + qrow * K + lane * kPer;
  int32_t* ri = li + qrow * K + lane * kPer;
  float e[kPer];
  int32_t d[kPer];
#pragma unroll
  for (int i = 0; i < kPer; ++i) {
    e[i] = rs[i];
    d[i] = ri[i];
  }
  int ge = 0;
#pragma unroll
  for (int i = 0; i < kPer; ++i) ge += e[i] >= x ? 1 : 0;
  const int pos = __reduce_add_sync(0xffffffffu, ge);  // entries that stay ahead of x
  const float prev_e = __shfl_up_sync(0xffffffffu, e[kPer - 1], 1);
  const int32_t prev_d = __shfl_up_sync(0xffffffffu, d[kPer - 1], 1);
  float ne[kPer];
  int32_t nd[kPer];
#pragma unroll
  for (int i = 0; i < kPer; ++i) {
    const int g = lane * kPer + i;
    const float below = i == 0 ? prev_e : e[i - 1];
    const int32_t below_d = i == 0 ? prev_d : d[i - 1];
    ne[i] = g < pos ? e[i] : (g == pos ? x : below);
    nd[i] = g < pos ? d[i] : (g == pos ? xi : below_d);
  }
#pragma unroll
  for (int i = 0; i < kPer; ++i) {
    rs[i] = ne[i];
    ri[i] = nd[i];
  }
  return __shfl_sync(0xffffffffu, ne[kPer - 1], 31);  // new last entry = new threshold
}

template <int K>
__device__ __forceinline__ void scan_chunk_coop(const uint32_t (&v)[32], float* ls, int32_t* li,
                                                int row_base, int lane, float& tau, int32_t id0,
                                                int valid, float floor_tau) {
  if (!__any_sync(0xffffffffu, chunk_max(v) > tau)) return;
  uint32_t mask = chunk_mask(v, tau, valid);
  // one candidate per iteration, lowest lane first; each lane's candidates in ascending row
  // order (its list keeps equal scores in id order)
  while (true) {
    const unsigned lanes = __ballot_sync(0xffffffffu, mask != 0);
    if (lanes == 0) break;
    const int src = __ffs(lanes) - 1;
    const int j = (__ffs(mask) - 1) & 31;
    const float x = pick32(v, j);
    if (lane == src) mask &= mask - 1;
    const int js = __shfl_sync(0xffffffffu, j, src);
    const float xs = __shfl_sync(0xffffffffu, x, src);
    const float ts = __shfl_sync(0xffffffffu, tau, src);
    if (xs > ts) {
      const float t_new = coop_list_insert<K>(ls, li, row_base + src, xs, id0 + js, lane);
      if (lane == src) tau = fmaxf(t_new, floor_tau);
    }
  }
}

// After each tile: adopt the best k-th score published by the other ranges of this query
// (`fkey`, loaded before the tile so the L2 latency is hidden) and publish our own once the
// list is full and has improved. `fl` is the admission bound scan_chunk(_coop) applies.
template <int KCAP, bool kSmemList, int kRegK>
__device__ __forceinline__ void share_floor(uint32_t* fslot, uint32_t fkey, const float (&s)[kRegK],
                                            const int32_t (&id)[kRegK], const float* list_s,
                                            const int32_t* list_i, int t_epi, float& fl,
                                            float& tau, float& published) {
  fl = fmaxf(fl, floor_admit(fkey));
  float kth;
  bool full;
  if constexpr (kSmemList) {
    __syncwarp();  // the list tail may have been written by another lane
    kth = list_s[t_epi * KCAP + KCAP - 1];
    full = list_i[t_epi * KCAP + KCAP - 1] >= 0;
    tau = fmaxf(tau, fl);
  } else {
    kth = s[kRegK - 1];
    full = id[kRegK - 1] >= 0;
  }
  if (fslot != nullptr && full && kth > published) {
    atomicMax(fslot, ord_key(kth));
    published = kth;
  }
}

template <int MB, int KCAP, bool TF32, int NB>
__global__ void __launch_bounds__(ScanCfg<MB, KCAP, TF32, NB>::kThreads, 1)
    scan_topk_kernel(const __grid_constant__ CUtensorMap tmap_q,
                     const __grid_constant__ CUtensorMap tmap_c,
                     const __grid_constant__ CUtensorMap tmap_q_lo,
                     const __grid_constant__ CUtensorMap tmap_c_lo, const ScanParams p) {
  using Cfg = ScanCfg<MB, KCAP, TF32, NB>;
  constexpr int kTileN = Cfg::kTileN;
  constexpr int kElemsPerKb = TF32 ? 32 : kBlockK;  // elements per 128-byte k-block row
  constexpr int kStages = Cfg::kStages;
  constexpr int kQG = MB * kBlockM;
  constexpr bool kSmemList = Cfg::kSmemList;
  constexpr bool kAppend = KCAP == kAppendCap;
  constexpr int kRegK = (kSmemList || kAppend) ? 1 : KCAP;
  if (threadIdx.x == 0) pdl_allow_dependents();

  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  float* list_s = reinterpret_cast<float*>(smem + kStages * Cfg::kStageBytes);
  int32_t* list_i = reinterpret_cast<int32_t*>(list_s + (kSmemList ? KCAP * kBlockM : 0));
  uint64_t* full_bar =
      reinterpret_cast<uint64_t*>(smem + kStages * Cfg::kStageBytes + Cfg::kListBytes);
  uint64_t* empty_bar = full_bar + kStages;
  uint64_t* tfull_bar = empty_bar + kStages;
  uint64_t* tempty_bar = tfull_bar + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_bar + 2);

  // shfl makes the warp index provably warp-uniform, so role branches are not divergent and
  // the producer / MMA loops keep their operands in uniform registers.
  const int warp = __shfl_sync(0xffffffffu, static_cast<int>(threadIdx.x >> 5), 0);
  const int lane = threadIdx.x & 31;

  if (warp == 0 && lane == 0) {
    ptx::tma_prefetch_desc(&tmap_q);
    ptx::tma_prefetch_desc(&tmap_c);
    for (int s = 0; s < kStages; ++s) {
      ptx::mbar_init(&full_bar[s], 1);
      ptx::mbar_init(&empty_bar[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      ptx::mbar_init(&tfull_bar[b], 1);
      ptx::mbar_init(&tempty_bar[b], Cfg::kEpiWarps * 32);
    }
    ptx::fence_mbar_init();
  }
  if (warp == 2) {
    ptx::tmem_alloc(tmem_slot, Cfg::kTmemCols);
    ptx::tmem_relinquish();
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  // Launched with programmatic stream serialisation: the setup above (barriers, TMEM, descriptor
  // prefetch) overlaps the tail of the kernel before (the query staging, a merge); from here on
  // its outputs (queries, floors, the gate) are visible.
  pdl_wait();
  const bool gated_off = p.gate != nullptr && *p.gate == 0;  // device-side skip (no host trip)

  const int num_items = ((p.flags & kFlagDiagSetupOnly) || gated_off) ? 0 : p.num_items;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    // The whole warp walks the loop (warp-uniform operands); one elected lane issues.
    const uint64_t pol_q = ptx::policy_evict_last();
    const uint64_t pol_c = ptx::policy_evict_normal();
    int stage = 0;
    uint32_t phase = 0;
    // range lockstep between the CTAs that stream the same corpus range (see the pair kernel)
    const bool lockstep = (p.flags & kFlagLockstep) && p.items == nullptr &&
                          num_items <= static_cast<int>(gridDim.x);
    volatile int32_t* progress = p.counter;
    const uint32_t stage_tx = (!TF32 && p.a_rows > 0)
                                  ? static_cast<uint32_t>(MB * p.a_rows * 128 + Cfg::kBBytes)
                                  : static_cast<uint32_t>(Cfg::kStageBytes);
    for (int i = blockIdx.x; i < num_items; i += gridDim.x) {
      ScanItem it;
      resolve_item(p, i, it, kQG, kTileN);
      const int64_t ntiles = (it.row_end - it.row_begin + kTileN - 1) / kTileN;
      const int my_qg = p.R > 0 ? i / p.R : 0, my_r = p.R > 0 ? i - my_qg * p.R : 0;
      const int nqg = p.R > 0 ? num_items / p.R : 1;
      bool lock_live = lockstep;  // cleared when a partner is not progressing (see below)
      for (int64_t t = 0; t < ntiles; ++t) {
        if (lockstep && lane == 0) {
          if ((t & 3) == 0) progress[i] = static_cast<int32_t>(t);
          if (lock_live && t >= 2 * kLockWindow) {
            for (int g = 0; g < nqg && lock_live; ++g)
              if (g != my_qg)
                lock_live = lock_wait(progress + g * p.R + my_r, t - 2 * kLockWindow);
          }
        }
        __syncwarp();
        const int32_t row0 = static_cast<int32_t>(it.row_begin + t * kTileN);
        for (int kb = 0; kb < p.num_kb; ++kb) {
          ptx::mbar_wait(&empty_bar[stage], phase ^ 1);
          uint8_t* st = smem + stage * Cfg::kStageBytes;
          ptx::mbar_arrive_expect_tx_warp(&full_bar[stage], stage_tx);
#pragma unroll
          for (int mb = 0; mb < MB; ++mb)
            ptx::tma_load_2d_warp(st + mb * Cfg::kABytes, &tmap_q, &full_bar[stage],
                                  kb * kElemsPerKb, it.q_begin + mb * kBlockM, pol_q);
#pragma unroll
          for (int h = 0; h < NB; ++h) {  // 128-row corpus boxes, stacked along N
            uint8_t* dst = st + MB * Cfg::kABytes + h * (kBlockN * 128);
            if (p.flags & kFlagTiled)  // row0 is a multiple of 128 in the tiled layout
              ptx::tma_load_3d_warp(dst, &tmap_c, &full_bar[stage], 0, 0,
                                    ((row0 >> 7) + h) * p.num_kb + kb, pol_c);
            else
              ptx::tma_load_2d_warp(dst, &tmap_c, &full_bar[stage], kb * kElemsPerKb,
                                    row0 + h * kBlockN, pol_c);
          }
          if constexpr (TF32) {  // lo planes follow the hi planes in the stage
            uint8_t* lo = st + MB * Cfg::kABytes + Cfg::kBBytes;
            ptx::tma_load_2d_warp(lo, &tmap_q_lo, &full_bar[stage], kb * kElemsPerKb,
                                  it.q_begin, pol_q);
            ptx::tma_load_2d_warp(lo + Cfg::kABytes, &tmap_c_lo, &full_bar[stage],
                                  kb * kElemsPerKb, row0, pol_c);
          }
          if (++stage == kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
      if (lockstep && lane == 0) progress[i] = 0x7fffffff;
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    // Warp-uniform loop; descriptors are built from the smem base plus compile-time offsets.
    constexpr uint32_t idesc = ptx::idesc_bf16_f32(kBlockM, kTileN);
    constexpr uint32_t idesc_tf32 = ptx::idesc_tf32_f32(kBlockM, kBlockN);
    const uint64_t desc0 = ptx::umma_desc_sw128(ptx::smem_u32(smem));
    int stage = 0;
    uint32_t phase = 0;
    int abuf = 0;
    uint32_t aphase = 0;
    for (int i = blockIdx.x; i < num_items; i += gridDim.x) {
      ScanItem it;
      resolve_item(p, i, it, kQG, kTileN);
      const int64_t ntiles = (it.row_end - it.row_begin + kTileN - 1) / kTileN;
      for (int64_t t = 0; t < ntiles; ++t) {
        ptx::mbar_wait(&tempty_bar[abuf], aphase ^ 1);
        ptx::tc_fence_after();
        const uint32_t d0 = tmem_base + abuf * Cfg::kAccCols;
        for (int kb = 0; kb < p.num_kb; ++kb) {
          ptx::mbar_wait(&full_bar[stage], phase);
          ptx::tc_fence_after();
          const uint64_t sdesc = desc0 + static_cast<uint64_t>((stage * Cfg::kStageBytes) >> 4);
          if constexpr (TF32) {
            // 3xTF32: hi*hi + hi*lo + lo*hi, each K=8 fp32 (32 bytes) per instruction
            const uint64_t a_hi = sdesc;
            const uint64_t b_hi = sdesc + static_cast<uint64_t>(Cfg::kABytes >> 4);
            const uint64_t a_lo = sdesc + static_cast<uint64_t>((Cfg::kABytes + Cfg::kBBytes) >> 4);
            const uint64_t b_lo = a_lo + static_cast<uint64_t>(Cfg::kABytes >> 4);
            const uint32_t d_main = d0 + (kb & 1) * kBlockN;
            const uint32_t d_small = d0 + 2 * kBlockN;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              ptx::mma_tf32_ss_warp(d_main, a_hi + 2 * k, b_hi + 2 * k, idesc_tf32,
                                    ((kb >> 1) | k) != 0 ? 1u : 0u);
              ptx::mma_tf32_ss_warp(d_small, a_hi + 2 * k, b_lo + 2 * k, idesc_tf32,
                                    (kb | k) != 0 ? 1u : 0u);
              ptx::mma_tf32_ss_warp(d_small, a_lo + 2 * k, b_hi + 2 * k, idesc_tf32, 1u);
            }
          } else {
#pragma unroll
          for (int k = 0; k < kBlockK / 16; ++k) {
#pragma unroll
            for (int mb = 0; mb < MB; ++mb) {
              ptx::mma_f16_ss_warp(d0 + mb * kTileN,
                                   sdesc + static_cast<uint64_t>((mb * Cfg::kABytes) >> 4) + 2 * k,
                                   sdesc + static_cast<uint64_t>((MB * Cfg::kABytes) >> 4) + 2 * k,
                                   idesc, (kb | k) != 0 ? 1u : 0u);
            }
          }
          }
          ptx::mma_commit_warp(&empty_bar[stage]);
          if (++stage == kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
        ptx::mma_commit_warp(&tfull_bar[abuf]);
        if (++abuf == Cfg::kAccBufs) {
          abuf = 0;
          aphase ^= 1;
        }
      }
    }
  } else if (warp >= kNumNonEpiWarps) {
    // ------------------------------------------------------------ epilogue
    const int e = warp - kNumNonEpiWarps;
    const int quad = warp & 3;          // TMEM lane quadrant this warp may access
    const int mb = e >> 2;              // which query tile of the group
    const int lq = mb * kBlockM + quad * 32 + lane;  // local query index within the item
    const uint32_t lane_addr = tmem_base + (static_cast<uint32_t>(quad * 32) << 16) + mb * kTileN;
    int abuf = 0;
    uint32_t aphase = 0;
    for (int i = blockIdx.x; i < num_items; i += gridDim.x) {
      ScanItem it;
      resolve_item(p, i, it, kQG, kTileN);
      float s[kRegK];
      int32_t id[kRegK];
      const int t_epi = quad * 32 + lane;  // row of this thread's shared-memory list
      // Padding query rows (lq >= q_count: the last group of a batch that is not a multiple of
      // the tile) admit nothing, so their lanes never enter the insertion paths that the
      // real lanes of the warp would otherwise wait for.
      const float tau_floor = lq >= it.q_count ? INFINITY
                              : (p.tau0 != nullptr ? p.tau0[it.q_begin + lq] : -FLT_MAX);
      float tau = tau_floor;
      uint32_t* const fslot =
          (p.floor_g != nullptr && lq < it.q_count) ? p.floor_g + it.q_begin + lq : nullptr;
      float fl = tau_floor, published = -FLT_MAX;
      // append mode: admit scores above tau0 (padding query rows admit nothing)
      const float athr = tau_floor;
      const int64_t qrow = static_cast<int64_t>(it.q_begin) + (lq < it.q_count ? lq : 0);
      int32_t* const ccnt = kAppend ? p.cand_count + qrow : nullptr;
      float* const cbs = kAppend ? p.out_scores + qrow * p.cand_cap : nullptr;
      int32_t* const cbi = kAppend ? p.out_ids + qrow * p.cand_cap : nullptr;
#pragma unroll
      for (int j = 0; j < kRegK; ++j) {
        s[j] = -FLT_MAX;
        id[j] = -1;
      }
      if constexpr (kSmemList) {
        for (int j = 0; j < KCAP; ++j) {
          list_s[t_epi * KCAP + j] = -FLT_MAX;
          list_i[t_epi * KCAP + j] = -1;
        }
        __syncwarp();
      }
      const int64_t ntiles = (it.row_end - it.row_begin + kTileN - 1) / kTileN;
      for (int64_t t = 0; t < ntiles; ++t) {
        const int64_t row0 = it.row_begin + t * kTileN;
        const int valid = static_cast<int>(it.row_end - row0 < kTileN ? it.row_end - row0 : kTileN);
        const int32_t id0 = static_cast<int32_t>(row0) + it.id_offset;
        const uint32_t fkey = fslot != nullptr ? floor_load(fslot) : 0u;  // used after this tile
        ptx::mbar_wait(&tfull_bar[abuf], aphase);
        ptx::tc_fence_after();
        const uint32_t taddr = lane_addr + abuf * Cfg::kAccCols;
        if constexpr (TF32) {
          // score = even-k hi*hi + odd-k hi*hi + (hi*lo + lo*hi), added round-to-nearest
#pragma unroll 1
          for (int c = 0; c < kBlockN; c += 32) {
            uint32_t va[32], vb[32], vc[32];
            ptx::tmem_ld_32x32b_x32(taddr + c, va);
            ptx::tmem_ld_32x32b_x32(taddr + kBlockN + c, vb);
            ptx::tmem_ld_32x32b_x32(taddr + 2 * kBlockN + c, vc);
            ptx::tmem_ld_wait();
            // With one k-block the odd-k accumulator is never written: its TMEM columns hold
            // whatever an earlier kernel left there (possibly NaN), so it is skipped by a select,
            // not multiplied by 0 (0 * NaN = NaN: the first fp32-mode search of a 16..32-dim index
            // after other tensor-core kernels admitted nothing).
            const bool has_odd = p.num_kb > 1;
#pragma unroll
            for (int j = 0; j < 32; ++j)
              va[j] = __float_as_uint(__uint_as_float(va[j]) + (has_odd ? __uint_as_float(vb[j]) : 0.f) +
                                      __uint_as_float(vc[j]));
            if constexpr (kSmemList)
              scan_chunk_coop<KCAP>(va, list_s, list_i, quad * 32, lane, tau, id0 + c, valid - c,
                                  fl);
            else
              scan_chunk<kRegK>(va, s, id, id0 + c, valid - c, fl);
          }
        } else {
#pragma unroll 1
        for (int c = 0; c < kTileN; c += 64) {
          uint32_t va[32], vb[32];
          ptx::tmem_ld_32x32b_x32(taddr + c, va);
          ptx::tmem_ld_32x32b_x32(taddr + c + 32, vb);
          ptx::tmem_ld_wait();
          if constexpr (kAppend) {
            scan_chunk_append(va, athr, id0 + c, valid - c, ccnt, cbs, cbi, p.cand_cap);
            scan_chunk_append(vb, athr, id0 + c + 32, valid - c - 32, ccnt, cbs, cbi, p.cand_cap);
          } else if constexpr (kSmemList) {
            scan_chunk_coop<KCAP>(va, list_s, list_i, quad * 32, lane, tau, id0 + c, valid - c,
                                  fl);
            scan_chunk_coop<KCAP>(vb, list_s, list_i, quad * 32, lane, tau, id0 + c + 32,
                                  valid - c - 32, fl);
          } else {
            scan_chunk<kRegK>(va, s, id, id0 + c, valid - c, fl);
            scan_chunk<kRegK>(vb, s, id, id0 + c + 32, valid - c - 32, fl);
          }
        }
        }
        ptx::tc_fence_before();
        ptx::mbar_arrive(&tempty_bar[abuf]);
        if (p.floor_g != nullptr)  // warp-uniform (the smem-list variant syncs the warp)
          share_floor<KCAP, kSmemList>(fslot, fkey, s, id, list_s, list_i, t_epi, fl, tau,
                                       published);
        if (++abuf == Cfg::kAccBufs) {
          abuf = 0;
          aphase ^= 1;
        }
      }
      if (!kAppend && lq < it.q_count) {
        float* os = p.out_scores + (it.out_row + lq) * p.out_k;
        int32_t* oi = p.out_ids + (it.out_row + lq) * p.out_k;
        if constexpr (kSmemList) {
          for (int j = 0; j < p.out_k; ++j) {
            const int32_t v = list_i[t_epi * KCAP + j];
            os[j] = v < 0 ? -INFINITY : list_s[t_epi * KCAP + j];
            oi[j] = v < 0 ? -1 : v;
          }
        } else {
#pragma unroll
          for (int j = 0; j < kRegK; ++j) {
            if (j < p.out_k) {
              const bool pad = id[j] < 0;
              os[j] = pad ? -INFINITY : s[j];
              oi[j] = pad ? -1 : id[j];
            }
          }
        }
      }
    }
  }

  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem_base, Cfg::kTmemCols);
  }
}

// ---------------------------------------------------------------------------------------------
// CTA-pair variant (cta_group::2). A pair of SMs computes M=256 queries x N=256 corpus rows per
// MMA: each CTA stages its 128 query rows and 128 corpus rows of every k-block, the leader CTA
// issues tcgen05.mma.cta_group::2 and each CTA's TMEM receives its own 128 query rows x 256
// columns. Per SM this halves the shared-memory operand bytes per MAC compared with the
// single-CTA 128x128 tile, which is what keeps the tensor pipe fed.
struct Pair {
  static constexpr int kTileRows = 256;                 // corpus rows per pair tile (N)
  static constexpr int kQG = 256;                       // queries per pair (M)
  static constexpr int kHalfBytes = 128 * kBlockK * 2;  // 16 KB: one CTA's half of A or B
  static constexpr int kAccCols = 256;
  static constexpr int kTmemCols = 512;                 // 2 accumulator buffers
  static constexpr int kEpiWarps = 4;
  static constexpr int kThreads = (kNumNonEpiWarps + kEpiWarps) * 32;
};

// Operand rings of the pair kernel: the query operand (A, L2-resident) and the corpus operand
// (B, streamed from HBM) have separate rings of 16 KB half-stages, each fed by its own producer
// warp, so the corpus ring runs kB k-blocks ahead independently of the short-latency query ring.
template <int KCAP>
struct PairStages {
  static constexpr int kListBytes = KCAP > kRegListMax ? 128 * KCAP * 8 : 0;
  static constexpr int kBarBytes = 512;
  static constexpr int kHalves = (227 * 1024 - 1024 - kBarBytes - kListBytes) / Pair::kHalfBytes;
  static constexpr int kA = kHalves >= 12 ? 4 : kHalves / 2;  // query k-blocks in flight
  static constexpr int kB = kHalves - kA;                      // corpus k-blocks in flight
  static constexpr int smem = kHalves * Pair::kHalfBytes + kListBytes + kBarBytes + 1024;
  static_assert(kA >= 2 && kB >= 2, "pair kernel: not enough shared memory for the rings");
  static_assert(2 * (kA + kB) * 8 + 4 * 8 + 16 <= kBarBytes, "pair kernel: barrier area");
};

template <int KCAP>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(Pair::kThreads, 1)
    scan_topk_pair_kernel(const __grid_constant__ CUtensorMap tmap_q,
                          const __grid_constant__ CUtensorMap tmap_c, const ScanParams p) {
  // k > 32: warp-cooperative lists in shared memory (128 query rows x KCAP), fewer stages
  constexpr bool kSmemList = KCAP > kRegListMax;
  using St = PairStages<KCAP>;
  constexpr int kListBytes = St::kListBytes;
  constexpr int kA = St::kA, kB = St::kB;
  constexpr bool kAppend = KCAP == kAppendCap;
  constexpr int kRegK = (kSmemList || kAppend) ? 1 : KCAP;
  if (threadIdx.x == 0) pdl_allow_dependents();
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint8_t* ring_a = smem;                                  // kA x [128 query rows x 64]
  uint8_t* ring_b = smem + kA * Pair::kHalfBytes;          // kB x [128 corpus rows x 64]
  float* list_s = reinterpret_cast<float*>(smem + St::kHalves * Pair::kHalfBytes);
  int32_t* list_i = reinterpret_cast<int32_t*>(list_s + (kSmemList ? 128 * KCAP : 0));
  uint64_t* fullA = reinterpret_cast<uint64_t*>(smem + St::kHalves * Pair::kHalfBytes + kListBytes);
  uint64_t* emptyA = fullA + kA;
  uint64_t* fullB = emptyA + kA;
  uint64_t* emptyB = fullB + kB;
  uint64_t* tfull_bar = emptyB + kB;
  uint64_t* tempty_bar = tfull_bar + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_bar + 2);

  const int warp = __shfl_sync(0xffffffffu, static_cast<int>(threadIdx.x >> 5), 0);
  const int lane = threadIdx.x & 31;
  const uint32_t rank = ptx::cluster_ctarank();
  const bool leader = rank == 0;
  const int pair = blockIdx.x >> 1;
  const int npairs = gridDim.x >> 1;

  if (warp == 0 && lane == 0) {
    ptx::tma_prefetch_desc(&tmap_q);
    ptx::tma_prefetch_desc(&tmap_c);
    for (int s = 0; s < kA; ++s) {
      ptx::mbar_init(&fullA[s], 1);
      ptx::mbar_init(&emptyA[s], 1);
    }
    for (int s = 0; s < kB; ++s) {
      ptx::mbar_init(&fullB[s], 1);
      ptx::mbar_init(&emptyB[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      ptx::mbar_init(&tfull_bar[b], 1);
      ptx::mbar_init(&tempty_bar[b], 2 * Pair::kEpiWarps);  // one arrival per epilogue warp
    }
    ptx::fence_mbar_init();
  }
  if (warp == 2) {
    ptx::tmem_alloc2(tmem_slot, Pair::kTmemCols);
    ptx::tmem_relinquish2();
  }
  ptx::tc_fence_before();
  ptx::cluster_sync();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  pdl_wait();  // (see scan_topk_kernel) the previous kernel's outputs are visible from here
  const bool gated_off = p.gate != nullptr && *p.gate == 0;
  const int num_items = gated_off ? 0 : p.num_items;

  if (warp == 3) {
    // ---- query producer (both CTAs): own half of A per k-block, completion on the leader
    const uint64_t pol_q = ptx::policy_evict_last();
    int stage = 0;
    uint32_t phase = 0;
    for (int i = pair; i < num_items; i += npairs) {
      ScanItem it;
      resolve_item(p, i, it, Pair::kQG, Pair::kTileRows);
      const int64_t ntiles = (it.row_end - it.row_begin + Pair::kTileRows - 1) / Pair::kTileRows;
      for (int64_t t = 0; t < ntiles; ++t) {
        const bool skip_a = (p.flags & kFlagDiagNoQueryLoad) && t > 0;
        for (int kb = 0; kb < p.num_kb; ++kb) {
          ptx::mbar_wait(&emptyA[stage], phase ^ 1);
          const uint32_t fb = ptx::mapa(ptx::smem_u32(&fullA[stage]), 0);
          if (leader) ptx::mbar_arrive_expect_tx_warp(&fullA[stage], skip_a ? 0 : 2 * Pair::kHalfBytes);
          if (!skip_a)
            ptx::tma_load_2d_pair_warp(ring_a + stage * Pair::kHalfBytes, &tmap_q, fb, kb * kBlockK,
                                       it.q_begin + rank * 128, pol_q);
          if (++stage == kA) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 0) {
    // ---- corpus producer (both CTAs): own half of B per k-block, completion on the leader
    const uint64_t pol_c = ptx::policy_evict_normal();
    int stage = 0;
    uint32_t phase = 0;
    // Range lockstep (flag bit 2): the pairs that stream the same corpus range for different
    // query groups publish their tile progress and none runs more than kLockWindow tiles ahead,
    // so each corpus tile is fetched from HBM once and served to the others from L2.
    // With range-major items several rounds are allowed: partners are the items of the same
    // range in the same round (a partner of a later round has not started and must not be
    // waited for).
    const bool range_major = (p.flags & kFlagRangeMajor) != 0;
    const bool lockstep = (p.flags & kFlagLockstep) && p.items == nullptr &&
                          (num_items <= npairs || range_major);
    volatile int32_t* progress = p.counter;
    for (int i = pair; i < num_items; i += npairs) {
      ScanItem it;
      resolve_item(p, i, it, Pair::kQG, Pair::kTileRows);
      const int64_t ntiles = (it.row_end - it.row_begin + Pair::kTileRows - 1) / Pair::kTileRows;
      const int nqg = range_major ? (p.B + Pair::kQG - 1) / Pair::kQG : num_items / p.R;
      const int my_qg = range_major ? i % nqg : i / p.R;
      const int my_r = range_major ? i / nqg : i - my_qg * p.R;
      const int round = i / npairs;
      bool lock_live = lockstep;  // cleared when a partner is not progressing (see below)
      for (int64_t t = 0; t < ntiles; ++t) {
        if (lockstep && leader && lane == 0) {
          const int w = p.lock_window > 0 ? p.lock_window : kLockWindow;
          if ((t & 1) == 0) progress[i] = static_cast<int32_t>(t);
          if (lock_live && t >= w) {
            for (int g = 0; g < nqg && lock_live; ++g) {
              if (g == my_qg) continue;
              const int j = range_major ? my_r * nqg + g : g * p.R + my_r;
              if (j / npairs != round) continue;
              lock_live = lock_wait(progress + j, t - w);
            }
          }
        }
        __syncwarp();
        const int64_t tt = (p.flags & kFlagDiagNoStream) ? 0 : t;
        const int32_t row0 = static_cast<int32_t>(it.row_begin + tt * Pair::kTileRows) + rank * 128;
        for (int kb = 0; kb < p.num_kb; ++kb) {
          ptx::mbar_wait(&emptyB[stage], phase ^ 1);
          uint8_t* st = ring_b + stage * Pair::kHalfBytes;
          const uint32_t fb = ptx::mapa(ptx::smem_u32(&fullB[stage]), 0);
          if (leader) ptx::mbar_arrive_expect_tx_warp(&fullB[stage], 2 * Pair::kHalfBytes);
          if (p.flags & kFlagTiled)
            ptx::tma_load_3d_pair_warp(st, &tmap_c, fb, 0, 0, (row0 >> 7) * p.num_kb + kb, pol_c);
          else
            ptx::tma_load_2d_pair_warp(st, &tmap_c, fb, kb * kBlockK, row0, pol_c);
          if (++stage == kB) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
      if (lockstep && leader && lane == 0) progress[i] = 0x7fffffff;  // range done
    }
  } else if (warp == 1) {
    // ---- MMA issuer (leader CTA only)
    if (leader) {
      constexpr uint32_t idesc = ptx::idesc_bf16_f32(256, 256);
      const uint64_t descA0 = ptx::umma_desc_sw128(ptx::smem_u32(ring_a));
      const uint64_t descB0 = ptx::umma_desc_sw128(ptx::smem_u32(ring_b));
      int sa = 0, sb = 0;
      uint32_t pa = 0, pb = 0;
      int abuf = 0;
      uint32_t aphase = 0;
      for (int i = pair; i < num_items; i += npairs) {
        ScanItem it;
        resolve_item(p, i, it, Pair::kQG, Pair::kTileRows);
        const int64_t ntiles = (it.row_end - it.row_begin + Pair::kTileRows - 1) / Pair::kTileRows;
        for (int64_t t = 0; t < ntiles; ++t) {
          ptx::mbar_wait(&tempty_bar[abuf], aphase ^ 1);
          ptx::tc_fence_after();
          const uint32_t d0 = tmem_base + abuf * Pair::kAccCols;
          for (int kb = 0; kb < p.num_kb; ++kb) {
            ptx::mbar_wait(&fullA[sa], pa);
            ptx::mbar_wait(&fullB[sb], pb);
            ptx::tc_fence_after();
            const uint64_t adesc = descA0 + static_cast<uint64_t>((sa * Pair::kHalfBytes) >> 4);
            const uint64_t bdesc = descB0 + static_cast<uint64_t>((sb * Pair::kHalfBytes) >> 4);
#pragma unroll
            for (int k = 0; k < kBlockK / 16; ++k)
              ptx::mma2_f16_ss_warp(d0, adesc + 2 * k, bdesc + 2 * k, idesc,
                                    (kb | k) != 0 ? 1u : 0u);
            ptx::mma2_commit_mc_warp(&emptyA[sa], 0x3);
            ptx::mma2_commit_mc_warp(&emptyB[sb], 0x3);
            if (++sa == kA) {
              sa = 0;
              pa ^= 1;
            }
            if (++sb == kB) {
              sb = 0;
              pb ^= 1;
            }
          }
          ptx::mma2_commit_mc_warp(&tfull_bar[abuf], 0x3);
          abuf ^= 1;
          if (abuf == 0) aphase ^= 1;
        }
      }
    }
  } else if (warp >= kNumNonEpiWarps) {
    // ---- epilogue (both CTAs): thread = one query row of this CTA's 128, 256 columns per tile
    const int quad = warp & 3;
    const int lq = static_cast<int>(rank) * 128 + quad * 32 + lane;
    const uint32_t lane_addr = tmem_base + (static_cast<uint32_t>(quad * 32) << 16);
    const uint32_t tempty_leader0 = ptx::mapa(ptx::smem_u32(&tempty_bar[0]), 0);
    int abuf = 0;
    uint32_t aphase = 0;
    for (int i = pair; i < num_items; i += npairs) {
      ScanItem it;
      resolve_item(p, i, it, Pair::kQG, Pair::kTileRows);
      float s[kRegK];
      int32_t id[kRegK];
      const int t_epi = quad * 32 + lane;
      // Padding query rows (lq >= q_count: the last group of a batch that is not a multiple of
      // the tile) admit nothing, so their lanes never enter the insertion paths that the
      // real lanes of the warp would otherwise wait for.
      const float tau_floor = lq >= it.q_count ? INFINITY
                              : (p.tau0 != nullptr ? p.tau0[it.q_begin + lq] : -FLT_MAX);
      float tau = tau_floor;
      uint32_t* const fslot =
          (p.floor_g != nullptr && lq < it.q_count) ? p.floor_g + it.q_begin + lq : nullptr;
      float fl = tau_floor, published = -FLT_MAX;
      // append mode: admit scores above tau0 (padding query rows admit nothing)
      const float athr = tau_floor;
      const int64_t qrow = static_cast<int64_t>(it.q_begin) + (lq < it.q_count ? lq : 0);
      int32_t* const ccnt = kAppend ? p.cand_count + qrow : nullptr;
      float* const cbs = kAppend ? p.out_scores + qrow * p.cand_cap : nullptr;
      int32_t* const cbi = kAppend ? p.out_ids + qrow * p.cand_cap : nullptr;
#pragma unroll
      for (int j = 0; j < kRegK; ++j) {
        s[j] = -FLT_MAX;
        id[j] = -1;
      }
      if constexpr (kSmemList) {
        for (int j = 0; j < KCAP; ++j) {
          list_s[t_epi * KCAP + j] = -FLT_MAX;
          list_i[t_epi * KCAP + j] = -1;
        }
        __syncwarp();
      }
      const int64_t ntiles = (it.row_end - it.row_begin + Pair::kTileRows - 1) / Pair::kTileRows;
      for (int64_t t = 0; t < ntiles; ++t) {
        const int64_t row0 = it.row_begin + t * Pair::kTileRows;
        const int valid = static_cast<int>(
            it.row_end - row0 < Pair::kTileRows ? it.row_end - row0 : Pair::kTileRows);
        const int32_t id0 = static_cast<int32_t>(row0) + it.id_offset;
        const uint32_t fkey = fslot != nullptr ? floor_load(fslot) : 0u;  // used after this tile
        ptx::mbar_wait(&tfull_bar[abuf], aphase);
        ptx::tc_fence_after();
        const uint32_t taddr = lane_addr + abuf * Pair::kAccCols;
        const bool diag_nofilter = (p.flags & kFlagDiagNoFilter) != 0;
        auto consume = [&](uint32_t (&v)[32], int col) {
          if (diag_nofilter) return;
          if constexpr (kAppend)
            scan_chunk_append(v, athr, id0 + col, valid - col, ccnt, cbs, cbi, p.cand_cap);
          else if constexpr (kSmemList)
            scan_chunk_coop<KCAP>(v, list_s, list_i, quad * 32, lane, tau, id0 + col,
                                  valid - col, fl);
          else
            scan_chunk<kRegK>(v, s, id, id0 + col, valid - col, fl);
        };
        // Ping-pong over 32-column chunks: the next chunk's tcgen05.ld is in flight while the
        // current one is filtered, so the TMEM load latency is off the epilogue's critical
        // path (it bounds the tile rate when D is small and the MMA per tile is short).
        uint32_t va[32], vb[32];
        ptx::tmem_ld_32x32b_x32(taddr, va);
        ptx::tmem_ld_wait();
        ptx::tmem_regs_ready(va);
#pragma unroll 1
        for (int c = 0; c < Pair::kTileRows; c += 64) {
          ptx::tmem_ld_32x32b_x32(taddr + c + 32, vb);
          consume(va, c);
          ptx::tmem_ld_wait();
          ptx::tmem_regs_ready(vb);
          if (c + 64 < Pair::kTileRows) ptx::tmem_ld_32x32b_x32(taddr + c + 64, va);
          consume(vb, c + 32);
          ptx::tmem_ld_wait();
          ptx::tmem_regs_ready(va);
        }
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive_remote(tempty_leader0 + abuf * 8);
        if (p.floor_g != nullptr)  // warp-uniform (the smem-list variant syncs the warp)
          share_floor<KCAP, kSmemList>(fslot, fkey, s, id, list_s, list_i, t_epi, fl, tau,
                                       published);
        abuf ^= 1;
        if (abuf == 0) aphase ^= 1;
      }
      if (!kAppend && lq < it.q_count) {
        float* os = p.out_scores + (it.out_row + lq) * p.out_k;
        int32_t* oi = p.out_ids + (it.out_row + lq) * p.out_k;
        if constexpr (kSmemList) {
          for (int j = 0; j < p.out_k; ++j) {
            const int32_t v = list_i[t_epi * KCAP + j];
            os[j] = v < 0 ? -INFINITY : list_s[t_epi * KCAP + j];
            oi[j] = v < 0 ? -1 : v;
          }
        } else {
#pragma unroll
          for (int j = 0; j < kRegK; ++j) {
            if (j < p.out_k) {
              const bool pad = id[j] < 0;
              os[j] = pad ? -INFINITY : s[j];
              oi[j] = pad ? -1 : id[j];
            }
          }
        }
      }
    }
  }

  ptx::tc_fence_before();
  ptx::cluster_sync();
  if (warp == 2) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc2(tmem_base, Pair::kTmemCols);
  }
}

// Scan launches use programmatic stream serialisation (PDL): the kernel may start while the
// previous kernel of the stream (query staging, a merge, the seed floor) is finishing and waits
// for its results in griddepcontrol.wait after its own setup. TSV_NO_PDL=1 launches normally.
template <typename... KArgs, typename... Args>
int launch_scan_pdl(void (*kern)(KArgs...), int grid, int threads, int smem, cudaStream_t stream,
                    Args&&... args) {
  static const bool no_pdl = getenv("TSV_NO_PDL") != nullptr && getenv("TSV_NO_PDL")[0] == '1';
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = no_pdl ? 0 : 1;
  return static_cast<int>(cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...));
}

template <int KCAP>
int launch_pair_impl(const CUtensorMap& tq, const CUtensorMap& tc, const ScanParams& p, int grid,
                     cudaStream_t stream) {
  auto kern = scan_topk_pair_kernel<KCAP>;
  constexpr int smem = PairStages<KCAP>::smem;
  static std::atomic<uint64_t> configured{0};
  if (first_on_device(configured)) {
    cudaError_t err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (err != cudaSuccess) return static_cast<int>(err);
  }
  return launch_scan_pdl(kern, grid, Pair::kThreads, smem, stream, tq, tc, p);
}

template <int MB, int KCAP, bool TF32 = false, int NB = 1>
int launch_impl(const CUtensorMap& tq, const CUtensorMap& tc, const ScanParams& p, int grid,
                cudaStream_t stream, const CUtensorMap* tq_lo = nullptr,
                const CUtensorMap* tc_lo = nullptr) {
  using Cfg = ScanCfg<MB, KCAP, TF32, NB>;
  auto kern = scan_topk_kernel<MB, KCAP, TF32, NB>;
  static std::atomic<uint64_t> configured{0};  // per instantiation and device
  if (first_on_device(configured)) {
    cudaError_t err =
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::kSmemBytes);
    if (err != cudaSuccess) return static_cast<int>(err);
  }
  return launch_scan_pdl(kern, grid, Cfg::kThreads, Cfg::kSmemBytes, stream, tq, tc,
                         tq_lo ? *tq_lo : tq, tc_lo ? *tc_lo : tc, p);
}

template <int MB>
int dispatch_kcap(int kcap, const CUtensorMap& tq, const CUtensorMap& tc, const ScanParams& p,
                  int grid, cudaStream_t stream) {
  switch (kcap) {
    case kAppendCap:
      if constexpr (MB == 1) return launch_impl<1, kAppendCap>(tq, tc, p, grid, stream);
      return static_cast<int>(cudaErrorInvalidValue);
    case 1: return launch_impl<MB, 1>(tq, tc, p, grid, stream);
    case 4: return launch_impl<MB, 4>(tq, tc, p, grid, stream);
    case 8: return launch_impl<MB, 8>(tq, tc, p, grid, stream);
    case 10: return launch_impl<MB, 10>(tq, tc, p, grid, stream);
    case 16: return launch_impl<MB, 16>(tq, tc, p, grid, stream);
    case 32: return launch_impl<MB, 32>(tq, tc, p, grid, stream);
    case 64:
      if constexpr (MB == 1) return launch_impl<1, 64>(tq, tc, p, grid, stream);
      return static_cast<int>(cudaErrorInvalidValue);
    case 128:
      if constexpr (MB == 1) return launch_impl<1, 128>(tq, tc, p, grid, stream);
      return static_cast<int>(cudaErrorInvalidValue);
    default: return static_cast<int>(cudaErrorInvalidValue);
  }
}

int dispatch_wide(int kcap, const CUtensorMap& tq, const CUtensorMap& tc, const ScanParams& p,
                  int grid, cudaStream_t stream) {
  switch (kcap) {
    case kAppendCap: return launch_impl<1, kAppendCap, false, 2>(tq, tc, p, grid, stream);
    case 1: return launch_impl<1, 1, false, 2>(tq, tc, p, grid, stream);
    case 4: return launch_impl<1, 4, false, 2>(tq, tc, p, grid, stream);
    case 8: return launch_impl<1, 8, false, 2>(tq, tc, p, grid, stream);
    case 10: return launch_impl<1, 10, false, 2>(tq, tc, p, grid, stream);
    case 16: return launch_impl<1, 16, false, 2>(tq, tc, p, grid, stream);
    case 32: return launch_impl<1, 32, false, 2>(tq, tc, p, grid, stream);
    default: return static_cast<int>(cudaErrorInvalidValue);
  }
}

int dispatch_pair(int kcap, const CUtensorMap& tq, const CUtensorMap& tc, const ScanParams& p,
                  int grid, cudaStream_t stream) {
  switch (kcap) {
    case kAppendCap: return launch_pair_impl<kAppendCap>(tq, tc, p, grid, stream);
    case 1: return launch_pair_impl<1>(tq, tc, p, grid, stream);
    case 4: return launch_pair_impl<4>(tq, tc, p, grid, stream);
    case 8: return launch_pair_impl<8>(tq, tc, p, grid, stream);
    case 10: return launch_pair_impl<10>(tq, tc, p, grid, stream);
    case 16: return launch_pair_impl<16>(tq, tc, p, grid, stream);
    case 32: return launch_pair_impl<32>(tq, tc, p, grid, stream);
    case 64: return launch_pair_impl<64>(tq, tc, p, grid, stream);
    case 128: return launch_pair_impl<128>(tq, tc, p, grid, stream);
    default: return static_cast<int>(cudaErrorInvalidValue);
  }
}

// ---------------------------------------------------------------------------------------------
// K2t: a latency-bound search (few queries, a short row range) in ONE launch on the tensor
// cores (BASELINE C1: 16 queries over a 10k x 384 corpus; reference: the naive-RAG Searching
// primitive, optimizer.py:178-198). The general scan puts queries on the UMMA M side and pays
// normalise + scan + merge launches and a per-item pipeline start for a 40-tile corpus (27 us).
// Here each CTA owns one 128-row tile with the rows on M and every query on N:
//  * TMA streams the tile's k-blocks (128 rows x 64 elements, SWIZZLE_128B: the arena's own
//    tensor map) into a ring while the four warps L2-normalise the queries (K5's arithmetic,
//    chunk-order sums) straight into the B operand in the canonical K-major SWIZZLE_128B
//    layout (16-byte chunk c of query r at chunk c ^ (r & 7) of its 128-byte row);
//  * one elected thread issues D[128 x NQ] += A[128 x 16] * B[NQ x 16]^T per k-step
//    (tcgen05.mma kind::f16, fp32 accumulators in TMEM, NQ columns);
//  * each thread tcgen05.ld's its row's NQ query scores, parks them in shared memory as
//    [query][row], and one warp per query takes the tile's top k (lane-local key lists, k
//    rounds of a warp max; (score, id) keys are unique, ties go to the smaller id);
//  * the last CTA to finish (arrival counter, self-resetting) merges the tiles' lists.
constexpr int kTinyRows = 128;
constexpr int kTinyThreads = 256;  // warps 0-3: TMEM lanes 0-127 (epilogue); all 8 stage / select

__device__ __forceinline__ uint64_t tk_key(float s, int32_t id) {
  uint32_t u = __float_as_uint(s);
  u = (u & 0x80000000u) ? ~u : (u | 0x80000000u);
  return (static_cast<uint64_t>(u) << 32) | static_cast<uint32_t>(~static_cast<uint32_t>(id));
}
__device__ __forceinline__ float tk_score(uint64_t k) {
  uint32_t u = static_cast<uint32_t>(k >> 32);
  u = (u & 0x80000000u) ? (u & 0x7FFFFFFFu) : ~u;
  return __uint_as_float(u);
}
__device__ __forceinline__ int32_t tk_id(uint64_t k) {
  return static_cast<int32_t>(~static_cast<uint32_t>(k & 0xFFFFFFFFu));
}
__device__ __forceinline__ uint64_t tk_pad() { return tk_key(-INFINITY, -1); }
// Two independent top-k selections interleaved (v[0, N): first set, v[N, 2N): second set):
// k rounds of (lane-local max below the previous round's key, warp max via shuffles).
template <int N>
__device__ __forceinline__ void tk_select2(const uint64_t (&v)[2 * N], int k, uint64_t* out0,
                                           uint64_t* out1, int lane) {
  const uint64_t pad = tk_pad();
  uint64_t p0 = ~0ull, p1 = ~0ull;
  for (int r = 0; r < k; ++r) {
    uint64_t b0 = pad, b1 = pad;
#pragma unroll
    for (int i = 0; i < N; ++i) {
      b0 = (v[i] < p0 && v[i] > b0) ? v[i] : b0;
      b1 = (v[N + i] < p1 && v[N + i] > b1) ? v[N + i] : b1;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const uint64_t y0 = __shfl_xor_sync(0xffffffffu, b0, o);
      const uint64_t y1 = __shfl_xor_sync(0xffffffffu, b1, o);
      b0 = y0 > b0 ? y0 : b0;
      b1 = y1 > b1 ? y1 : b1;
    }
    if (lane == 0) out0[r] = b0;
    if (lane == 1 && out1 != nullptr) out1[r] = b1;
    p0 = b0;
    p1 = b1;
  }
}
__device__ __forceinline__ uint32_t tk_pack(float a, float b) {
  const __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<const uint32_t*>(&h);
}
// 8 consecutive elements (index o) of the raw query matrix staged in shared memory, as fp32
__device__ __forceinline__ void tk_load8s(const uint8_t* qraw, int q_is_f32, int64_t o, float (&x)[8]) {
  if (q_is_f32) {
    const float4 a = *reinterpret_cast<const float4*>(qraw + o * 4);
    const float4 b = *reinterpret_cast<const float4*>(qraw + o * 4 + 16);
    x[0] = a.x; x[1] = a.y; x[2] = a.z; x[3] = a.w;
    x[4] = b.x; x[5] = b.y; x[6] = b.z; x[7] = b.w;
  } else {
    const uint4 w = *reinterpret_cast<const uint4*>(qraw + o * 2);
    const uint32_t ww[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      x[2 * t] = __uint_as_float(ww[t] << 16);
      x[2 * t + 1] = __uint_as_float(ww[t] & 0xFFFF0000u);
    }
  }
}

template <int NQ>
__global__ void __launch_bounds__(kTinyThreads, 1) tiny_scan_kernel(
    const __grid_constant__ CUtensorMap tmap_c, const void* __restrict__ q, int q_is_f32,
    int do_normalize, int B, int dim, int64_t row_beg, int64_t row_end, int32_t id_offset, int k,
    int stages, int tiled, int split_merge, uint64_t* __restrict__ part_keys,
    int32_t* __restrict__ arrive,
    float* __restrict__ out_s, int32_t* __restrict__ out_i, unsigned long long* __restrict__ trace) {
  // (trace: development timestamps per CTA and phase, TSV_SMALL_TRACE; null in production)
  auto stamp = [&](int ph) {
    if (trace != nullptr && threadIdx.x == 0) trace[blockIdx.x * 8 + ph] = global_ns();
  };
  stamp(0);
  // split_merge: the merge runs in tiny_merge_kernel, launched behind this one with
  // programmatic serialisation; let it launch now (it waits in griddepcontrol.wait)
  if (split_merge && threadIdx.x == 0) pdl_allow_dependents();
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  const int num_kb = (dim + kBlockK - 1) / kBlockK;
  constexpr int kABytes = kTinyRows * 128;           // one k-block of the row tile
  constexpr int kBkb = NQ * 128;                     // one k-block of the queries
  uint8_t* ring = smem;                              // [stages][16 KB]
  uint8_t* qtile = ring + static_cast<size_t>(stages) * kABytes;  // [num_kb][NQ x 128 B]
  float* sc = reinterpret_cast<float*>(qtile + static_cast<size_t>(num_kb) * kBkb);  // [NQ][128]
  uint8_t* qraw = reinterpret_cast<uint8_t*>(sc + NQ * kTinyRows);  // [B][dim] as given
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(
      qraw + ((static_cast<size_t>(B) * dim * (q_is_f32 ? 4 : 2) + 15) & ~static_cast<size_t>(15)));
  uint64_t* empty_bar = full_bar + stages;
  uint64_t* acc_bar = empty_bar + stages;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_bar + 1);
  __shared__ int last_s;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t row0 = row_beg + static_cast<int64_t>(blockIdx.x) * kTinyRows;
  const int nvalid = static_cast<int>(min(static_cast<int64_t>(kTinyRows), row_end - row0));
  constexpr uint32_t kTmemCols = NQ < 32 ? 32 : NQ;
  if (tid == 0) {
    ptx::tma_prefetch_desc(&tmap_c);
    for (int s_ = 0; s_ < stages; ++s_) {
      ptx::mbar_init(&full_bar[s_], 1);
      ptx::mbar_init(&empty_bar[s_], 1);
    }
    ptx::mbar_init(acc_bar, 1);
    ptx::fence_mbar_init();
  }
  if (warp == 1) {
    ptx::tmem_alloc(tmem_slot, kTmemCols);
    ptx::tmem_relinquish();
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  pdl_wait();  // the queries (and rows) may be the previous kernel's output
  stamp(1);
  const uint64_t pol = ptx::policy_evict_normal();
  // k-block kb of the tile: a 2-D box of the row-major arena, or (tiled arena, row0 a multiple
  // of 128) the contiguous [128 x 64] block ((row0 / 128) * num_kb + kb): the same operand bytes,
  // so both layouts give bit-identical scores
  auto load_kb = [&](int kb, int slot) {  // whole warp; one elected lane issues
    ptx::mbar_arrive_expect_tx_warp(&full_bar[slot], kABytes);
    if (tiled)
      ptx::tma_load_3d_warp(ring + slot * kABytes, &tmap_c, &full_bar[slot], 0, 0,
                            static_cast<int32_t>((row0 >> 7) * num_kb + kb), pol);
    else
      ptx::tma_load_2d_warp(ring + slot * kABytes, &tmap_c, &full_bar[slot], kb * kBlockK,
                            static_cast<int32_t>(row0), pol);
  };
  if (warp == 0)  // first ring-full of k-blocks in flight before the queries are staged
    for (int kb = 0; kb < min(stages, num_kb); ++kb) load_kb(kb, kb);
  // raw queries -> shared memory in one round trip (cp.async, all threads), then normalised
  // (K5's arithmetic, chunk-order sums) into the B operand: query r, 16-byte chunk ch
  // (elements 8 ch ..) goes to k-block ch / 8, chunk position (ch % 8) ^ (r % 8) of row r;
  // 8-row atoms 1024 B apart; padding queries are zero
  const int chunks = dim >> 3;
  const int esz = q_is_f32 ? 4 : 2;
  const int raw_chunks = B * dim * esz / 16;  // 16-byte chunks of the raw query matrix
  for (int c = tid; c < raw_chunks; c += kTinyThreads) {
    const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(qraw + c * 16));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d),
                 "l"(reinterpret_cast<const uint8_t*>(q) + static_cast<int64_t>(c) * 16)
                 : "memory");
  }
  asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory");
  __syncthreads();
  for (int r = warp; r < NQ; r += kTinyThreads / 32) {
    float ss = 0.f;
    if (r < B && do_normalize) {
      for (int ch = lane; ch < chunks; ch += 32) {
        float x[8];
        tk_load8s(qraw, q_is_f32, static_cast<int64_t>(r) * dim + ch * 8, x);
#pragma unroll
        for (int t = 0; t < 8; ++t) ss = fmaf(x[t], x[t], ss);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
    }
    const float scale = (do_normalize && ss > 0.f) ? rsqrtf(ss) : 1.f;
    for (int ch = lane; ch < num_kb * 8; ch += 32) {
      uint4 w = make_uint4(0, 0, 0, 0);
      if (r < B && ch < chunks) {
        float x[8];
        tk_load8s(qraw, q_is_f32, static_cast<int64_t>(r) * dim + ch * 8, x);
        w.x = tk_pack(x[0] * scale, x[1] * scale);
        w.y = tk_pack(x[2] * scale, x[3] * scale);
        w.z = tk_pack(x[4] * scale, x[5] * scale);
        w.w = tk_pack(x[6] * scale, x[7] * scale);
      }
      const int kb = ch >> 3, c = ch & 7;
      *reinterpret_cast<uint4*>(qtile + kb * kBkb + (r >> 3) * 1024 + (r & 7) * 128 +
                                ((c ^ (r & 7)) << 4)) = w;
    }
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic writes -> UMMA reads
  __syncthreads();
  stamp(2);
  if (warp == 0) {
    // producer: the rest of the k-blocks through the ring
    int stage = 0;
    uint32_t phase = 0;
    for (int kb = 0; kb < num_kb; ++kb) {
      if (kb >= stages) {
        ptx::mbar_wait(&empty_bar[stage], phase ^ 1);
        load_kb(kb, stage);
      }
      if (++stage == stages) {
        stage = 0;
        phase ^= 1;
      }
    }
  } else if (warp == 1) {
    // MMA issuer (warp-uniform loop, one elected lane issues)
    constexpr uint32_t idesc = ptx::idesc_bf16_f32(kTinyRows, NQ);
    const uint64_t adesc0 = ptx::umma_desc_sw128(ptx::smem_u32(ring));
    const uint64_t bdesc0 = ptx::umma_desc_sw128(ptx::smem_u32(qtile));
    int stage = 0;
    uint32_t phase = 0;
    for (int kb = 0; kb < num_kb; ++kb) {
      ptx::mbar_wait(&full_bar[stage], phase);
      ptx::tc_fence_after();
      const uint64_t ad = adesc0 + static_cast<uint64_t>((stage * kABytes) >> 4);
      const uint64_t bd = bdesc0 + static_cast<uint64_t>((kb * kBkb) >> 4);
#pragma unroll
      for (int kk = 0; kk < kBlockK / 16; ++kk)
        ptx::mma_f16_ss_warp(tmem_base, ad + 2 * kk, bd + 2 * kk, idesc, (kb | kk) != 0 ? 1u : 0u);
      ptx::mma_commit_warp(&empty_bar[stage]);
      if (++stage == stages) {
        stage = 0;
        phase ^= 1;
      }
    }
    ptx::mma_commit_warp(acc_bar);
  }
  // epilogue: thread = row (TMEM lane), NQ query scores -> shared memory [query][row]
  if (warp < 4) {
    ptx::mbar_wait(acc_bar, 0);
    ptx::tc_fence_after();
    const uint32_t taddr = tmem_base + (static_cast<uint32_t>(warp * 32) << 16);
    const int row = warp * 32 + lane;
#pragma unroll
    for (int c = 0; c < NQ; c += 32) {
      uint32_t v[32];
      ptx::tmem_ld_32x32b_x32(taddr + c, v);
      ptx::tmem_ld_wait();
      ptx::tmem_regs_ready(v);
#pragma unroll
      for (int j = 0; j < 32; ++j)
        if (c + j < NQ) sc[(c + j) * kTinyRows + row] = __uint_as_float(v[j]);
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  stamp(3);
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem_base, kTmemCols);
  }
  // the tile's top k per query -> scratch [query][tile][k]
  const uint64_t pad = tk_pad();
  const int nblk = gridDim.x;
  for (int qa = warp; qa < B; qa += 2 * (kTinyThreads / 32)) {
    const int qb = qa + kTinyThreads / 32;
    uint64_t v[2 * (kTinyRows / 32)];  // two queries' rows, one chain each in tk_select2
#pragma unroll
    for (int u = 0; u < kTinyRows / 32; ++u) {
      const int r = lane + 32 * u;
      const int32_t id = static_cast<int32_t>(row0 + r) + id_offset;
      v[u] = r < nvalid ? tk_key(sc[qa * kTinyRows + r], id) : pad;
      v[kTinyRows / 32 + u] = (r < nvalid && qb < B) ? tk_key(sc[qb * kTinyRows + r], id) : pad;
    }
    tk_select2<kTinyRows / 32>(v, k, part_keys + (static_cast<int64_t>(qa) * nblk + blockIdx.x) * k,
                               qb < B ? part_keys + (static_cast<int64_t>(qb) * nblk + blockIdx.x) * k
                                      : nullptr,
                               lane);
  }
  stamp(4);
  if (split_merge) return;  // (the merge kernel reads the lists after this grid completes)
  __threadfence();
  __syncthreads();
  if (tid == 0) last_s = atomicAdd(arrive, 1) == nblk - 1;
  __syncthreads();
  stamp(5);
  if (!last_s) return;
  __threadfence();
  // last CTA: one warp per query. Every tile's list is sorted, and tile t alone holds k keys
  // >= its k-th key, so the global k-th key is >= tau = max_t (k-th key of tile t): only keys
  // >= tau can be in the result. One warp max finds tau, a ballot compacts the survivors
  // (usually a few more than k) into shared memory, and each survivor's output position is
  // the number of survivors above it. (More than 64 survivors: k rounds of a warp max.)
  // every tile's lists of every query -> shared memory with 16-byte async copies (one L2 round
  // trip; the ring is free now), then everything below reads shared memory
  const int total = nblk * k;   // <= 512 keys per query (checked on the host)
  const int all_n = B * total;  // <= 64 x 512 keys: fits the ring (checked on the host)
  uint64_t* allk = reinterpret_cast<uint64_t*>(ring);
#pragma unroll 1
  for (int e = 2 * tid; e < all_n; e += 2 * kTinyThreads) {
    const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(allk + e));
    if (e + 1 < all_n)
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(part_keys + e) : "memory");
    else
      allk[e] = static_cast<uint64_t>(__ldcg(reinterpret_cast<const unsigned long long*>(part_keys + e)));
  }
  asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory");
  __syncthreads();
  stamp(6);
  // one warp per two queries (interleaved: two independent dependency chains): k rounds of
  // (lane-local max below the previous round's key, warp max) over the keys in shared memory
  constexpr int kW = kTinyThreads / 32;
#pragma unroll 1
  for (int q0 = warp; q0 < B; q0 += 2 * kW) {
    const int q1 = q0 + kW < B ? q0 + kW : q0;  // (odd count: the second chain repeats q0)
    const uint64_t* s0 = allk + static_cast<int64_t>(q0) * total;
    const uint64_t* s1 = allk + static_cast<int64_t>(q1) * total;
    uint64_t p0 = ~0ull, p1 = ~0ull;
#pragma unroll 1
    for (int r = 0; r < k; ++r) {
      uint64_t b0 = pad, b1 = pad;
#pragma unroll 4
      for (int e = lane; e < total; e += 32) {
        const uint64_t x0 = s0[e], x1 = s1[e];
        b0 = (x0 < p0 && x0 > b0) ? x0 : b0;
        b1 = (x1 < p1 && x1 > b1) ? x1 : b1;
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const uint64_t y0 = __shfl_xor_sync(0xffffffffu, b0, o);
        const uint64_t y1 = __shfl_xor_sync(0xffffffffu, b1, o);
        b0 = y0 > b0 ? y0 : b0;
        b1 = y1 > b1 ? y1 : b1;
      }
      if (lane == 0) {
        out_s[static_cast<int64_t>(q0) * k + r] = b0 == pad ? -INFINITY : tk_score(b0);
        out_i[static_cast<int64_t>(q0) * k + r] = b0 == pad ? -1 : tk_id(b0);
      } else if (lane == 1) {
        out_s[static_cast<int64_t>(q1) * k + r] = b1 == pad ? -INFINITY : tk_score(b1);
        out_i[static_cast<int64_t>(q1) * k + r] = b1 == pad ? -1 : tk_id(b1);
      }
      p0 = b0;
      p1 = b1;
    }
  }
  if (tid == 0) *arrive = 0;  // ready for the next launch on this scratch
  __syncthreads();
  stamp(7);
}

// The cross-tile merge of K2t as its own grid (one CTA per query, launched with programmatic
// serialisation behind the scan, which allows it at its start): the 16 queries' merges run on 16
// SMs at once instead of one after another in the scan's last CTA, and the scan needs no
// arrival counter or fence. Each CTA loads its query's nblk * k keys (<= 512: two per thread,
// one round trip), every warp selects the top k of its 64 keys (k rounds of a warp max below
// the previous round's key), then warp 0 the top k of those.
__global__ void __launch_bounds__(256) tiny_merge_kernel(const uint64_t* __restrict__ part_keys,
                                                         int nblk, int k,
                                                         float* __restrict__ out_s,
                                                         int32_t* __restrict__ out_i) {
  __shared__ uint64_t wsel[8][16];
  __shared__ uint64_t fin[16];
  pdl_wait();
  const int q = blockIdx.x, tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int total = nblk * k;
  const uint64_t* src = part_keys + static_cast<int64_t>(q) * total;
  const uint64_t pad = tk_pad();
  uint64_t v[2];
#pragma unroll
  for (int u = 0; u < 2; ++u) {
    const int e = tid + 256 * u;
    v[u] = e < total ? static_cast<uint64_t>(__ldcg(reinterpret_cast<const unsigned long long*>(src + e)))
                     : pad;
  }
  auto rounds = [&](const uint64_t* vals, int n, uint64_t* out) {
    uint64_t prev = ~0ull;
    for (int r = 0; r < k; ++r) {
      uint64_t best = pad;
      for (int i = 0; i < n; ++i) best = (vals[i] < prev && vals[i] > best) ? vals[i] : best;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const uint64_t y = __shfl_xor_sync(0xffffffffu, best, o);
        best = y > best ? y : best;
      }
      if (lane == 0) out[r] = best;
      prev = best;
    }
  };
  rounds(v, 2, wsel[warp]);
  __syncthreads();
  if (warp != 0) return;
  uint64_t w[4];  // 8 warps x k <= 16 keys
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int e = lane + 32 * u, ww = e >> 4, r = e & 15;
    w[u] = r < k ? wsel[ww][r] : pad;
  }
  rounds(w, 4, fin);
  __syncwarp();
  for (int r = lane; r < k; r += 32) {
    const uint64_t m = fin[r];
    const int32_t id = m == pad ? -1 : tk_id(m);
    out_s[static_cast<int64_t>(q) * k + r] = id < 0 ? -INFINITY : tk_score(m);
    out_i[static_cast<int64_t>(q) * k + r] = id;
  }
}

template <int NQ>
int launch_tiny_v(const CUtensorMap& tmap_c, const void* q, int q_is_f32, int do_normalize,
                  int B, int dim, int64_t row_beg, int64_t row_end, int32_t id_offset, int k,
                  uint64_t* part_keys, int32_t* arrive, float* out_s, int32_t* out_i,
                  cudaStream_t stream, unsigned long long* trace, int tiled, int split) {
  const int num_kb = (dim + kBlockK - 1) / kBlockK;
  const int stages = num_kb < 6 ? num_kb : 6;
  const size_t qraw = (static_cast<size_t>(B) * dim * (q_is_f32 ? 4 : 2) + 15) & ~size_t(15);
  const size_t smem = 1024 + static_cast<size_t>(stages) * kTinyRows * 128 +
                      static_cast<size_t>(num_kb) * NQ * 128 + NQ * kTinyRows * 4 + qraw +
                      (2 * stages + 2) * 8 + 16;
  const int64_t tiles = (row_end - row_beg + kTinyRows - 1) / kTinyRows;
  if (smem > 200 * 1024 || tiles * k > 512) return static_cast<int>(cudaErrorInvalidValue);
  auto kern = tiny_scan_kernel<NQ>;
  static std::atomic<uint64_t> configured{0};
  if (first_on_device(configured)) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         200 * 1024);
    if (e != cudaSuccess) return static_cast<int>(e);
  }
  const int nblk = static_cast<int>((row_end - row_beg + kTinyRows - 1) / kTinyRows);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(nblk);
  cfg.blockDim = dim3(kTinyThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, tmap_c, q, q_is_f32, do_normalize, B, dim,
                                     row_beg, row_end, id_offset, k, stages, tiled, split,
                                     part_keys, arrive, out_s, out_i, trace);
  if (e != cudaSuccess || !split) return static_cast<int>(e);
  cudaLaunchConfig_t mc = cfg;
  mc.gridDim = dim3(B);
  mc.blockDim = dim3(256);
  mc.dynamicSmemBytes = 0;
  return static_cast<int>(cudaLaunchKernelEx(&mc, tiny_merge_kernel,
                                             static_cast<const uint64_t*>(part_keys), nblk, k,
                                             out_s, out_i));
}

}  // namespace

int dispatch_tf32(int kcap, const CUtensorMap& tq, const CUtensorMap& tc, const CUtensorMap& tq_lo,
                  const CUtensorMap& tc_lo, const ScanParams& p, int grid, cudaStream_t stream) {
  switch (kcap) {
    case 1: return launch_impl<1, 1, true>(tq, tc, p, grid, stream, &tq_lo, &tc_lo);
    case 4: return launch_impl<1, 4, true>(tq, tc, p, grid, stream, &tq_lo, &tc_lo);
    case 8: return launch_impl<1, 8, true>(tq, tc, p, grid, stream, &tq_lo, &tc_lo);
    case 10: return launch_impl<1, 10, true>(tq, tc, p, grid, stream, &tq_lo, &tc_lo);
    case 16: return launch_impl<1, 16, true>(tq, tc, p, grid, stream, &tq_lo, &tc_lo);
    case 32: return launch_impl<1, 32, true>(tq, tc, p, grid, stream, &tq_lo, &tc_lo);
    case 64: return launch_impl<1, 64, true>(tq, tc, p, grid, stream, &tq_lo, &tc_lo);
    default: return static_cast<int>(cudaErrorInvalidValue);
  }
}

int scan_kcap_for(int k) {
  static const int caps[] = {1, 4, 8, 10, 16, 32, 64, 128};
  for (int c : caps)
    if (k <= c) return c;
  return 0;
}

int launch_scan_topk_tf32(int kcap, const CUtensorMap& tmap_q, const CUtensorMap& tmap_c,
                          const CUtensorMap& tmap_q_lo, const CUtensorMap& tmap_c_lo,
                          const ScanParams& p, int grid, cudaStream_t stream) {
  if (grid <= 0) return 0;
  return dispatch_tf32(kcap, tmap_q, tmap_c, tmap_q_lo, tmap_c_lo, p, grid, stream);
}

int tiny_scan_blocks(int64_t n) { return static_cast<int>((n + kTinyRows - 1) / kTinyRows); }

int launch_tiny_scan(const CUtensorMap& tmap_c, const void* q, int q_is_f32, int do_normalize,
                     int B, int dim, int64_t row_beg, int64_t row_end, int32_t id_offset, int k,
                     uint64_t* part_keys, int32_t* arrive, float* out_s, int32_t* out_i,
                     cudaStream_t stream, unsigned long long* trace, int tiled, int split) {
  if (B <= 0 || B > 64 || k > 16 || dim % 8 != 0 || (tiled && row_beg % kTinyRows != 0))
    return static_cast<int>(cudaErrorInvalidValue);
#define TSV_TINY(NQ) launch_tiny_v<NQ>(tmap_c, q, q_is_f32, do_normalize, B, dim, row_beg, row_end, id_offset, k, part_keys, arrive, out_s, out_i, stream, trace, tiled, split)
  if (B <= 16) return TSV_TINY(16);
  if (B <= 32) return TSV_TINY(32);
  return TSV_TINY(64);
#undef TSV_TINY
}

int launch_scan_topk(int mb, int kcap, const CUtensorMap& tmap_q, const CUtensorMap& tmap_c,
                     const ScanParams& p, int grid, cudaStream_t stream) {
  if (grid <= 0) return 0;
  if (mb == kWideMode) return dispatch_wide(kcap, tmap_q, tmap_c, p, grid, stream);
  if (mb == 2) return dispatch_kcap<2>(kcap, tmap_q, tmap_c, p, grid, stream);
  if (mb == 1) return dispatch_kcap<1>(kcap, tmap_q, tmap_c, p, grid, stream);
  if (mb == kPairMode) return dispatch_pair(kcap, tmap_q, tmap_c, p, grid, stream);
  return static_cast<int>(cudaErrorInvalidValue);
}

}  // namespace tsv
