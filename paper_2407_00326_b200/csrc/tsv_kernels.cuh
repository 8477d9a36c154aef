// Shared declarations for the retrieval kernels (K1 scan+top-k, K3 rerank, K4 merge, K5 normalize).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>

namespace tsv {

// True the first time it is called on the current device for a given mask (kernel function
// attributes are per device; setting them on every launch costs a driver call).
inline bool first_on_device(std::atomic<uint64_t>& mask) {
  int d = 0;
  cudaGetDevice(&d);
  const uint64_t bit = 1ull << (d & 63);
  return (mask.fetch_or(bit) & bit) == 0;
}

// Programmatic dependent launch (PDL): the merge-side kernels are launched with programmatic
// stream serialisation, so their launch overlaps the tail of the scan before them; they wait
// for the scan's completion (and memory) in griddepcontrol.wait. The scan CTAs allow the early
// launch at their start.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_allow_dependents() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// Geometry of the fused scan (K1). Queries sit on the UMMA M side (one TMEM lane per query),
// corpus rows on the N side; K is the embedding dimension, streamed 64 bf16 (one 128 B swizzle
// row) per k-block.
constexpr int kBlockM = 128;   // queries per UMMA tile
constexpr int kBlockN = 128;   // corpus rows per tile
constexpr int kBlockK = 64;    // bf16 elements per k-block (128 B rows, SWIZZLE_128B)
constexpr int kNumNonEpiWarps = 4;  // warp 0 TMA, warp 1 MMA, warp 2 TMEM alloc, warp 3 (pair: query TMA)

// One unit of scan work: a block of up to MB*128 consecutive queries against a contiguous
// corpus row range. Each query of the item produces one sorted partial list of KCAP
// (score, id) pairs at partial row `out_row + local_query`.
struct ScanItem {
  int32_t q_begin;
  int32_t q_count;
  int64_t row_begin;
  int64_t row_end;
  int64_t out_row;
  int32_t id_offset;  // emitted id = corpus row + id_offset
  int32_t pad_;
};

struct ScanParams {
  const ScanItem* items;  // nullptr: implicit (query-group x range) grid
  int32_t num_items;
  // implicit-grid description (items == nullptr)
  int32_t B;          // number of queries
  int32_t R;          // corpus ranges per query group
  int32_t id_offset;  // emitted id = row + id_offset
  int64_t row_beg;    // scanned rows [row_beg, row_end)
  int64_t row_end;
  int32_t num_kb;     // ceil(dim / 64)
  int32_t out_k;      // entries written per partial row (<= KCAP)
  float* out_scores;  // [rows][out_k]
  int32_t* out_ids;
  // lockstep progress counters, one per item (zeroed before the launch)
  int32_t* counter;
  int32_t flags;  // kFlag* bits below
  // Optional per-query admission floor (k > 32 lists): a lower bound of the query's final k-th
  // score (from a sample pass); candidates at or below it can never be in the result.
  const float* tau0;
  int32_t lock_window;  // lockstep: max tiles ahead of range partners (0 = default)
  // Single-CTA bf16 kernel: query rows per A-tile TMA box (0 = kBlockM). With B < 128 the box
  // covers only the real queries (rounded up to the 8-row swizzle atom); the TMEM lanes of the
  // rows it leaves untouched are never emitted.
  int32_t a_rows;
  // Shared admission floor (nullptr = off), one order-preserving key per query row, zeroed
  // before the launch. Every corpus range of a query publishes the k-th score of its full list
  // (atomicMax) and admits only candidates at or above the best published one: that range's
  // list already holds k rows scoring at least that much, so nothing below it can reach the
  // merged top-k. Without it each range's threshold starts from scratch and the insertions
  // of the first tiles of every range dominate short scans.
  uint32_t* floor_g;
  // Candidate mode (KCAP == kAppendCap, k > 32 after a seeding pass): every row scoring above
  // the query's tau0 is appended to its candidate row out_scores/out_ids[q * cand_cap, ...);
  // cand_count[q] (zeroed before the launch) counts them, and may exceed cand_cap (overflow:
  // the entries past cand_cap are dropped and the caller's gated fallback reruns the query set).
  int32_t* cand_count;
  int32_t cand_cap;
  // Device-side gate (nullptr = always run): the kernel returns at once unless *gate != 0. Used
  // for the overflow fallback, so the decision needs no host round trip.
  const int32_t* gate;
  // Sample pass of a seeded search (> 1): every implicit-grid range scans only its first
  // ceil(1/sample_div) of its tiles, so the sample is spread over the whole row range.
  int32_t sample_div;
};

// List-capacity value selecting candidate (append) mode in launch_scan_topk.
constexpr int kAppendCap = 0;
// Candidate-row capacity per query in append mode. Seeding from a 1/16 sample leaves about
// 16 k rows above tau0 for a uniformly spread corpus (k = 128: ~2k +- 0.2k).
constexpr int kCandCap = 8192;
int launch_cand_select(const float* buf_s, const int32_t* buf_i, const int32_t* cnt, int cap,
                       int B, int kout, float* out_s, int32_t* out_id, int32_t* overflow,
                       cudaStream_t stream);

constexpr int kFlagTiled = 2;
constexpr int kFlagLockstep = 4;  // static pair kernel: bound drift between range partners
// Implicit grid in range-major order (pair kernel): item i covers corpus range i / nqg for query
// group i % nqg, so the items of one range are adjacent and, when nqg * R is a multiple of the
// worker count, all workers stay busy over several rounds while each range is still streamed
// once (its query groups run in the same round, in lockstep).
constexpr int kFlagRangeMajor = 8;
// Diagnostic flags (TSV_DIAG, pair kernel; results are wrong by design): attribute the step's
// energy under the power cap. 16: epilogue loads the accumulators but filters nothing;
// 32: every tile re-reads the range's first corpus tile (L2-resident, no HBM stream).
constexpr int kFlagDiagNoFilter = 16;
constexpr int kFlagDiagNoStream = 32;
// 64: query tiles are loaded for the first corpus tile only (later tiles reuse stale smem).
constexpr int kFlagDiagNoQueryLoad = 64;
// 128 (single-CTA kernel): set up and tear down only (no items): the launch's fixed cost.
constexpr int kFlagDiagSetupOnly = 128;
// Tiled arena layout: row i, element d at ((i/128 * KB + d/64) * 128 + i%128) * 64 + d%64,
// KB = ceil(dim/64): every [128 rows x 64 elements] k-block tile is one contiguous 16 KB block.
int launch_seed_floor(const float* s, const int32_t* id, int B, int k, float* floor_out,
                      cudaStream_t stream);
size_t peer_buffer_bytes(int world, int max_b, int max_k);
int launch_peer_exchange_merge(void* const* peers_dev, int rank, int world, int B, int k,
                               int max_b, int max_k, uint32_t epoch, uint64_t timeout_ns,
                               const float* local_s, const int32_t* local_i, float* out_s,
                               int32_t* out_i, uint32_t* err_word, int num_sms,
                               cudaStream_t stream);
int launch_scatter_tiled(const void* src, int src_is_f32, int64_t n, int dim, int do_normalize,
                         void* arena, int64_t first_row, cudaStream_t stream);

// `mb` argument of launch_scan_topk selecting the CTA-pair kernel: 256 queries x 256 corpus
// rows per pair tile (tcgen05 cta_group::2); the tensor map for queries then uses 128-row
// boxes and the corpus map 128-row boxes (each CTA loads its half).
constexpr int kPairMode = 4;
constexpr int kPairQG = 256;
constexpr int kPairTileRows = 256;
// `mb` selecting the single-CTA kernel with 256-row corpus tiles (M=128 x N=256 per MMA; k <= 32
// or candidate append; 128 queries per group).
constexpr int kWideMode = 5;
constexpr int kWideTileRows = 256;

// Host-side launchers (return cudaError_t as int).
int launch_scan_topk(int mb, int kcap, const CUtensorMap& tmap_q, const CUtensorMap& tmap_c,
                     const ScanParams& p, int grid, cudaStream_t stream);
int scan_kcap_for(int k);  // smallest supported list capacity >= k (0 if unsupported)
// fp32 mode (3xTF32): hi / lo planes of queries and corpus, single-CTA kernel, k <= 64
int launch_scan_topk_tf32(int kcap, const CUtensorMap& tmap_q, const CUtensorMap& tmap_c,
                          const CUtensorMap& tmap_q_lo, const CUtensorMap& tmap_c_lo,
                          const ScanParams& p, int grid, cudaStream_t stream);
constexpr int kMaxKF32 = 64;
// Split rows into tf32 hi / residual lo planes (fp32 storage), optionally L2-normalised.
int launch_split_f32(const void* src, int src_is_f32, int64_t n, int dim, int do_normalize,
                     float* hi, float* lo, cudaStream_t stream);
constexpr int kMaxRegK = 32;   // larger k uses shared-memory lists (single-CTA, 128 queries)
constexpr int kMaxK = 128;

int launch_merge_topk(const float* in_s, const int32_t* in_id, int lists, int B, int kin,
                      int64_t list_stride_rows, int kout, float* out_s, int32_t* out_id,
                      cudaStream_t stream, int dedup = 0, const int32_t* gate = nullptr);

int launch_rerank(const void* arena, const float* arena_hi, const float* arena_lo, int64_t nrows,
                  int dim, const void* q, const float* q_lo, int q_is_f32, int B,
                  const int32_t* cand, int C, int k, float* out_s, int32_t* out_id,
                  cudaStream_t stream, int tiled = 0, const int32_t* offs = nullptr);

// K3 over a bf16 arena with the gather pipelined through shared memory (cp.async rings);
// offs (optional, device [B]): candidate ids of question b are relative to arena row offs[b].
// splits > 1 (k <= 32): question b's candidates spread over `splits` blocks; part_keys
// [B * splits * k] and arrivals [B] (zeroed once; the kernel leaves them zero) are scratch.
int launch_rerank_ring(const void* arena, int64_t nrows, int dim, const void* q, int q_is_f32,
                       int B, const int32_t* cand, int C, int k, const int32_t* offs,
                       float* out_s, int32_t* out_id, cudaStream_t stream, int tiled,
                       int splits, uint64_t* part_keys, int32_t* arrivals, int num_sms);
int rerank_lists_splits(int B, int C, int k, int dim, int num_sms);

// Contextual chain in one launch: per query, search its own arena segment (q_rows [B][2],
// <= max_rows <= 1024 rows; bf16 / tiled arenas, dim % 8 == 0, dim <= 2048), top k_s, rerank
// those against qr (null: the query itself), top k_r. Questions are normalised in-kernel when
// do_normalize.
size_t search_rerank_seg_smem(int dim, int max_rows, int k_s);
int launch_search_rerank_seg(const void* arena, int64_t nrows, int dim, int tiled, const void* qs,
                             const void* qr, int q_is_f32, int do_normalize,
                             const int64_t* q_rows, int B, int max_rows, int k_s, int k_r,
                             int local_ids, float* os_s, int32_t* os_i, float* or_s,
                             int32_t* or_i, cudaStream_t stream);
constexpr int kFusedSegMaxRows = 1024;

// K2s: one-launch search for latency-bound shapes (few queries, short row ranges; bf16 / tiled
// arenas, dim % 8 == 0, dim <= 1024, k <= 16). Grid (nblk row blocks) x (query groups of
// small_scan_qg(dim)); part_keys [groups * nblk * QG * 16] and arrive [groups] (zeroed once; the
// kernel leaves them zero) are scratch. Queries are normalised in-kernel when do_normalize.
int small_scan_qg(int dim);
int launch_small_scan(const void* arena, int dim, int tiled, const void* q, int q_is_f32,
                      int do_normalize, int B, int64_t row_beg, int64_t row_end, int32_t id_offset,
                      int k, int nblk, uint64_t* part_keys, int32_t* arrive, float* out_s,
                      int32_t* out_i, cudaStream_t stream, unsigned long long* trace = nullptr);

// K2t: one-launch tensor-core search for few queries (B <= 64) over a short row range of a
// bf16 arena (row-major, or tiled with row_beg % 128 == 0): one CTA per 128-row tile (rows on UMMA M, queries on N), per-tile top k
// to part_keys [B * tiles * k], the last CTA merges; arrive (one int, zeroed once) is left zero.
int tiny_scan_blocks(int64_t n);
int launch_tiny_scan(const CUtensorMap& tmap_c, const void* q, int q_is_f32, int do_normalize,
                     int B, int dim, int64_t row_beg, int64_t row_end, int32_t id_offset, int k,
                     uint64_t* part_keys, int32_t* arrive, float* out_s, int32_t* out_i,
                     cudaStream_t stream, unsigned long long* trace = nullptr, int tiled = 0,
                     int split = 0);  // split: cross-tile merge as a second (PDL) grid

int launch_normalize(const void* src, int src_is_f32, int64_t n, int dim, int do_normalize,
                     void* dst_bf16, cudaStream_t stream);

}  // namespace tsv
