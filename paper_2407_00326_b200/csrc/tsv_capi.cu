// C ABI of the retrieval backend (declared in include/tsv.h). Host-side orchestration only:
// argument checking, arena / workspace management, TMA descriptor encoding, work-item
// planning and kernel launches. No computation happens on the host.
#include "../../include/tsv.h"
#include "tsv_kernels.cuh"

#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <map>
#include <set>
#include <numeric>
#include <mutex>
#include <string>
#include <vector>

namespace {

thread_local std::string g_last_error;
std::atomic<int64_t> g_launches{0};

int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return code;
}

int cuda_fail(cudaError_t e, const char* what) {
  return fail(TSV_ERR_DEVICE, "%s: %s", what, cudaGetErrorString(e));
}

#define TSV_CUDA(call, what)                      \
  do {                                            \
    cudaError_t e__ = (call);                     \
    if (e__ != cudaSuccess) return cuda_fail(e__, what); \
  } while (0)

PFN_cuTensorMapEncodeTiled_v12000 get_encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

// 2-D bf16 row-major [rows, dim] map with a [box_rows, 64] box and 128 B swizzle.
int encode_rows_map(CUtensorMap* map, const void* base, int64_t rows, int dim, int box_rows,
                    bool f32 = false) {
  auto fn = get_encode_fn();
  if (fn == nullptr) return fail(TSV_ERR_DEVICE, "cuTensorMapEncodeTiled unavailable");
  const cuuint64_t esize = f32 ? 4 : 2;
  cuuint64_t gdim[2] = {static_cast<cuuint64_t>(dim), static_cast<cuuint64_t>(std::max<int64_t>(rows, 1))};
  cuuint64_t gstride[1] = {static_cast<cuuint64_t>(dim) * esize};
  // one 128-byte swizzle row per box row: 64 bf16 or 32 fp32 elements
  cuuint32_t box[2] = {static_cast<cuuint32_t>(128 / esize), static_cast<cuuint32_t>(box_rows)};
  cuuint32_t estride[2] = {1, 1};
  CUtensorMapL2promotion promo = CU_TENSOR_MAP_L2_PROMOTION_NONE;
  if (const char* e = getenv("TSV_L2_PROMO")) {
    const int v = atoi(e);
    promo = v == 0 ? CU_TENSOR_MAP_L2_PROMOTION_NONE
                   : v == 64 ? CU_TENSOR_MAP_L2_PROMOTION_L2_64B
                             : v == 128 ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B
                                        : CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
  }
  CUresult r = fn(map, f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
                  const_cast<void*>(base), gdim, gstride,
                  box, estride, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, promo,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(TSV_ERR_DEVICE, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return TSV_OK;
}

// Tiled arena (TSV_BF16_TILED): 3-D view {64 elements, 128 rows, tiles * kblocks}; each box is
// one contiguous 16 KB [128 x 64] k-block tile.
int encode_tiled_map(CUtensorMap* map, const void* base, int64_t cap_rows, int dim) {
  auto fn = get_encode_fn();
  if (fn == nullptr) return fail(TSV_ERR_DEVICE, "cuTensorMapEncodeTiled unavailable");
  const int64_t kbs = (dim + 63) / 64;
  const int64_t tiles = (cap_rows + 127) / 128;
  cuuint64_t gdim[3] = {64, 128, static_cast<cuuint64_t>(tiles * kbs)};
  cuuint64_t gstride[2] = {128, 128 * 128};
  cuuint32_t box[3] = {64, 128, 1};
  cuuint32_t estride[3] = {1, 1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), gdim, gstride,
                  box, estride, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(TSV_ERR_DEVICE, "cuTensorMapEncodeTiled (3d) failed (%d)", (int)r);
  return TSV_OK;
}

// Per-(index, stream) scratch owner: the stream the buffers are used on, and whether a CUDA
// graph captured on that stream has baked their addresses in (then they may not move).
struct WsState {
  cudaStream_t stream = nullptr;
  bool captured = false;
};

// The library's own stream-ordered memory pool on the current device, with an unlimited release
// threshold: memory freed by workspace growth stays mapped and is reused instead of being
// returned to the OS at every synchronisation point (the default pool's threshold is 0).
static cudaMemPool_t workspace_pool() {
  static std::mutex mu;
  static std::map<int, cudaMemPool_t> pools;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return nullptr;
  std::lock_guard<std::mutex> lock(mu);
  auto it = pools.find(dev);
  if (it != pools.end()) return it->second;
  cudaMemPoolProps props = {};
  props.allocType = cudaMemAllocationTypePinned;
  props.location.type = cudaMemLocationTypeDevice;
  props.location.id = dev;
  cudaMemPool_t pool = nullptr;
  if (cudaMemPoolCreate(&pool, &props) != cudaSuccess) return nullptr;
  uint64_t keep = ~0ull;
  cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
  pools.emplace(dev, pool);
  return pool;
}

// Workspace buffer that grows on demand. Growth is stream-ordered (cudaFreeAsync /
// cudaMallocFromPoolAsync on the workspace's stream): no device-wide synchronisation inside a
// search call, and the old buffer is released only after the work queued before it. Once a
// graph was captured on the stream, growth is refused instead (the graph would keep the old
// address).
template <typename T>
struct DevBuf {
  T* ptr = nullptr;
  size_t cap = 0;  // elements
  const WsState* ws = nullptr;
  int ensure(size_t n) {
    if (n <= cap) return TSV_OK;
    cudaStream_t st = ws ? ws->stream : nullptr;
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(st, &cs);
    if ((ws && ws->captured) || cs != cudaStreamCaptureStatusNone)
      return fail(TSV_ERR_CAPACITY,
                  "workspace would grow from %zu to %zu elements on a stream with a captured "
                  "CUDA graph; run the largest shape on it before capturing", cap, n);
    if (ptr) cudaFreeAsync(ptr, st);
    ptr = nullptr;
    cap = 0;
    cudaMemPool_t pool = workspace_pool();
    cudaError_t e = pool == nullptr ? cudaErrorMemoryAllocation
                                    : cudaMallocFromPoolAsync(reinterpret_cast<void**>(&ptr),
                                                              std::max<size_t>(n, 1) * sizeof(T),
                                                              pool, st);
    if (e != cudaSuccess) return cuda_fail(e, "workspace cudaMallocAsync");
    cap = n;
    return TSV_OK;
  }
  void release() {
    if (ptr) cudaFree(ptr);
    ptr = nullptr;
    cap = 0;
  }
};

struct Workspace {
  WsState state;
  DevBuf<int32_t> counter;     // lockstep progress counters + shared admission floors
  DevBuf<uint16_t> qbuf;       // bf16 staged queries
  DevBuf<float> qhi, qlo;      // fp32-mode query planes
  DevBuf<float> seed_s, tau0;  // threshold seeding for k > 32
  DevBuf<int32_t> seed_i;
  DevBuf<float> part_s;        // partial lists
  DevBuf<int32_t> part_i;
  DevBuf<float> cand_s;        // append mode: candidate rows [B][kCandCap]
  DevBuf<int32_t> cand_i;
  DevBuf<int32_t> cand_cnt;    // [B] candidate counts, then the overflow flag
  DevBuf<tsv::ScanItem> items;
  DevBuf<uint64_t> rr_keys;     // K3 split mode: per-block top-k keys
  DevBuf<int32_t> rr_arrive;    // K3 split mode: per-question arrival counters (kept zero)
  DevBuf<uint64_t> sm_keys;     // K2s: per-row-block top-k keys
  DevBuf<int64_t> qrows;        // segment kernel: per-query (row_begin, row_end)
  DevBuf<int32_t> roffs;        // K3 over per-query indexes: row offsets uploaded from the host
  std::vector<int64_t> host_rows;
  DevBuf<int32_t> sm_arrive;    // K2s: per-query-group arrival counters (kept zero)
  std::vector<tsv::ScanItem> host_items;
  // Pinned staging for the item table so its upload is a true async copy. A ring of slots,
  // each with an event marking when its upload drained: the host only waits when it laps a
  // slot whose copy is still queued, so back-to-back segmented searches stay asynchronous.
  static constexpr int kPinnedSlots = 4;
  struct Pinned {
    tsv::ScanItem* ptr = nullptr;
    size_t cap = 0;
    cudaEvent_t done = nullptr;
  } pinned[kPinnedSlots];
  int pinned_next = 0;
  // Item tables uploaded by CUDA graphs captured on this stream: the captured memcpy node
  // reads its host source at every replay, so each capture takes a region of this pinned pool
  // (allocated by the first segmented search outside capture; pinned allocation is not
  // permitted while a stream captures) and keeps it for the workspace's lifetime.
  static constexpr size_t kCapturePoolBytes = 1 << 20;
  uint8_t* capture_pool = nullptr;
  size_t capture_used = 0;
  void bind(cudaStream_t st) {  // first use on stream st
    state.stream = st;
    for (auto* b : {&counter, &seed_i, &part_i, &cand_i, &cand_cnt}) b->ws = &state;
    for (auto* b : {&qhi, &qlo, &seed_s, &tau0, &part_s, &cand_s}) b->ws = &state;
    qbuf.ws = &state;
    items.ws = &state;
    rr_keys.ws = &state;
    rr_arrive.ws = &state;
    sm_keys.ws = &state;
    qrows.ws = &state;
    roffs.ws = &state;
    sm_arrive.ws = &state;
  }
  void release() {
    for (auto& s : pinned) {
      if (s.ptr) cudaFreeHost(s.ptr);
      if (s.done) cudaEventDestroy(s.done);
      s = Pinned{};
    }
    if (capture_pool) cudaFreeHost(capture_pool);
    capture_pool = nullptr;
    capture_used = 0;
    counter.release();
    qbuf.release();
    qhi.release();
    qlo.release();
    seed_s.release();
    tau0.release();
    seed_i.release();
    part_s.release();
    part_i.release();
    cand_s.release();
    cand_i.release();
    cand_cnt.release();
    items.release();
    rr_keys.release();
    rr_arrive.release();
  }
};

struct TimedLaunch {
  cudaEvent_t a, b;
};

}  // namespace

struct tsv_index {
  int device = 0;
  int dim = 0;
  int metric = TSV_METRIC_IP;
  int64_t cap_rows = 0;
  int64_t rows = 0;
  bool owns = true;
  void* arena = nullptr;
  CUtensorMap tmap_c;
  int storage = TSV_BF16;       // TSV_F32: arena = tf32 "hi" plane, arena_lo = residual plane
  float* arena_lo = nullptr;
  CUtensorMap tmap_c_lo;
  int num_sms = 148;
  std::map<cudaStream_t, Workspace> ws;
  bool timing = false;
  std::vector<TimedLaunch> timed;
  double timed_ms = 0.0;
  int64_t timed_launches = 0;
};

namespace {

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) == cudaSuccess && prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur;
    if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
  }
};

// The (index, stream) workspace; a call issued while the stream captures a CUDA graph pins
// the workspace's buffers for good (see DevBuf).
Workspace& ws_for(tsv_index* idx, cudaStream_t st) {
  auto it = idx->ws.find(st);
  if (it == idx->ws.end()) {
    it = idx->ws.emplace(st, Workspace()).first;
    it->second.bind(st);
  }
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(st, &cs) == cudaSuccess && cs != cudaStreamCaptureStatusNone)
    it->second.state.captured = true;
  return it->second;
}

int check_dim(int dim) {
  if (dim <= 0 || dim % 8 != 0 || dim > 16384)
    return fail(TSV_ERR_CONFIG, "dim must be a positive multiple of 8 (<= 16384), got %d", dim);
  return TSV_OK;
}

int check_dtype(int dt) {
  if (dt != TSV_BF16 && dt != TSV_F32) return fail(TSV_ERR_CONFIG, "unknown dtype %d", dt);
  return TSV_OK;
}

constexpr int kMergeCap = 16384;  // candidates per query the merge kernel sorts in smem
constexpr int kMinTilesPerRange = 1;
constexpr int64_t kMinSampleTiles = 8;  // tiles per sample-pass item (TSV_SAMPLE_MIN_TILES)
constexpr int64_t kWideMinRows = 1 << 19;  // scans shorter than this keep 128-row tiles (TSV_WIDE=0/1 forces)

bool env_flag(const char* name) {
  const char* v = getenv(name);
  return v != nullptr && v[0] != '\0' && v[0] != '0';
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

// bf16 query matrix the scan reads: the caller's buffer when it is already bf16 and needs no
// normalisation, otherwise a staged copy converted (and normalised for cosine) by K5.
int stage_queries(tsv_index* idx, Workspace& w, const void* q, int q_dtype, int64_t B,
                  cudaStream_t st, const void** out) {
  const bool need = q_dtype != TSV_BF16 || idx->metric == TSV_METRIC_COSINE || !aligned16(q);
  if (!need) {
    *out = q;
    return TSV_OK;
  }
  int rc = w.qbuf.ensure(static_cast<size_t>(B) * idx->dim);
  if (rc) return rc;
  int e = tsv::launch_normalize(q, q_dtype == TSV_F32, B, idx->dim,
                                idx->metric == TSV_METRIC_COSINE, w.qbuf.ptr, st);
  if (e) return cuda_fail(static_cast<cudaError_t>(e), "normalize queries");
  g_launches++;
  *out = w.qbuf.ptr;
  return TSV_OK;
}

// Query tensor maps are cached per (pointer, rows, dim): staged queries live in a stable
// per-stream workspace buffer, so repeated searches skip the host-side encode.
int query_map(const void* qb, int64_t B, int dim, CUtensorMap* out, int box_rows = tsv::kBlockM) {
  struct Key {
    const void* p;
    int64_t b;
    int d;
    int box;
    bool operator<(const Key& o) const {
      return p != o.p ? p < o.p : (b != o.b ? b < o.b : (d != o.d ? d < o.d : box < o.box));
    }
  };
  static std::mutex mu;
  static std::map<Key, CUtensorMap> cache;
  std::lock_guard<std::mutex> lock(mu);
  auto it = cache.find(Key{qb, B, dim, box_rows});
  if (it != cache.end()) {
    *out = it->second;
    return TSV_OK;
  }
  int rc = encode_rows_map(out, qb, B, dim, box_rows);
  if (rc) return rc;
  if (cache.size() > 4096) cache.clear();
  cache.emplace(Key{qb, B, dim, box_rows}, *out);
  return TSV_OK;
}

int run_scan(tsv_index* idx, int mb, int kcap, const void* qb, int64_t B, tsv::ScanParams& p,
             int grid, cudaStream_t st) {
  // One query group of fewer than 128 queries: load only its rows (TMA out-of-bounds fill of
  // the rest of a 128-row box costs as much as real rows and halves the HBM-bound scan rate).
  // (Segmented searches set a_rows from their largest query group before the call.)
  if (p.a_rows == 0 && (mb == 1 || mb == tsv::kWideMode) && p.items == nullptr && B < tsv::kBlockM &&
      !getenv("TSV_FULL_QBOX"))
    p.a_rows = static_cast<int>((B + 7) & ~7);
  if (getenv("TSV_FULL_QBOX")) p.a_rows = 0;
  CUtensorMap tq;
  int rc = query_map(qb, B, idx->dim, &tq, p.a_rows ? p.a_rows : tsv::kBlockM);
  if (rc) return rc;
  TimedLaunch tl{};
  if (idx->timing) {
    TSV_CUDA(cudaEventCreate(&tl.a), "cudaEventCreate");
    TSV_CUDA(cudaEventCreate(&tl.b), "cudaEventCreate");
    TSV_CUDA(cudaEventRecord(tl.a, st), "cudaEventRecord");
  }
  int e = tsv::launch_scan_topk(mb, kcap, tq, idx->tmap_c, p, grid, st);
  if (e) return cuda_fail(static_cast<cudaError_t>(e), "scan_topk launch");
  g_launches++;
  if (idx->timing) {
    TSV_CUDA(cudaEventRecord(tl.b, st), "cudaEventRecord");
    idx->timed.push_back(tl);
  }
  return TSV_OK;
}

// fp32 mode: split queries into (hi, lo) planes (normalised for cosine).
int stage_queries_f32(tsv_index* idx, Workspace& w, const void* q, int q_dtype, int64_t B,
                      cudaStream_t st) {
  int rc = w.qhi.ensure(static_cast<size_t>(B) * idx->dim);
  if (rc) return rc;
  rc = w.qlo.ensure(static_cast<size_t>(B) * idx->dim);
  if (rc) return rc;
  int e = tsv::launch_split_f32(q, q_dtype == TSV_F32, B, idx->dim,
                                idx->metric == TSV_METRIC_COSINE, w.qhi.ptr, w.qlo.ptr, st);
  if (e) return cuda_fail(static_cast<cudaError_t>(e), "split queries");
  g_launches++;
  return TSV_OK;
}

int run_scan_f32(tsv_index* idx, int kcap, Workspace& w, int64_t B, tsv::ScanParams& p, int grid,
                 cudaStream_t st) {
  CUtensorMap tq, tq_lo;
  int rc = encode_rows_map(&tq, w.qhi.ptr, B, idx->dim, tsv::kBlockM, true);
  if (rc) return rc;
  rc = encode_rows_map(&tq_lo, w.qlo.ptr, B, idx->dim, tsv::kBlockM, true);
  if (rc) return rc;
  TimedLaunch tl{};
  if (idx->timing) {
    TSV_CUDA(cudaEventCreate(&tl.a), "cudaEventCreate");
    TSV_CUDA(cudaEventCreate(&tl.b), "cudaEventCreate");
    TSV_CUDA(cudaEventRecord(tl.a, st), "cudaEventRecord");
  }
  int e = tsv::launch_scan_topk_tf32(kcap, tq, idx->tmap_c, tq_lo, idx->tmap_c_lo, p, grid, st);
  if (e) return cuda_fail(static_cast<cudaError_t>(e), "scan_topk (fp32) launch");
  g_launches++;
  if (idx->timing) {
    TSV_CUDA(cudaEventRecord(tl.b, st), "cudaEventRecord");
    idx->timed.push_back(tl);
  }
  return TSV_OK;
}

}  // namespace

extern "C" {

int tsv_abi_version(void) { return TSV_ABI_VERSION; }
const char* tsv_last_error(void) { return g_last_error.c_str(); }
int64_t tsv_launch_count(void) { return g_launches.load(); }

static int create_common(int device, int dim, int metric, tsv_index** out) {
  if (out == nullptr) return fail(TSV_ERR_ARGUMENT, "out is null");
  *out = nullptr;
  int rc = check_dim(dim);
  if (rc) return rc;
  if (metric != TSV_METRIC_IP && metric != TSV_METRIC_COSINE)
    return fail(TSV_ERR_CONFIG, "unknown metric %d", metric);
  int ndev = 0;
  TSV_CUDA(cudaGetDeviceCount(&ndev), "cudaGetDeviceCount");
  if (device < 0 || device >= ndev) return fail(TSV_ERR_CONFIG, "bad device %d", device);
  int major = 0;
  TSV_CUDA(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device),
           "cudaDeviceGetAttribute");
  if (major != 10) return fail(TSV_ERR_DEVICE, "device %d is not sm_100 (major=%d)", device, major);
  return TSV_OK;
}

}  // extern "C"

// Live indexes, so that destroying a library stream can drop the per-stream workspaces it left
// in them: the driver reuses stream handles, and a later stream with the same handle must not
// inherit a workspace (possibly marked as captured by a CUDA graph) of a destroyed one.
static std::mutex g_index_mu;
static std::set<tsv_index*> g_indexes;
static void register_index(tsv_index* idx) {
  std::lock_guard<std::mutex> lock(g_index_mu);
  g_indexes.insert(idx);
}
static void unregister_index(tsv_index* idx) {
  std::lock_guard<std::mutex> lock(g_index_mu);
  g_indexes.erase(idx);
}

extern "C" {

int tsv_index_create2(int device, int dim, int metric, int storage, int64_t cap_rows,
                      tsv_index** out) {
  int rc = create_common(device, dim, metric, out);
  if (rc) return rc;
  if (storage != TSV_BF16 && storage != TSV_F32 && storage != TSV_BF16_TILED)
    return fail(TSV_ERR_CONFIG, "unknown storage %d", storage);
  if (cap_rows <= 0 || cap_rows > (int64_t(1) << 31) - 1)
    return fail(TSV_ERR_CAPACITY, "cap_rows out of range: %lld", (long long)cap_rows);
  DeviceGuard g(device);
  auto* idx = new tsv_index();
  idx->device = device;
  idx->dim = dim;
  idx->metric = metric;
  idx->storage = storage;
  idx->cap_rows = cap_rows;
  cudaDeviceGetAttribute(&idx->num_sms, cudaDevAttrMultiProcessorCount, device);
  const bool f32 = storage == TSV_F32;
  const bool tiled = storage == TSV_BF16_TILED;
  const size_t bytes = tiled ? static_cast<size_t>((cap_rows + 127) / 128) * 128 *
                                   ((dim + 63) / 64) * 64 * 2
                             : static_cast<size_t>(cap_rows) * dim * (f32 ? 4 : 2);
  cudaError_t e = cudaMalloc(&idx->arena, bytes);
  if (e == cudaSuccess && f32) e = cudaMalloc(&idx->arena_lo, bytes);
  if (e == cudaSuccess && tiled) e = cudaMemset(idx->arena, 0, bytes);  // zero k padding
  if (e != cudaSuccess) {
    if (idx->arena) cudaFree(idx->arena);
    delete idx;
    return cuda_fail(e, "arena cudaMalloc");
  }
  rc = tiled ? encode_tiled_map(&idx->tmap_c, idx->arena, cap_rows, dim)
             : encode_rows_map(&idx->tmap_c, idx->arena, cap_rows, dim, tsv::kBlockN, f32);
  if (!rc && f32) rc = encode_rows_map(&idx->tmap_c_lo, idx->arena_lo, cap_rows, dim, tsv::kBlockN, true);
  if (rc) {
    cudaFree(idx->arena);
    if (idx->arena_lo) cudaFree(idx->arena_lo);
    delete idx;
    return rc;
  }
  register_index(idx);
  *out = idx;
  return TSV_OK;
}

int tsv_index_create(int device, int dim, int metric, int64_t cap_rows, tsv_index** out) {
  return tsv_index_create2(device, dim, metric, TSV_BF16, cap_rows, out);
}

int tsv_index_create_view(int device, int dim, int metric, const void* rows_dev, int64_t n_rows,
                          tsv_index** out) {
  int rc = create_common(device, dim, metric, out);
  if (rc) return rc;
  if (rows_dev == nullptr || !aligned16(rows_dev))
    return fail(TSV_ERR_ARGUMENT, "rows_dev must be a 16-byte aligned device pointer");
  if (n_rows <= 0 || n_rows > (int64_t(1) << 31) - 1)
    return fail(TSV_ERR_CAPACITY, "n_rows out of range: %lld", (long long)n_rows);
  DeviceGuard g(device);
  auto* idx = new tsv_index();
  idx->device = device;
  idx->dim = dim;
  idx->metric = metric;
  idx->cap_rows = n_rows;
  idx->rows = n_rows;
  idx->owns = false;
  idx->arena = const_cast<void*>(rows_dev);
  cudaDeviceGetAttribute(&idx->num_sms, cudaDevAttrMultiProcessorCount, device);
  rc = encode_rows_map(&idx->tmap_c, idx->arena, n_rows, dim, tsv::kBlockN);
  if (rc) {
    delete idx;
    return rc;
  }
  register_index(idx);
  *out = idx;
  return TSV_OK;
}

int tsv_index_destroy(tsv_index* idx) {
  if (idx == nullptr) return TSV_OK;
  unregister_index(idx);
  DeviceGuard g(idx->device);
  for (auto& kv : idx->ws) kv.second.release();
  for (auto& t : idx->timed) {
    cudaEventDestroy(t.a);
    cudaEventDestroy(t.b);
  }
  if (idx->owns && idx->arena) cudaFree(idx->arena);
  if (idx->arena_lo) cudaFree(idx->arena_lo);
  delete idx;
  return TSV_OK;
}

int tsv_index_append(tsv_index* idx, const void* rows_dev, int src_dtype, int64_t n,
                     int64_t* first_row, void* stream) {
  if (idx == nullptr) return fail(TSV_ERR_ARGUMENT, "index is null");
  if (!idx->owns) return fail(TSV_ERR_CONFIG, "cannot append to a view index");
  int rc = check_dtype(src_dtype);
  if (rc) return rc;
  if (n < 0) return fail(TSV_ERR_CAPACITY, "negative row count");
  if (idx->rows + n > idx->cap_rows)
    return fail(TSV_ERR_CAPACITY, "arena overflow: %lld + %lld > %lld", (long long)idx->rows,
                (long long)n, (long long)idx->cap_rows);
  if (first_row) *first_row = idx->rows;
  if (n == 0) return TSV_OK;
  if (rows_dev == nullptr) return fail(TSV_ERR_ARGUMENT, "rows_dev is null");
  DeviceGuard g(idx->device);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (idx->storage == TSV_F32) {
    const size_t off = static_cast<size_t>(idx->rows) * idx->dim;
    int e = tsv::launch_split_f32(rows_dev, src_dtype == TSV_F32, n, idx->dim,
                                  idx->metric == TSV_METRIC_COSINE,
                                  static_cast<float*>(idx->arena) + off, idx->arena_lo + off, st);
    if (e) return cuda_fail(static_cast<cudaError_t>(e), "split rows");
    g_launches++;
    idx->rows += n;
    return TSV_OK;
  }
  if (idx->storage == TSV_BF16_TILED) {
    int e = tsv::launch_scatter_tiled(rows_dev, src_dtype == TSV_F32, n, idx->dim,
                                      idx->metric == TSV_METRIC_COSINE, idx->arena, idx->rows, st);
    if (e) return cuda_fail(static_cast<cudaError_t>(e), "scatter rows");
    g_launches++;
    idx->rows += n;
    return TSV_OK;
  }
  void* dst = static_cast<uint8_t*>(idx->arena) + static_cast<size_t>(idx->rows) * idx->dim * 2;
  if (src_dtype == TSV_BF16 && idx->metric == TSV_METRIC_IP) {
    TSV_CUDA(cudaMemcpyAsync(dst, rows_dev, static_cast<size_t>(n) * idx->dim * 2,
                             cudaMemcpyDeviceToDevice, st),
             "append copy");
  } else {
    int e = tsv::launch_normalize(rows_dev, src_dtype == TSV_F32, n, idx->dim,
                                  idx->metric == TSV_METRIC_COSINE, dst, st);
    if (e) return cuda_fail(static_cast<cudaError_t>(e), "normalize rows");
    g_launches++;
  }
  idx->rows += n;
  return TSV_OK;
}

int tsv_index_reserve(tsv_index* idx, int64_t n, int64_t* first_row) {
  if (idx == nullptr) return fail(TSV_ERR_ARGUMENT, "index is null");
  if (!idx->owns) return fail(TSV_ERR_CONFIG, "cannot reserve rows in a view index");
  if (n < 0) return fail(TSV_ERR_CAPACITY, "negative row count");
  if (idx->rows + n > idx->cap_rows)
    return fail(TSV_ERR_CAPACITY, "arena overflow: %lld + %lld > %lld", (long long)idx->rows,
                (long long)n, (long long)idx->cap_rows);
  if (first_row) *first_row = idx->rows;
  idx->rows += n;
  return TSV_OK;
}

int tsv_index_truncate(tsv_index* idx, int64_t n) {
  if (idx == nullptr) return fail(TSV_ERR_ARGUMENT, "index is null");
  if (n < 0 || n > idx->rows) return fail(TSV_ERR_CAPACITY, "bad truncate length");
  if (!idx->owns) return fail(TSV_ERR_CONFIG, "cannot truncate a view index");
  idx->rows = n;
  return TSV_OK;
}

int64_t tsv_index_rows(const tsv_index* idx) { return idx ? idx->rows : -1; }
int tsv_index_dim(const tsv_index* idx) { return idx ? idx->dim : -1; }
int tsv_index_metric(const tsv_index* idx) { return idx ? idx->metric : -1; }
const void* tsv_index_data(const tsv_index* idx) { return idx ? idx->arena : nullptr; }
const void* tsv_index_data_lo(const tsv_index* idx) { return idx ? idx->arena_lo : nullptr; }
int tsv_index_storage(const tsv_index* idx) { return idx ? idx->storage : -1; }

int tsv_index_set_timing(tsv_index* idx, int enable) {
  if (idx == nullptr) return fail(TSV_ERR_ARGUMENT, "index is null");
  idx->timing = enable != 0;
  return TSV_OK;
}

int tsv_index_scan_time(tsv_index* idx, double* total_ms, int64_t* launches) {
  if (idx == nullptr) return fail(TSV_ERR_ARGUMENT, "index is null");
  DeviceGuard g(idx->device);
  for (auto& t : idx->timed) {
    TSV_CUDA(cudaEventSynchronize(t.b), "cudaEventSynchronize");
    float ms = 0.f;
    TSV_CUDA(cudaEventElapsedTime(&ms, t.a, t.b), "cudaEventElapsedTime");
    idx->timed_ms += ms;
    idx->timed_launches++;
    cudaEventDestroy(t.a);
    cudaEventDestroy(t.b);
  }
  idx->timed.clear();
  if (total_ms) *total_ms = idx->timed_ms;
  if (launches) *launches = idx->timed_launches;
  idx->timed_ms = 0.0;
  idx->timed_launches = 0;
  return TSV_OK;
}

// Variants of one search pass (the seeded k > 32 search chains several).
struct PassOpts {
  const float* tau0 = nullptr;    // per-query admission floor (seeded passes)
  int list_cap = 0;               // > 0: per-range lists of list_cap < k entries (sample pass;
                                  // the merge returns the best k of their union)
  const int32_t* gate = nullptr;  // every launch skipped on the device unless *gate != 0
  bool append = false;            // candidate mode (needs tau0): rows above tau0 go to
                                  // per-query candidate rows, a select kernel writes the top
                                  // k; an overflow sets the flag at cand_cnt[B], which the
                                  // caller passes as the gate of a list-mode fallback pass
  bool staged = false;            // q_dev is already the bf16 (normalised) matrix the scan reads
  int sample_div = 0;             // > 1: every range scans only its first 1/sample_div
  int cand_cap = 0;               // candidate-row capacity (0 = tsv::kCandCap)
};

// Range lockstep (workers scanning one corpus range for different query groups stay within a
// few tiles of each other, so each corpus tile comes from HBM once and from L2 for the rest).
// Measured: with range-major rounds (short items) a clear win up to 4 query groups
// (B <= 1024) and a loss with 8 or 16 (every pair waits for the slowest of many partners,
// while their drift over a short item fits in L2 anyway); with one round of long items (the
// single-CTA fp32 mode, 8 groups of 128) it still wins (91.5-94.1 vs 98-99 ms).
constexpr int kMaxLockGroups = 4;
// Candidate mode keeps kCandCap (score, id) slots per query (64 KB): beyond this many queries
// per call the k > 32 search uses shared-memory lists instead.
constexpr int kMaxCandQueries = 32768;
bool lockstep_wanted(int nqg, int num_items, int units, bool range_major) {
  if (env_flag("TSV_NO_LOCKSTEP")) return false;
  if (range_major && nqg > kMaxLockGroups && !env_flag("TSV_LOCKSTEP_ALL")) return false;
  return nqg > 1 && (num_items <= units || range_major);
}

static int search_impl(tsv_index* idx, const void* q_dev, int q_dtype, int B, int k,
                       int64_t row_beg, int64_t row_end, int32_t id_offset, float* scores_dev,
                       int32_t* ids_dev, void* stream, const PassOpts& o = PassOpts()) {
  const float* tau0 = o.tau0;
  const int list_cap = o.list_cap;
  const int32_t* gate = o.gate;
  const bool append = o.append, staged = o.staged;
  const int sample_div = o.sample_div;
  const int cand_cap = o.cand_cap > 0 ? o.cand_cap : tsv::kCandCap;
  if (idx == nullptr) return fail(TSV_ERR_ARGUMENT, "index is null");
  int rc = check_dtype(q_dtype);
  if (rc) return rc;
  if (B <= 0) return fail(TSV_ERR_CAPACITY, "empty batch");
  if (k <= 0) return fail(TSV_ERR_CONFIG, "k must be >= 1");
  if (tsv::scan_kcap_for(k) == 0)
    return fail(TSV_ERR_CONFIG, "k=%d exceeds the supported maximum (128)", k);
  int kcap = list_cap > 0 ? tsv::scan_kcap_for(list_cap) : tsv::scan_kcap_for(k);
  if (q_dev == nullptr || scores_dev == nullptr || ids_dev == nullptr)
    return fail(TSV_ERR_ARGUMENT, "null buffer");
  if (row_beg < 0 || row_end > idx->rows || row_beg > row_end)
    return fail(TSV_ERR_CAPACITY, "row range [%lld, %lld) outside arena of %lld rows",
                (long long)row_beg, (long long)row_end, (long long)idx->rows);
  DeviceGuard g(idx->device);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  Workspace& w = ws_for(idx, st);
  const bool f32 = idx->storage == TSV_F32;
  const bool tiled = idx->storage == TSV_BF16_TILED;
  if (tiled && row_beg % 128 != 0)
    return fail(TSV_ERR_CONFIG, "tiled index: row_beg must be a multiple of 128");
  if (f32 && kcap > tsv::kMaxKF32)
    return fail(TSV_ERR_CONFIG, "k=%d exceeds the fp32-mode maximum (%d)", k, tsv::kMaxKF32);

  const void* qb = staged ? q_dev : nullptr;
  if (!staged) {
    rc = f32 ? stage_queries_f32(idx, w, q_dev, q_dtype, B, st)
             : stage_queries(idx, w, q_dev, q_dtype, B, st, &qb);
    if (rc) return rc;
  }

  // B > 128: CTA-pair kernel (256 queries x 256 rows per pair tile); otherwise one CTA per
  // 128-query group with 128-row tiles.
  const bool pair = !f32 && B > tsv::kBlockM && !env_flag("TSV_NO_PAIR");
  const int64_t n = row_end - row_beg;
  // 96 < B <= 128 on long scans with register lists: 256-row corpus tiles (M=128 x N=256 MMAs;
  // the query operand is re-read from L2 once per 256 corpus rows instead of 128). ~3% at
  // 10M x 1024, B=128, where the scan runs at the power cap; even at B <= 96 and in
  // candidate mode, so those keep 128-row tiles.
  bool wide = !pair && !f32 && B > 96 && n >= kWideMinRows && kcap <= tsv::kMaxRegK && !append;
  if (const char* e = getenv("TSV_WIDE")) wide = !pair && !f32 && atoi(e) != 0 &&
                                                 (kcap <= tsv::kMaxRegK || append);
  const int mb = pair ? tsv::kPairMode : (wide ? tsv::kWideMode : 1);
  const int qg = pair ? tsv::kPairQG : tsv::kBlockM;
  const int tile_rows = pair ? tsv::kPairTileRows : (wide ? tsv::kWideTileRows : tsv::kBlockN);
  const int units = pair ? idx->num_sms / 2 : idx->num_sms;  // concurrent workers
  const int nqg = (B + qg - 1) / qg;
  const int64_t tiles = std::max<int64_t>(1, (n + tile_rows - 1) / tile_rows);
  // Ranges per query group: one round over all workers when nqg divides them. Otherwise the
  // pair kernel takes its items in range-major order over whole rounds (nqg * R a multiple of
  // the worker count, at most 4 rounds): every pair is busy and each range's query groups
  // still run in the same round, so the corpus is streamed once. Failing that, one round if
  // it idles at most ~3% of the workers, else two full rounds (corpus streamed twice).
  int R = std::max(1, units / nqg);
  bool range_major = false;
  if (pair && nqg > 1 && (units % nqg != 0 || getenv("TSV_ROUNDS")) &&
      !env_flag("TSV_NO_RANGE_MAJOR")) {
    // Whole rounds need nqg * R to be a multiple of the worker count: rounds must be a
    // multiple of base = lcm(units, nqg) / units. About 4 rounds measured best at B=1024 (finer
    // items even out the pairs' finishing times), so take the multiple of base nearest 4.
    const int base = nqg / std::gcd(units, nqg);
    int rounds = base * std::max(1, (4 + base / 2) / base);
    if (const char* e = getenv("TSV_ROUNDS")) rounds = atoi(e);
    if (const char* e = getenv("TSV_SAMPLE_ROUNDS"); e && sample_div > 1) rounds = atoi(e);
    if (rounds >= 2 && (static_cast<int64_t>(rounds) * units) % nqg == 0 &&
        tiles >= 8 * (static_cast<int64_t>(rounds) * units / nqg)) {
      R = rounds * units / nqg;
      range_major = true;
    }
  }
  if (!range_major && nqg * R < units * 97 / 100 && (2 * units) % nqg == 0) R = 2 * units / nqg;
  if (const char* e = getenv("TSV_SCAN_RANGES")) {
    R = std::max(1, atoi(e));
    range_major = false;
  }
  // at least kMinTilesPerRange tiles per range: tiny scans gain nothing from more workers, and
  // every extra range is one more list for the merge
  R = static_cast<int>(std::min<int64_t>(R, std::max<int64_t>(1, tiles / kMinTilesPerRange)));
  // A sample pass reads 1/sample_div of every range: keep >= kMinSampleTiles tiles per item
  // where that still fills a round, or per-item pipeline fill and first-tile insertions
  // dominate it (1M rows at B=1024 would otherwise run 4 rounds of 296 two-tile items).
  // The floor is the k-th best of the ranges' lists together, so keep >= 2k list entries.
  if (sample_div > 1) {
    const int r0 = R;
    int64_t min_tiles = kMinSampleTiles;
    if (const char* e = getenv("TSV_SAMPLE_MIN_TILES")) min_tiles = std::max(1, atoi(e));
    // (never below one round of items: with few workers busy the sample costs more than the
    // per-item overhead it saves, e.g. 300K x 4096 or 100K-row scans)
    const int64_t one_round = (units + nqg - 1) / nqg;
    R = static_cast<int>(std::min<int64_t>(
        R, std::max<int64_t>(one_round, tiles / (sample_div * min_tiles))));
    R = std::max(R, std::min(r0, (2 * k + kcap - 1) / kcap));
    if (nqg * R > units && nqg * R < 2 * units) R = std::max(1, units / nqg);  // one round
  }
  if (!append) R = std::min(R, kMergeCap / kcap);  // the range merge holds R * kcap per query
  // Sample pass: 16-entry lists when the ranges' lists still hold >= 2k entries. The floor is
  // the k-th best of their union (exact whenever no range holds more than 16 of the sample's
  // top k); shorter lists halve the first-tile insertion chains of the short sample items.
  if (sample_div > 1 && kcap == tsv::kMaxRegK && static_cast<int64_t>(R) * 16 >= 2 * k &&
      !env_flag("TSV_SAMPLE_LIST32"))
    kcap = 16;
  const int num_items = nqg * R;
  const int grid = pair ? 2 * std::min(num_items, units) : std::min(num_items, units);

  tsv::ScanParams p{};
  p.items = nullptr;
  p.num_items = num_items;
  p.B = B;
  p.R = R;
  p.id_offset = id_offset;
  p.row_beg = row_beg;
  p.row_end = row_end;
  p.tau0 = tau0;
  p.gate = gate;
  p.sample_div = sample_div;
  if (range_major) p.flags |= tsv::kFlagRangeMajor;
  const int kb_elems = f32 ? 32 : tsv::kBlockK;  // elements per 128-byte k-block row
  p.num_kb = (idx->dim + kb_elems - 1) / kb_elems;
  if (tiled) p.flags |= tsv::kFlagTiled;
  if (const char* e = getenv("TSV_DIAG"))
    p.flags |= atoi(e) & (tsv::kFlagDiagNoFilter | tsv::kFlagDiagNoStream |
                          tsv::kFlagDiagNoQueryLoad | tsv::kFlagDiagSetupOnly);

  if (append) {
    const bool lock = lockstep_wanted(nqg, num_items, units, range_major);
    const size_t nc = lock ? static_cast<size_t>(num_items) : 0;
    rc = w.cand_s.ensure(static_cast<size_t>(B) * cand_cap);
    if (!rc) rc = w.cand_i.ensure(static_cast<size_t>(B) * cand_cap);
    if (!rc) rc = w.cand_cnt.ensure(static_cast<size_t>(B) + 1);
    if (!rc && lock) rc = w.counter.ensure(nc);
    if (rc) return rc;
    TSV_CUDA(cudaMemsetAsync(w.cand_cnt.ptr, 0, sizeof(int32_t) * (B + 1), st), "count reset");
    if (lock) {
      TSV_CUDA(cudaMemsetAsync(w.counter.ptr, 0, sizeof(int32_t) * nc, st), "progress reset");
      p.counter = w.counter.ptr;
      p.flags |= tsv::kFlagLockstep;
      if (const char* e = getenv("TSV_LOCK_WINDOW")) p.lock_window = std::max(1, atoi(e));
    }
    p.out_k = 0;
    p.out_scores = w.cand_s.ptr;
    p.out_ids = w.cand_i.ptr;
    p.cand_count = w.cand_cnt.ptr;
    p.cand_cap = cand_cap;
    rc = run_scan(idx, mb, tsv::kAppendCap, qb, B, p, grid, st);
    if (rc) return rc;
    int e = tsv::launch_cand_select(w.cand_s.ptr, w.cand_i.ptr, w.cand_cnt.ptr, cand_cap, B, k,
                                    scores_dev, ids_dev, w.cand_cnt.ptr + B, st);
    if (e) return cuda_fail(static_cast<cudaError_t>(e), "candidate select launch");
    g_launches++;
    return TSV_OK;
  }
  const bool lock = lockstep_wanted(nqg, num_items, units, range_major);
  const bool floor = R > 1 && !env_flag("TSV_NO_FLOOR");
  if (lock || floor) {  // one zeroed buffer: [progress counters][per-query floors]
    const size_t nc = lock ? static_cast<size_t>(num_items) : 0;
    const size_t n = nc + (floor ? static_cast<size_t>(B) : 0);
    rc = w.counter.ensure(n);
    if (rc) return rc;
    TSV_CUDA(cudaMemsetAsync(w.counter.ptr, 0, sizeof(int32_t) * n, st), "progress reset");
    if (lock) {
      p.counter = w.counter.ptr;
      p.flags |= tsv::kFlagLockstep;
      if (const char* e = getenv("TSV_LOCK_WINDOW")) p.lock_window = std::max(1, atoi(e));
    }
    if (floor) p.floor_g = reinterpret_cast<uint32_t*>(w.counter.ptr + nc);
  }
  if (R == 1 && kcap >= k) {
    p.out_k = k;
    p.out_scores = scores_dev;
    p.out_ids = ids_dev;
    return f32 ? run_scan_f32(idx, kcap, w, B, p, grid, st)
               : run_scan(idx, mb, kcap, qb, B, p, grid, st);
  }
  p.out_k = kcap;
  rc = w.part_s.ensure(static_cast<size_t>(R) * B * kcap);
  if (rc) return rc;
  rc = w.part_i.ensure(static_cast<size_t>(R) * B * kcap);
  if (rc) return rc;
  p.out_scores = w.part_s.ptr;
  p.out_ids = w.part_i.ptr;
  rc = f32 ? run_scan_f32(idx, kcap, w, B, p, grid, st)
           : run_scan(idx, mb, kcap, qb, B, p, grid, st);
  if (rc) return rc;
  int e = tsv::launch_merge_topk(w.part_s.ptr, w.part_i.ptr, R, B, kcap, B, k, scores_dev, ids_dev,
                                 st, 0, gate);
  if (e) return cuda_fail(static_cast<cudaError_t>(e), "merge launch");
  g_launches++;
  return TSV_OK;
}

// Development: TSV_SMALL_TRACE=1 makes the one-launch searches (K2s / K2t) stamp per-block phase
// times; each launch then synchronises and prints min / median / max per phase to stderr.
static unsigned long long* small_trace_buffer() {
  static unsigned long long* trace = nullptr;
  if (!env_flag("TSV_SMALL_TRACE")) return nullptr;
  if (trace == nullptr && cudaMalloc(&trace, sizeof(unsigned long long) * 8 * 4096) != cudaSuccess)
    return nullptr;
  cudaMemset(trace, 0, sizeof(unsigned long long) * 8 * 4096);
  return trace;
}

static void small_trace_print(unsigned long long* trace, int nb_total, cudaStream_t st) {
  if (trace == nullptr || nb_total > 4096) return;
  std::vector<unsigned long long> h(8 * static_cast<size_t>(nb_total));
  cudaMemcpyAsync(h.data(), trace, h.size() * 8, cudaMemcpyDeviceToHost, st);
  cudaStreamSynchronize(st);
  unsigned long long t0 = ~0ull;
  for (int b = 0; b < nb_total; ++b) t0 = std::min(t0, h[b * 8]);
  fprintf(stderr, "one-launch search trace (%d blocks, ns from first entry): phase min/med/max\n",
          nb_total);
  for (int ph = 0; ph < 8; ++ph) {
    std::vector<long long> v;
    for (int b = 0; b < nb_total; ++b)
      if (h[b * 8 + ph]) v.push_back(static_cast<long long>(h[b * 8 + ph] - t0));
    if (v.empty()) continue;
    std::sort(v.begin(), v.end());
    fprintf(stderr, "  phase %d: n=%zu min %lld med %lld max %lld\n", ph, v.size(), v.front(),
            v[v.size() / 2], v.back());
  }
}

// ~128 rows per block (16 per warp: about three ring refills), at most one block per SM over
// all query groups: few partial lists, so the last block merges them in one L2 round trip.
static int small_scan_blocks(const tsv_index* idx, int groups, int64_t n) {
  return std::max(1, static_cast<int>(std::min<int64_t>((n + 127) / 128,
                                                        std::max(1, idx->num_sms / groups))));
}

// K2s routing: few queries over a short row range (the scan's fixed costs dominate; at most a
// few L2-resident passes over the rows, one per query group) -> one small-scan launch.
static bool small_scan_fits(const tsv_index* idx, int B, int k, int64_t n) {
  if (idx->storage == TSV_F32 || idx->dim % 8 != 0 || idx->dim > 1024 || k > 16 || B > 64 ||
      n <= 0 || n > 65536 || env_flag("TSV_NO_SMALL"))
    return false;
  // where K2s beats the general scan (scripts/small_route_sweep.py, CUDA-graph replays): up to
  // 4k rows at any k <= 16, up to 16k rows at k <= 8; longer ranges or k = 16 lose to it
  // (e.g. 10k x 384, B=1, k=16: 37 vs 27 us) — those shapes go to K2t or the general scan
  if (!(n <= 4096 || (n <= 16384 && k <= 8)) && !env_flag("TSV_FORCE_SMALL")) return false;
  const int qg = tsv::small_scan_qg(idx->dim);
  const int groups = (B + qg - 1) / qg;
  if (n * idx->dim * 2 * groups > (int64_t(48) << 20)) return false;
  const int64_t per = (n + small_scan_blocks(idx, groups, n) - 1) / small_scan_blocks(idx, groups, n);
  return per <= 1024;  // the block's scores stay in shared memory ([QG][per] fp32)
}

static int small_scan(tsv_index* idx, const void* q_dev, int q_dtype, int B, int k,
                      int64_t row_beg, int64_t row_end, int32_t id_offset, float* scores_dev,
                      int32_t* ids_dev, cudaStream_t st) {
  if (row_beg < 0 || row_end > idx->rows || row_beg > row_end)
    return fail(TSV_ERR_CAPACITY, "row range [%lld, %lld) outside arena of %lld rows",
                (long long)row_beg, (long long)row_end, (long long)idx->rows);
  Workspace& w = ws_for(idx, st);
  const int qg = tsv::small_scan_qg(idx->dim);
  const int groups = (B + qg - 1) / qg;
  const int64_t n = row_end - row_beg;
  const int nblk = small_scan_blocks(idx, groups, n);
  int rc = w.sm_keys.ensure(static_cast<size_t>(groups) * nblk * qg * k);
  if (rc) return rc;
  const size_t had = w.sm_arrive.cap;
  rc = w.sm_arrive.ensure(static_cast<size_t>(groups));
  if (rc) return rc;
  if (w.sm_arrive.cap != had)
    TSV_CUDA(cudaMemsetAsync(w.sm_arrive.ptr, 0, w.sm_arrive.cap * sizeof(int32_t), st),
             "arrivals reset");
  const int nb_total = nblk * groups;
  unsigned long long* trace = small_trace_buffer();
  int e = tsv::launch_small_scan(idx->arena, idx->dim, idx->storage == TSV_BF16_TILED, q_dev,
                                 q_dtype == TSV_F32, idx->metric == TSV_METRIC_COSINE, B, row_beg,
                                 row_end, id_offset, k, nblk, w.sm_keys.ptr, w.sm_arrive.ptr,
                                 scores_dev, ids_dev, st, trace);
  if (e) return cuda_fail(static_cast<cudaError_t>(e), "small scan launch");
  g_launches++;
  small_trace_print(trace, nb_total, st);
  return TSV_OK;
}

// K2t routing: the tensor-core one-launch search (bf16 arena, B <= 64, k <= 16, at
// most two 128-row tiles per SM so the last CTA's merge stays short, queries <= 64 KB of smem).
static bool tiny_scan_fits(const tsv_index* idx, int B, int k, int64_t n) {
  if ((idx->storage != TSV_BF16 && idx->storage != TSV_BF16_TILED) || idx->dim % 8 != 0 ||
      k > 16 || B > 64 || n <= 0 ||
      env_flag("TSV_NO_TINY") || env_flag("TSV_NO_SMALL"))
    return false;
  const int nq = B <= 16 ? 16 : (B <= 32 ? 32 : 64);
  const int num_kb = (idx->dim + 63) / 64;
  const int stages = std::min(num_kb, 6);
  const int64_t tiles = tsv::tiny_scan_blocks(n);
  // the queries (raw fp32 at most) and the tiles' lists (merged in the ring) must fit on chip
  return tiles <= 2 * idx->num_sms && num_kb * nq * 128 <= 64 * 1024 &&
         int64_t(B) * idx->dim * 4 <= 64 * 1024 && tiles * k <= 512 &&
         int64_t(B) * tiles * k * 8 <= stages * 16384;  // the last CTA stages every list in the ring
}

static int tiny_scan(tsv_index* idx, const void* q_dev, int q_dtype, int B, int k,
                     int64_t row_beg, int64_t row_end, int32_t id_offset, float* scores_dev,
                     int32_t* ids_dev, cudaStream_t st) {
  if (row_beg < 0 || row_end > idx->rows || row_beg > row_end)
    return fail(TSV_ERR_CAPACITY, "row range [%lld, %lld) outside arena of %lld rows",
                (long long)row_beg, (long long)row_end, (long long)idx->rows);
  Workspace& w = ws_for(idx, st);
  const int nblk = tsv::tiny_scan_blocks(row_end - row_beg);
  int rc = w.sm_keys.ensure(static_cast<size_t>(B) * nblk * k);
  if (rc) return rc;
  const size_t had = w.sm_arrive.cap;
  rc = w.sm_arrive.ensure(1);
  if (rc) return rc;
  if (w.sm_arrive.cap != had)
    TSV_CUDA(cudaMemsetAsync(w.sm_arrive.ptr, 0, w.sm_arrive.cap * sizeof(int32_t), st),
             "arrivals reset");
  unsigned long long* trace = small_trace_buffer();
  // The cross-tile merge as a second grid launched behind the scan (PDL): the queries' merges
  // run in parallel on B SMs instead of one after another in the scan's last CTA (C1 in a CUDA
  // graph: 16.0 vs 20.0 us). Issued call by call the extra launch costs more host time than
  // it saves on the device (back-to-back calls: 25.1 vs 20.2 us), so the split is used where
  // launches are free: under graph capture. TSV_TINY_SPLIT=0/1 forces either.
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(st, &cap);
  int split = cap != cudaStreamCaptureStatusNone ? 1 : 0;
  if (const char* v = getenv("TSV_TINY_SPLIT")) split = atoi(v) != 0;
  int e = tsv::launch_tiny_scan(idx->tmap_c, q_dev, q_dtype == TSV_F32,
                                idx->metric == TSV_METRIC_COSINE, B, idx->dim, row_beg, row_end,
                                id_offset, k, w.sm_keys.ptr, w.sm_arrive.ptr, scores_dev, ids_dev,
                                st, trace, idx->storage == TSV_BF16_TILED, split);
  if (e) return cuda_fail(static_cast<cudaError_t>(e), "tiny scan launch");
  g_launches += split ? 2 : 1;  // scan (+ merge grid, PDL-overlapped)
  small_trace_print(trace, nblk, st);
  return TSV_OK;
}

int tsv_search(tsv_index* idx, const void* q_dev, int q_dtype, int B, int k, int64_t row_beg,
               int64_t row_end, int32_t id_offset, float* scores_dev, int32_t* ids_dev,
               void* stream) {
  if (idx != nullptr && B > 0 && k > 0 && q_dev != nullptr && scores_dev != nullptr &&
      ids_dev != nullptr && check_dtype(q_dtype) == TSV_OK &&
      tiny_scan_fits(idx, B, k, row_end - row_beg) && aligned16(q_dev) &&
      (idx->storage != TSV_BF16_TILED || row_beg % 128 == 0)) {
    DeviceGuard g(idx->device);
    return tiny_scan(idx, q_dev, q_dtype, B, k, row_beg, row_end, id_offset, scores_dev, ids_dev,
                     reinterpret_cast<cudaStream_t>(stream));
  }
  if (idx != nullptr && B > 0 && k > 0 && q_dev != nullptr && scores_dev != nullptr &&
      ids_dev != nullptr && check_dtype(q_dtype) == TSV_OK &&
      small_scan_fits(idx, B, k, row_end - row_beg) &&
      (idx->storage != TSV_BF16_TILED || row_beg % 128 == 0)) {
    DeviceGuard g(idx->device);
    return small_scan(idx, q_dev, q_dtype, B, k, row_beg, row_end, id_offset, scores_dev, ids_dev,
                      reinterpret_cast<cudaStream_t>(stream));
  }
  // k > 32: a top-k over a 1/32 (k > 100: 1/16) sample of the rows bounds every query's final k-th score from
  // below; the main scan then only has to keep rows above that floor (candidate mode), which
  // keeps the result exact. Ranges of at most kCandCap rows skip the sample: every row is a
  // candidate and no candidate row can overflow. (Shared-memory lists, the fallback, insert
  // one candidate per warp step and are slow when many rows qualify.)
  const int kcap = tsv::scan_kcap_for(k);
  const int64_t n = row_end - row_beg;
  if (idx != nullptr && kcap > tsv::kMaxRegK && idx->storage != TSV_F32 && B > 0 &&
      B <= kMaxCandQueries && n > 0 && !env_flag("TSV_NO_SEED")) {
    // Sample fraction: about frac * k rows then clear the floor, so 1/32 up to k = 100 (<= ~3.2k
    // candidates per query, 2.5x inside kCandCap) and 1/16 above (~2k at k = 128). 10M x 1024:
    // k=64 16.6-17.3 -> 16.1-16.2 ms, k=100 17.0-17.1 -> 16.6-16.7 ms at 1/32.
    int frac = k <= 100 ? 32 : 16;
    if (const char* e = getenv("TSV_SEED_FRAC")) frac = std::max(2, atoi(e));
    DeviceGuard g(idx->device);
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    Workspace& w = ws_for(idx, st);
    int rc = check_dtype(q_dtype);
    if (!rc && q_dev == nullptr) rc = fail(TSV_ERR_ARGUMENT, "null buffer");
    if (!rc) rc = w.seed_s.ensure(static_cast<size_t>(B) * k);
    if (!rc) rc = w.seed_i.ensure(static_cast<size_t>(B) * k);
    if (!rc) rc = w.tau0.ensure(static_cast<size_t>(B));
    if (rc) return rc;
    // stage (convert / normalise) the queries once for the three passes
    const void* qb = nullptr;
    rc = stage_queries(idx, w, q_dev, q_dtype, B, st, &qb);
    if (rc) return rc;
    if (n <= tsv::kCandCap) {
      PassOpts all_rows;
      all_rows.append = true;
      all_rows.staged = true;
      all_rows.cand_cap = static_cast<int>((n + 31) & ~int64_t(31));
      return search_impl(idx, qb, TSV_BF16, B, k, row_beg, row_end, id_offset, scores_dev,
                         ids_dev, stream, all_rows);
    }
    // Sample pass with 32-entry register lists per corpus range, each range scanning only the
    // first 1/frac of its tiles (a sample spread over the whole row range, so a corpus stored
    // in topical order still yields a tight floor): the k-th best of the union of those lists
    // is a lower bound of the final k-th score (the union holds k distinct rows scoring at
    // least that much) and, with the top rows spread over many ranges, usually equal to the
    // sample's k-th best.
    PassOpts sample_pass;
    sample_pass.list_cap = tsv::kMaxRegK;
    sample_pass.staged = true;
    if (env_flag("TSV_SEED_CONTIG")) {  // A/B: the first 1/frac of the rows instead
      rc = search_impl(idx, qb, TSV_BF16, B, k, row_beg, row_beg + ((n / frac + 255) / 256) * 256,
                       0, w.seed_s.ptr, w.seed_i.ptr, stream, sample_pass);
    } else {
      sample_pass.sample_div = frac;
      rc = search_impl(idx, qb, TSV_BF16, B, k, row_beg, row_end, 0, w.seed_s.ptr, w.seed_i.ptr,
                       stream, sample_pass);
    }
    if (rc) return rc;
    int e = tsv::launch_seed_floor(w.seed_s.ptr, w.seed_i.ptr, B, k, w.tau0.ptr, st);
    if (e) return cuda_fail(static_cast<cudaError_t>(e), "seed floor");
    g_launches++;
    PassOpts list_pass;  // k-entry shared-memory lists admitting only rows above tau0
    list_pass.tau0 = w.tau0.ptr;
    list_pass.staged = true;
    if (env_flag("TSV_NO_APPEND"))
      return search_impl(idx, qb, TSV_BF16, B, k, row_beg, row_end, id_offset, scores_dev,
                         ids_dev, stream, list_pass);
    // Main pass in candidate mode: the register-list pipeline depth (no shared-memory lists),
    // every row above tau0 appended to its query's candidate row, exact top-k selected from
    // those. If any candidate row overflowed, the device-gated list-mode pass recomputes the
    // batch (exact either way; no host round trip decides it).
    PassOpts cand_pass = list_pass;
    cand_pass.append = true;
    rc = search_impl(idx, qb, TSV_BF16, B, k, row_beg, row_end, id_offset, scores_dev, ids_dev,
                     stream, cand_pass);
    if (rc) return rc;
    list_pass.gate = w.cand_cnt.ptr + B;
    return search_impl(idx, qb, TSV_BF16, B, k, row_beg, row_end, id_offset, scores_dev,
                       ids_dev, stream, list_pass);
  }
  return search_impl(idx, q_dev, q_dtype, B, k, row_beg, row_end, id_offset, scores_dev, ids_dev,
                     stream);
}

// Host table -> device buffer, asynchronously: through a ring of pinned slots (the host waits
// only when it laps a slot whose copy is still queued), or, under CUDA-graph capture, from a
// never-reused region of the per-stream capture pool (the captured memcpy node reads its host
// source at every replay).
static int upload_table(Workspace& w, const void* host, size_t bytes, void* dev, cudaStream_t st) {
  cudaStreamCaptureStatus capturing = cudaStreamCaptureStatusNone;
  TSV_CUDA(cudaStreamIsCapturing(st, &capturing), "cudaStreamIsCapturing");
  if (capturing != cudaStreamCaptureStatusNone) {
    const size_t need = (bytes + 255) & ~size_t(255);
    if (w.capture_pool == nullptr || w.capture_used + need > Workspace::kCapturePoolBytes)
      return fail(TSV_ERR_CAPACITY,
                  "segmented search under graph capture: run it once on this stream outside "
                  "the capture first (pinned pool %s)",
                  w.capture_pool == nullptr ? "not allocated" : "exhausted");
    uint8_t* hp = w.capture_pool + w.capture_used;
    w.capture_used += need;
    std::memcpy(hp, host, bytes);
    TSV_CUDA(cudaMemcpyAsync(dev, hp, bytes, cudaMemcpyHostToDevice, st),
             "table upload (graph capture)");
    return TSV_OK;
  }
  if (w.capture_pool == nullptr)
    TSV_CUDA(cudaMallocHost(&w.capture_pool, Workspace::kCapturePoolBytes), "cudaMallocHost");
  Workspace::Pinned& slot = w.pinned[w.pinned_next];
  w.pinned_next = (w.pinned_next + 1) % Workspace::kPinnedSlots;
  if (slot.done == nullptr)
    TSV_CUDA(cudaEventCreateWithFlags(&slot.done, cudaEventDisableTiming), "cudaEventCreate");
  else
    TSV_CUDA(cudaEventSynchronize(slot.done), "cudaEventSynchronize");
  const size_t items = (bytes + sizeof(tsv::ScanItem) - 1) / sizeof(tsv::ScanItem);
  if (items > slot.cap) {
    if (slot.ptr) cudaFreeHost(slot.ptr);
    slot.ptr = nullptr;
    TSV_CUDA(cudaMallocHost(&slot.ptr, items * 2 * sizeof(tsv::ScanItem)), "cudaMallocHost");
    slot.cap = items * 2;
  }
  std::memcpy(slot.ptr, host, bytes);
  TSV_CUDA(cudaMemcpyAsync(dev, slot.ptr, bytes, cudaMemcpyHostToDevice, st), "table upload");
  TSV_CUDA(cudaEventRecord(slot.done, st), "cudaEventRecord");
  return TSV_OK;
}

int tsv_search_segmented(tsv_index* idx, const void* q_dev, int q_dtype, int nseg,
                         const int32_t* seg_q_beg, const int64_t* seg_row_beg,
                         const int64_t* seg_row_end, int k, int local_ids, float* scores_dev,
                         int32_t* ids_dev, void* stream) {
  if (idx == nullptr) return fail(TSV_ERR_ARGUMENT, "index is null");
  int rc = check_dtype(q_dtype);
  if (rc) return rc;
  if (nseg <= 0) return fail(TSV_ERR_CAPACITY, "empty batch");
  if (seg_q_beg == nullptr || seg_row_beg == nullptr || seg_row_end == nullptr)
    return fail(TSV_ERR_ARGUMENT, "null segment table");
  if (k <= 0) return fail(TSV_ERR_CONFIG, "k must be >= 1");
  const int kcap = tsv::scan_kcap_for(k);
  if (kcap == 0) return fail(TSV_ERR_CONFIG, "k=%d exceeds the supported maximum (128)", k);
  const int B = seg_q_beg[nseg] - seg_q_beg[0];
  if (seg_q_beg[0] != 0 || B <= 0) return fail(TSV_ERR_CAPACITY, "bad query offsets");
  int max_q = 0;
  int64_t max_rows = 0;
  for (int s = 0; s < nseg; ++s) {
    if (seg_q_beg[s + 1] < seg_q_beg[s]) return fail(TSV_ERR_ARGUMENT, "query offsets decrease");
    if (seg_row_beg[s] < 0 || seg_row_end[s] > idx->rows || seg_row_beg[s] > seg_row_end[s])
      return fail(TSV_ERR_CAPACITY, "segment %d row range outside arena", s);
    max_q = std::max(max_q, seg_q_beg[s + 1] - seg_q_beg[s]);
    max_rows = std::max<int64_t>(max_rows, seg_row_end[s] - seg_row_beg[s]);
  }
  DeviceGuard g(idx->device);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  // one segment: a plain range search (ids shifted to the segment when local), which routes
  // short ranges to the one-launch kernels
  if (nseg == 1 && seg_row_beg[0] <= INT32_MAX)
    return tsv_search(idx, q_dev, q_dtype, B, k, seg_row_beg[0], seg_row_end[0],
                      local_ids ? static_cast<int32_t>(-seg_row_beg[0]) : 0, scores_dev, ids_dev,
                      stream);
  Workspace& w = ws_for(idx, st);
  const bool f32 = idx->storage == TSV_F32;
  const bool tiled = idx->storage == TSV_BF16_TILED;
  // short segments (<= 1024 rows each, the per-query indexes of a topology-aware batch): one
  // launch of the segment kernel in search-only mode, a block per query over its own segment
  if (!f32 && idx->dim <= 2048 && idx->dim % 8 == 0 && max_rows <= tsv::kFusedSegMaxRows &&
      !env_flag("TSV_NO_SEG_FUSED")) {
    std::vector<int64_t>& qr = w.host_rows;
    qr.resize(2 * static_cast<size_t>(B));
    for (int s_ = 0; s_ < nseg; ++s_)
      for (int qi = seg_q_beg[s_]; qi < seg_q_beg[s_ + 1]; ++qi) {
        qr[2 * qi] = seg_row_beg[s_];
        qr[2 * qi + 1] = seg_row_end[s_];
      }
    rc = w.qrows.ensure(qr.size());
    if (rc) return rc;
    rc = upload_table(w, qr.data(), qr.size() * sizeof(int64_t), w.qrows.ptr, st);
    if (rc) return rc;
    const int mr = static_cast<int>(std::max<int64_t>(max_rows, 1));
    int e = tsv::launch_search_rerank_seg(idx->arena, idx->rows, idx->dim, tiled, q_dev, nullptr,
                                          q_dtype == TSV_F32, idx->metric == TSV_METRIC_COSINE,
                                          w.qrows.ptr, B, mr, k, 0, local_ids, scores_dev, ids_dev,
                                          nullptr, nullptr, st);
    if (e) return cuda_fail(static_cast<cudaError_t>(e), "segment search launch");
    g_launches++;
    return TSV_OK;
  }
  for (int s_ = 0; tiled && s_ < nseg; ++s_)
    if (seg_row_beg[s_] % 128 != 0)
      return fail(TSV_ERR_CONFIG, "tiled index: segment %d must start at a multiple of 128", s_);
  if (f32 && kcap > tsv::kMaxKF32)
    return fail(TSV_ERR_CONFIG, "k=%d exceeds the fp32-mode maximum (%d)", k, tsv::kMaxKF32);
  const void* qb = nullptr;
  rc = f32 ? stage_queries_f32(idx, w, q_dev, q_dtype, B, st)
           : stage_queries(idx, w, q_dev, q_dtype, B, st, &qb);
  if (rc) return rc;

  // k > 32 with every segment at most kCandCap rows: candidate mode with every row a candidate
  // (no lists, no overflow possible), as tsv_search does for small ranges
  const bool append_all = !f32 && kcap > tsv::kMaxRegK && max_rows <= tsv::kCandCap &&
                          B <= kMaxCandQueries && !env_flag("TSV_NO_SEED");
  const int mb = (!f32 && max_q > tsv::kBlockM && kcap <= tsv::kMaxRegK) ? 2 : 1;
  const int qg = mb * tsv::kBlockM;
  int units = 0;
  for (int s = 0; s < nseg; ++s) units += (seg_q_beg[s + 1] - seg_q_beg[s] + qg - 1) / qg;
  const int64_t max_tiles = std::max<int64_t>(1, (max_rows + tsv::kBlockN - 1) / tsv::kBlockN);
  int R = std::max(1, idx->num_sms / std::max(1, units));
  R = static_cast<int>(std::min<int64_t>(R, std::max<int64_t>(1, max_tiles / kMinTilesPerRange)));
  R = std::min(R, kMergeCap / kcap);

  auto& hi = w.host_items;
  hi.clear();
  for (int s = 0; s < nseg; ++s) {
    const int q0 = seg_q_beg[s], q1 = seg_q_beg[s + 1];
    const int64_t rb = seg_row_beg[s], re = seg_row_end[s];
    const int64_t tiles = (re - rb + tsv::kBlockN - 1) / tsv::kBlockN;
    for (int qs = q0; qs < q1; qs += qg) {
      for (int r = 0; r < R; ++r) {
        tsv::ScanItem it{};
        it.q_begin = qs;
        it.q_count = std::min(qg, q1 - qs);
        it.row_begin = rb + (tiles * r / R) * tsv::kBlockN;
        it.row_end = std::min(re, rb + (tiles * (r + 1) / R) * tsv::kBlockN);
        if (it.row_end < it.row_begin) it.row_end = it.row_begin;
        it.out_row = static_cast<int64_t>(r) * B + qs;
        it.id_offset = local_ids ? static_cast<int32_t>(-rb) : 0;
        hi.push_back(it);
      }
    }
  }
  rc = w.items.ensure(hi.size());
  if (rc) return rc;
  rc = upload_table(w, hi.data(), hi.size() * sizeof(tsv::ScanItem), w.items.ptr, st);
  if (rc) return rc;
  tsv::ScanParams p{};
  p.items = w.items.ptr;
  p.num_items = static_cast<int>(hi.size());
  // query box = the largest query group (rows past an item's own queries are never emitted)
  if (mb == 1 && !f32 && max_q < tsv::kBlockM) p.a_rows = (max_q + 7) & ~7;
  const int kb_elems = f32 ? 32 : tsv::kBlockK;
  p.num_kb = (idx->dim + kb_elems - 1) / kb_elems;
  if (tiled) p.flags |= tsv::kFlagTiled;
  const int grid = std::min(p.num_items, idx->num_sms);
  if (append_all) {
    const int cap = static_cast<int>((std::max<int64_t>(max_rows, 1) + 31) & ~int64_t(31));
    rc = w.cand_s.ensure(static_cast<size_t>(B) * cap);
    if (!rc) rc = w.cand_i.ensure(static_cast<size_t>(B) * cap);
    if (!rc) rc = w.cand_cnt.ensure(static_cast<size_t>(B) + 1);
    if (rc) return rc;
    TSV_CUDA(cudaMemsetAsync(w.cand_cnt.ptr, 0, sizeof(int32_t) * (B + 1), st), "count reset");
    p.out_k = 0;
    p.out_scores = w.cand_s.ptr;
    p.out_ids = w.cand_i.ptr;
    p.cand_count = w.cand_cnt.ptr;
    p.cand_cap = cap;
    rc = run_scan(idx, 1, tsv::kAppendCap, qb, B, p, grid, st);
    if (rc) return rc;
    int e = tsv::launch_cand_select(w.cand_s.ptr, w.cand_i.ptr, w.cand_cnt.ptr, cap, B, k,
                                    scores_dev, ids_dev, w.cand_cnt.ptr + B, st);
    if (e) return cuda_fail(static_cast<cudaError_t>(e), "candidate select launch");
    g_launches++;
    return TSV_OK;
  }
  if (R > 1 && !env_flag("TSV_NO_FLOOR")) {  // shared admission floors (see ScanParams)
    rc = w.counter.ensure(static_cast<size_t>(B));
    if (rc) return rc;
    TSV_CUDA(cudaMemsetAsync(w.counter.ptr, 0, sizeof(int32_t) * B, st), "floor reset");
    p.floor_g = reinterpret_cast<uint32_t*>(w.counter.ptr);
  }
  if (R == 1) {
    p.out_k = k;
    p.out_scores = scores_dev;
    p.out_ids = ids_dev;
    return f32 ? run_scan_f32(idx, kcap, w, B, p, grid, st)
               : run_scan(idx, mb, kcap, qb, B, p, grid, st);
  }
  p.out_k = kcap;
  rc = w.part_s.ensure(static_cast<size_t>(R) * B * kcap);
  if (rc) return rc;
  rc = w.part_i.ensure(static_cast<size_t>(R) * B * kcap);
  if (rc) return rc;
  p.out_scores = w.part_s.ptr;
  p.out_ids = w.part_i.ptr;
  rc = f32 ? run_scan_f32(idx, kcap, w, B, p, grid, st)
           : run_scan(idx, mb, kcap, qb, B, p, grid, st);
  if (rc) return rc;
  int e = tsv::launch_merge_topk(w.part_s.ptr, w.part_i.ptr, R, B, kcap, B, k, scores_dev, ids_dev,
                                 st);
  if (e) return cuda_fail(static_cast<cudaError_t>(e), "merge launch");
  g_launches++;
  return TSV_OK;
}

static int rerank_impl(tsv_index* idx, const void* q_dev, int q_dtype, int B,
                       const int32_t* cand_ids_dev, int C, const int32_t* row_offsets_dev, int k,
                       float* scores_dev, int32_t* ids_dev, void* stream) {
  if (idx == nullptr) return fail(TSV_ERR_ARGUMENT, "index is null");
  int rc = check_dtype(q_dtype);
  if (rc) return rc;
  if (B <= 0 || C <= 0) return fail(TSV_ERR_CAPACITY, "empty batch");
  if (C > 8192) return fail(TSV_ERR_CAPACITY, "candidate_count %d exceeds 8192", C);
  if (k <= 0) return fail(TSV_ERR_CONFIG, "k must be >= 1");
  if (q_dev == nullptr || cand_ids_dev == nullptr || scores_dev == nullptr || ids_dev == nullptr)
    return fail(TSV_ERR_ARGUMENT, "null buffer");
  DeviceGuard g(idx->device);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const void* q = q_dev;
  const float* q_lo = nullptr;
  int q_f32 = q_dtype == TSV_F32;
  const bool f32 = idx->storage == TSV_F32;
  if (f32) {  // exact fp32 question (hi + lo) against the hi + lo rows
    Workspace& w = ws_for(idx, st);
    rc = stage_queries_f32(idx, w, q_dev, q_dtype, B, st);
    if (rc) return rc;
    q = w.qhi.ptr;
    q_lo = w.qlo.ptr;
    q_f32 = 1;
  } else if (idx->metric == TSV_METRIC_COSINE) {
    Workspace& w = ws_for(idx, st);
    rc = stage_queries(idx, w, q_dev, q_dtype, B, st, &q);
    if (rc) return rc;
    q_f32 = 0;
  }
  const bool tiled = idx->storage == TSV_BF16_TILED;
  int e;
  // (rows up to 4 KB: two ring slots per warp fit next to the question vector)
  if (!f32 && idx->dim <= 2048 && !env_flag("TSV_RERANK_LDG")) {
    // bf16 arenas: gather pipelined through per-warp shared-memory rings (cp.async)
    const int splits = tsv::rerank_lists_splits(B, C, k, idx->dim, idx->num_sms);
    uint64_t* part_keys = nullptr;
    int32_t* arrivals = nullptr;
    if (splits > 1) {
      Workspace& w = ws_for(idx, st);
      rc = w.rr_keys.ensure(static_cast<size_t>(B) * splits * k);
      if (rc) return rc;
      const size_t had = w.rr_arrive.cap;
      rc = w.rr_arrive.ensure(static_cast<size_t>(B));
      if (rc) return rc;
      if (w.rr_arrive.cap != had)
        TSV_CUDA(cudaMemsetAsync(w.rr_arrive.ptr, 0, w.rr_arrive.cap * sizeof(int32_t), st),
                 "arrivals reset");
      part_keys = w.rr_keys.ptr;
      arrivals = w.rr_arrive.ptr;
    }
    e = tsv::launch_rerank_ring(idx->arena, idx->rows, idx->dim, q, q_f32, B, cand_ids_dev, C, k,
                                row_offsets_dev, scores_dev, ids_dev, st, tiled, splits,
                                part_keys, arrivals, idx->num_sms);
  } else {
    e = tsv::launch_rerank(f32 ? nullptr : idx->arena,
                           f32 ? static_cast<const float*>(idx->arena) : nullptr,
                           f32 ? idx->arena_lo : nullptr, idx->rows, idx->dim, q, q_lo, q_f32, B,
                           cand_ids_dev, C, k, scores_dev, ids_dev, st, tiled, row_offsets_dev);
  }
  if (e) return cuda_fail(static_cast<cudaError_t>(e), "rerank launch");
  g_launches++;
  return TSV_OK;
}

int tsv_search_rerank_segmented(tsv_index* idx, const void* q_search_dev,
                                const void* q_rerank_dev, int q_dtype, int B,
                                const int64_t* q_rows_dev, int max_rows, int k_search,
                                int k_rerank, int local_ids, float* search_scores_dev,
                                int32_t* search_ids_dev, float* rerank_scores_dev,
                                int32_t* rerank_ids_dev, void* stream) {
  if (idx == nullptr) return fail(TSV_ERR_ARGUMENT, "index is null");
  int rc = check_dtype(q_dtype);
  if (rc) return rc;
  if (B <= 0) return fail(TSV_ERR_CAPACITY, "empty batch");
  if (k_search <= 0 || k_rerank <= 0) return fail(TSV_ERR_CONFIG, "k must be >= 1");
  if (k_rerank > k_search)
    return fail(TSV_ERR_CONFIG, "k_rerank=%d exceeds k_search=%d", k_rerank, k_search);
  if (max_rows <= 0 || max_rows > tsv::kFusedSegMaxRows)
    return fail(TSV_ERR_CAPACITY, "max_rows=%d outside [1, %d] (use tsv_search_segmented + "
                "tsv_rerank for larger segments)", max_rows, tsv::kFusedSegMaxRows);
  if (idx->storage == TSV_F32 || idx->dim > 2048)
    return fail(TSV_ERR_CONFIG, "fused search+rerank needs a bf16 arena with dim <= 2048");
  if (q_search_dev == nullptr || q_rows_dev == nullptr || search_scores_dev == nullptr ||
      search_ids_dev == nullptr || rerank_scores_dev == nullptr || rerank_ids_dev == nullptr)
    return fail(TSV_ERR_ARGUMENT, "null buffer");
  DeviceGuard g(idx->device);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  int e = tsv::launch_search_rerank_seg(
      idx->arena, idx->rows, idx->dim, idx->storage == TSV_BF16_TILED, q_search_dev, q_rerank_dev,
      q_dtype == TSV_F32, idx->metric == TSV_METRIC_COSINE, q_rows_dev, B, max_rows, k_search,
      k_rerank, local_ids, search_scores_dev, search_ids_dev, rerank_scores_dev, rerank_ids_dev, st);
  if (e) return cuda_fail(static_cast<cudaError_t>(e), "search+rerank launch");
  g_launches++;
  return TSV_OK;
}

int tsv_search_rerank_segmented_host(tsv_index* idx, const void* q_search_dev,
                                     const void* q_rerank_dev, int q_dtype, int B,
                                     const int64_t* q_rows_host, int max_rows, int k_search,
                                     int k_rerank, int local_ids, float* search_scores_dev,
                                     int32_t* search_ids_dev, float* rerank_scores_dev,
                                     int32_t* rerank_ids_dev, void* stream) {
  if (idx == nullptr) return fail(TSV_ERR_ARGUMENT, "index is null");
  if (q_rows_host == nullptr) return fail(TSV_ERR_ARGUMENT, "q_rows_host is null");
  if (B <= 0) return fail(TSV_ERR_CAPACITY, "empty batch");
  DeviceGuard g(idx->device);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  Workspace& w = ws_for(idx, st);
  int rc = w.qrows.ensure(2 * static_cast<size_t>(B));
  if (rc) return rc;
  rc = upload_table(w, q_rows_host, 2 * static_cast<size_t>(B) * sizeof(int64_t), w.qrows.ptr, st);
  if (rc) return rc;
  return tsv_search_rerank_segmented(idx, q_search_dev, q_rerank_dev, q_dtype, B, w.qrows.ptr,
                                     max_rows, k_search, k_rerank, local_ids, search_scores_dev,
                                     search_ids_dev, rerank_scores_dev, rerank_ids_dev, stream);
}

int tsv_rerank(tsv_index* idx, const void* q_dev, int q_dtype, int B, const int32_t* cand_ids_dev,
               int C, int k, float* scores_dev, int32_t* ids_dev, void* stream) {
  return rerank_impl(idx, q_dev, q_dtype, B, cand_ids_dev, C, nullptr, k, scores_dev, ids_dev,
                     stream);
}

int tsv_rerank_segmented(tsv_index* idx, const void* q_dev, int q_dtype, int B,
                         const int32_t* cand_ids_dev, int C, const int32_t* row_offsets_dev, int k,
                         float* scores_dev, int32_t* ids_dev, void* stream) {
  if (row_offsets_dev == nullptr) return fail(TSV_ERR_ARGUMENT, "row_offsets_dev is null");
  return rerank_impl(idx, q_dev, q_dtype, B, cand_ids_dev, C, row_offsets_dev, k, scores_dev,
                     ids_dev, stream);
}

int tsv_rerank_segmented_host(tsv_index* idx, const void* q_dev, int q_dtype, int B,
                              const int32_t* cand_ids_dev, int C, const int32_t* row_offsets_host,
                              int k, float* scores_dev, int32_t* ids_dev, void* stream) {
  if (idx == nullptr) return fail(TSV_ERR_ARGUMENT, "index is null");
  if (row_offsets_host == nullptr) return fail(TSV_ERR_ARGUMENT, "row_offsets_host is null");
  if (B <= 0) return fail(TSV_ERR_CAPACITY, "empty batch");
  DeviceGuard g(idx->device);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  Workspace& w = ws_for(idx, st);
  int rc = w.roffs.ensure(static_cast<size_t>(B));
  if (rc) return rc;
  rc = upload_table(w, row_offsets_host, static_cast<size_t>(B) * sizeof(int32_t), w.roffs.ptr, st);
  if (rc) return rc;
  return rerank_impl(idx, q_dev, q_dtype, B, cand_ids_dev, C, w.roffs.ptr, k, scores_dev, ids_dev,
                     stream);
}

int tsv_merge_topk(const float* in_scores, const int32_t* in_ids, int lists, int B, int kin,
                   int kout, int dedup, float* out_scores, int32_t* out_ids, void* stream) {
  if (lists <= 0 || B <= 0 || kin <= 0 || kout <= 0) return fail(TSV_ERR_CAPACITY, "empty merge");
  if (static_cast<int64_t>(lists) * kin > 16384)
    return fail(TSV_ERR_CAPACITY, "merge of %d x %d candidates exceeds 16384", lists, kin);
  if (!in_scores || !in_ids || !out_scores || !out_ids) return fail(TSV_ERR_ARGUMENT, "null buffer");
  int e = tsv::launch_merge_topk(in_scores, in_ids, lists, B, kin, B, kout, out_scores, out_ids,
                                 reinterpret_cast<cudaStream_t>(stream), dedup);
  if (e) return cuda_fail(static_cast<cudaError_t>(e), "merge launch");
  g_launches++;
  return TSV_OK;
}

}  // extern "C"

struct tsv_peer_group {
  int device = 0, world = 1, rank = 0, max_b = 0, max_k = 0, num_sms = 148;
  void* buf = nullptr;
  std::vector<void*> peers;     // mapped base of every rank's buffer (own = buf)
  std::vector<bool> opened;     // peers mapped through IPC (closed on destroy)
  void** d_peers = nullptr;     // device copy of `peers`
  bool dirty = true;
  uint32_t epoch = 0;
  uint64_t timeout_ns = 60ull * 1000 * 1000 * 1000;  // a wait longer than this aborts the group
  uint32_t* err_host = nullptr;  // host-mapped error word written by the kernel (1 = aborted)
  uint32_t* err_dev = nullptr;
};

extern "C" {

int tsv_peer_create(int device, int world, int rank, int max_b, int max_k, tsv_peer_group** out) {
  if (out == nullptr) return fail(TSV_ERR_ARGUMENT, "out is null");
  *out = nullptr;
  if (world < 1 || world > 64 || rank < 0 || rank >= world)
    return fail(TSV_ERR_CONFIG, "bad world/rank %d/%d", world, rank);
  if (max_b <= 0 || max_k <= 0 || max_k > tsv::kMaxK)
    return fail(TSV_ERR_CAPACITY, "bad max_b/max_k %d/%d", max_b, max_k);
  DeviceGuard g(device);
  auto* pg = new tsv_peer_group();
  pg->device = device;
  pg->world = world;
  pg->rank = rank;
  pg->max_b = max_b;
  pg->max_k = max_k;
  cudaDeviceGetAttribute(&pg->num_sms, cudaDevAttrMultiProcessorCount, device);
  if (const char* t = getenv("TSV_PEER_TIMEOUT_MS"))
    pg->timeout_ns = static_cast<uint64_t>(std::max(1L, atol(t))) * 1000000ull;
  const size_t bytes = tsv::peer_buffer_bytes(world, max_b, max_k);
  cudaError_t e = cudaMalloc(&pg->buf, bytes);
  if (e == cudaSuccess) e = cudaMemset(pg->buf, 0, bytes);
  if (e == cudaSuccess) e = cudaMalloc(&pg->d_peers, sizeof(void*) * world);
  if (e == cudaSuccess)
    e = cudaHostAlloc(reinterpret_cast<void**>(&pg->err_host), sizeof(uint32_t), cudaHostAllocMapped);
  if (e == cudaSuccess) {
    *pg->err_host = 0;
    e = cudaHostGetDevicePointer(reinterpret_cast<void**>(&pg->err_dev), pg->err_host, 0);
  }
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    if (pg->buf) cudaFree(pg->buf);
    if (pg->d_peers) cudaFree(pg->d_peers);
    if (pg->err_host) cudaFreeHost(pg->err_host);
    delete pg;
    return cuda_fail(e, "peer buffer");
  }
  pg->peers.assign(world, nullptr);
  pg->opened.assign(world, false);
  pg->peers[rank] = pg->buf;
  *out = pg;
  return TSV_OK;
}

int tsv_peer_handle(tsv_peer_group* pg, void* handle_out, int* handle_bytes) {
  if (pg == nullptr || handle_out == nullptr) return fail(TSV_ERR_ARGUMENT, "null argument");
  DeviceGuard g(pg->device);
  cudaIpcMemHandle_t h;
  TSV_CUDA(cudaIpcGetMemHandle(&h, pg->buf), "cudaIpcGetMemHandle");
  std::memcpy(handle_out, &h, sizeof(h));
  if (handle_bytes) *handle_bytes = static_cast<int>(sizeof(h));
  return TSV_OK;
}

int tsv_peer_open(tsv_peer_group* pg, int peer, const void* handle) {
  if (pg == nullptr || handle == nullptr) return fail(TSV_ERR_ARGUMENT, "null argument");
  if (peer < 0 || peer >= pg->world) return fail(TSV_ERR_CONFIG, "bad peer %d", peer);
  if (peer == pg->rank) return TSV_OK;
  DeviceGuard g(pg->device);
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, sizeof(h));
  void* ptr = nullptr;
  TSV_CUDA(cudaIpcOpenMemHandle(&ptr, h, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
  pg->peers[peer] = ptr;
  pg->opened[peer] = true;
  pg->dirty = true;
  return TSV_OK;
}

int tsv_peer_attach(tsv_peer_group* pg, int peer, tsv_peer_group* other) {
  if (pg == nullptr || other == nullptr) return fail(TSV_ERR_ARGUMENT, "null argument");
  if (peer < 0 || peer >= pg->world || other->world != pg->world || other->rank != peer)
    return fail(TSV_ERR_CONFIG, "group of rank %d (world %d) cannot be peer %d of world %d",
                other->rank, other->world, peer, pg->world);
  if (other->max_b != pg->max_b || other->max_k != pg->max_k)
    return fail(TSV_ERR_CONFIG, "peer groups differ in max_b / max_k");
  if (peer == pg->rank) return TSV_OK;
  if (other->device != pg->device) {
    DeviceGuard g(pg->device);
    int can = 0;
    TSV_CUDA(cudaDeviceCanAccessPeer(&can, pg->device, other->device), "cudaDeviceCanAccessPeer");
    if (!can) return fail(TSV_ERR_DEVICE, "device %d cannot access device %d", pg->device, other->device);
    cudaError_t e = cudaDeviceEnablePeerAccess(other->device, 0);
    if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
    else if (e != cudaSuccess) return cuda_fail(e, "cudaDeviceEnablePeerAccess");
  }
  pg->peers[peer] = other->buf;
  pg->opened[peer] = false;  // not an IPC mapping: nothing to close
  pg->dirty = true;
  return TSV_OK;
}

int tsv_peer_allgather_merge(tsv_peer_group* pg, const float* local_s, const int32_t* local_i,
                             int B, int k, float* out_s, int32_t* out_i, void* stream) {
  if (pg == nullptr) return fail(TSV_ERR_ARGUMENT, "peer group is null");
  if (B <= 0 || k <= 0) return fail(TSV_ERR_CAPACITY, "empty exchange");
  if (B > pg->max_b || k > pg->max_k) return fail(TSV_ERR_CAPACITY, "exchange exceeds buffer");
  if (!local_s || !local_i || !out_s || !out_i) return fail(TSV_ERR_ARGUMENT, "null buffer");
  if (*reinterpret_cast<volatile uint32_t*>(pg->err_host) != 0)
    return fail(TSV_ERR_DEVICE, "peer exchange aborted: a peer did not deliver within %llu ms "
                "(dead rank or mismatched call sequence); recreate the group",
                (unsigned long long)(pg->timeout_ns / 1000000ull));
  for (int r = 0; r < pg->world; ++r)
    if (pg->peers[r] == nullptr) return fail(TSV_ERR_CONFIG, "peer %d not opened", r);
  DeviceGuard g(pg->device);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (pg->dirty) {
    TSV_CUDA(cudaMemcpyAsync(pg->d_peers, pg->peers.data(), sizeof(void*) * pg->world,
                             cudaMemcpyHostToDevice, st),
             "peer table upload");
    TSV_CUDA(cudaStreamSynchronize(st), "peer table upload");
    pg->dirty = false;
  }
  pg->epoch++;
  int e = tsv::launch_peer_exchange_merge(pg->d_peers, pg->rank, pg->world, B, k, pg->max_b,
                                          pg->max_k, pg->epoch, pg->timeout_ns, local_s, local_i,
                                          out_s, out_i, pg->err_dev, pg->num_sms, st);
  if (e) return cuda_fail(static_cast<cudaError_t>(e), "peer exchange launch");
  g_launches++;
  return TSV_OK;
}

int tsv_peer_set_timeout_ms(tsv_peer_group* pg, int64_t ms) {
  if (pg == nullptr) return fail(TSV_ERR_ARGUMENT, "peer group is null");
  if (ms <= 0) return fail(TSV_ERR_CONFIG, "timeout must be positive");
  pg->timeout_ns = static_cast<uint64_t>(ms) * 1000000ull;
  return TSV_OK;
}

int tsv_peer_status(tsv_peer_group* pg, int* aborted) {
  if (pg == nullptr || aborted == nullptr) return fail(TSV_ERR_ARGUMENT, "null argument");
  *aborted = *reinterpret_cast<volatile uint32_t*>(pg->err_host) != 0;
  if (*aborted)
    return fail(TSV_ERR_DEVICE, "peer exchange aborted: a peer did not deliver within %llu ms",
                (unsigned long long)(pg->timeout_ns / 1000000ull));
  return TSV_OK;
}

int tsv_peer_destroy(tsv_peer_group* pg) {
  if (pg == nullptr) return TSV_OK;
  DeviceGuard g(pg->device);
  cudaDeviceSynchronize();
  for (int r = 0; r < pg->world; ++r)
    if (pg->opened[r]) cudaIpcCloseMemHandle(pg->peers[r]);
  if (pg->err_host) cudaFreeHost(pg->err_host);
  if (pg->d_peers) cudaFree(pg->d_peers);
  if (pg->buf) cudaFree(pg->buf);
  delete pg;
  return TSV_OK;
}

}  // extern "C"

// ---- corpus-sharded search within one process (single process, several devices) ----
struct tsv_sharded {
  struct Shard {
    tsv_index* idx = nullptr;
    int64_t id_offset = 0;
    cudaStream_t stream = nullptr;  // the shard's own stream on its device
    cudaEvent_t done = nullptr;     // shard's part of a call finished (root waits on it)
    cudaEvent_t go = nullptr;       // recorded on the root stream: queries ready
    void* q = nullptr;              // query copy on the shard's device (root's own otherwise)
    float* part_s = nullptr;        // shard-local top-k, copied to root when not peer-writable
    int32_t* part_i = nullptr;
    bool direct = false;            // the shard writes straight into root memory (peer access)
  };
  std::vector<Shard> shards;
  int root = 0, dim = 0, max_b = 0, max_k = 0;
  float* gather_s = nullptr;  // [G][max_b][max_k] on root (slot stride B*k per call)
  int32_t* gather_i = nullptr;
};

extern "C" {

int tsv_sharded_create(tsv_index* const* shards, const int64_t* id_offsets, int nshards, int root,
                       int max_b, int max_k, tsv_sharded** out) {
  if (out == nullptr || shards == nullptr || id_offsets == nullptr)
    return fail(TSV_ERR_ARGUMENT, "null argument");
  *out = nullptr;
  if (nshards < 1 || nshards > 64) return fail(TSV_ERR_CONFIG, "bad shard count %d", nshards);
  if (max_b <= 0 || max_k <= 0 || max_k > tsv::kMaxK)
    return fail(TSV_ERR_CAPACITY, "bad max_b/max_k %d/%d", max_b, max_k);
  if (static_cast<int64_t>(nshards) * max_k > kMergeCap)
    return fail(TSV_ERR_CAPACITY, "%d shards x k=%d exceed the merge capacity", nshards, max_k);
  int ndev = 0;
  TSV_CUDA(cudaGetDeviceCount(&ndev), "cudaGetDeviceCount");
  if (root < 0 || root >= ndev) return fail(TSV_ERR_CONFIG, "bad root device %d", root);
  for (int g = 0; g < nshards; ++g) {
    if (shards[g] == nullptr) return fail(TSV_ERR_ARGUMENT, "shard %d is null", g);
    if (shards[g]->dim != shards[0]->dim || shards[g]->metric != shards[0]->metric ||
        shards[g]->storage != shards[0]->storage)
      return fail(TSV_ERR_CONFIG, "shard %d differs in dim / metric / storage", g);
  }
  auto* sh = new tsv_sharded();
  sh->root = root;
  sh->dim = shards[0]->dim;
  sh->max_b = max_b;
  sh->max_k = max_k;
  auto cleanup = [&](int rc) {
    tsv_sharded_destroy(sh);
    return rc;
  };
  sh->shards.resize(nshards);
  {
    DeviceGuard g(root);
    const size_t n = static_cast<size_t>(nshards) * max_b * max_k;
    cudaError_t e = cudaMalloc(&sh->gather_s, n * sizeof(float));
    if (e == cudaSuccess) e = cudaMalloc(&sh->gather_i, n * sizeof(int32_t));
    if (e != cudaSuccess) return cleanup(cuda_fail(e, "gather buffer"));
  }
  for (int g = 0; g < nshards; ++g) {
    auto& s = sh->shards[g];
    s.idx = shards[g];
    s.id_offset = id_offsets[g];
    const int dev = s.idx->device;
    DeviceGuard guard(dev);
    cudaError_t e = cudaStreamCreateWithFlags(&s.stream, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&s.done, cudaEventDisableTiming);
    if (e != cudaSuccess) return cleanup(cuda_fail(e, "shard stream"));
    {
      DeviceGuard rg(root);
      e = cudaEventCreateWithFlags(&s.go, cudaEventDisableTiming);
      if (e != cudaSuccess) return cleanup(cuda_fail(e, "shard event"));
    }
    if (dev != root) {
      int can = 0;
      cudaDeviceCanAccessPeer(&can, dev, root);
      if (can) {
        e = cudaDeviceEnablePeerAccess(root, 0);
        if (e == cudaErrorPeerAccessAlreadyEnabled) {
          cudaGetLastError();
          e = cudaSuccess;
        }
        s.direct = e == cudaSuccess;
        if (e != cudaSuccess) cudaGetLastError();
      }
      // queries arrive as bf16 or f32: room for the wider one
      e = cudaMalloc(&s.q, static_cast<size_t>(max_b) * sh->dim * 4);
      if (e == cudaSuccess && !s.direct) {
        e = cudaMalloc(&s.part_s, static_cast<size_t>(max_b) * max_k * sizeof(float));
        if (e == cudaSuccess) e = cudaMalloc(&s.part_i, static_cast<size_t>(max_b) * max_k * sizeof(int32_t));
      }
      if (e != cudaSuccess) return cleanup(cuda_fail(e, "shard buffers"));
    } else {
      s.direct = true;
    }
  }
  *out = sh;
  return TSV_OK;
}

int tsv_sharded_search(tsv_sharded* sh, const void* q_dev, int q_dtype, int B, int k,
                       float* scores_dev, int32_t* ids_dev, void* stream) {
  if (sh == nullptr) return fail(TSV_ERR_ARGUMENT, "sharded index is null");
  int rc = check_dtype(q_dtype);
  if (rc) return rc;
  if (B <= 0) return fail(TSV_ERR_CAPACITY, "empty batch");
  if (k <= 0) return fail(TSV_ERR_CONFIG, "k must be >= 1");
  if (B > sh->max_b || k > sh->max_k)
    return fail(TSV_ERR_CAPACITY, "B=%d / k=%d exceed the sharded index's %d / %d", B, k,
                sh->max_b, sh->max_k);
  if (q_dev == nullptr || scores_dev == nullptr || ids_dev == nullptr)
    return fail(TSV_ERR_ARGUMENT, "null buffer");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const int G = static_cast<int>(sh->shards.size());
  const size_t qbytes = static_cast<size_t>(B) * sh->dim * (q_dtype == TSV_F32 ? 4 : 2);
  const size_t plane = static_cast<size_t>(B) * k;
  // 1. every shard stream waits for the caller's queries (stream order on the root)
  {
    DeviceGuard g(sh->root);
    for (auto& s : sh->shards) TSV_CUDA(cudaEventRecord(s.go, st), "cudaEventRecord");
  }
  // 2. per shard: queries to its device, fused scan + top-k with global ids, results to root
  for (int gi = 0; gi < G; ++gi) {
    auto& s = sh->shards[gi];
    DeviceGuard g(s.idx->device);
    TSV_CUDA(cudaStreamWaitEvent(s.stream, s.go, 0), "cudaStreamWaitEvent");
    const void* q = q_dev;
    if (s.idx->device != sh->root) {
      TSV_CUDA(cudaMemcpyPeerAsync(s.q, s.idx->device, q_dev, sh->root, qbytes, s.stream),
               "query copy to shard");
      q = s.q;
    }
    float* os = s.direct ? sh->gather_s + gi * plane : s.part_s;
    int32_t* oi = s.direct ? sh->gather_i + gi * plane : s.part_i;
    rc = tsv_search(s.idx, q, q_dtype, B, k, 0, s.idx->rows,
                    static_cast<int32_t>(s.id_offset), os, oi, s.stream);
    if (rc) return rc;
    if (!s.direct) {
      TSV_CUDA(cudaMemcpyPeerAsync(sh->gather_s + gi * plane, sh->root, s.part_s, s.idx->device,
                                   plane * sizeof(float), s.stream), "result copy to root");
      TSV_CUDA(cudaMemcpyPeerAsync(sh->gather_i + gi * plane, sh->root, s.part_i, s.idx->device,
                                   plane * sizeof(int32_t), s.stream), "result copy to root");
    }
    TSV_CUDA(cudaEventRecord(s.done, s.stream), "cudaEventRecord");
  }
  // 3. the caller's stream waits for every shard, then merges G x k -> k (K4)
  DeviceGuard g(sh->root);
  for (auto& s : sh->shards) TSV_CUDA(cudaStreamWaitEvent(st, s.done, 0), "cudaStreamWaitEvent");
  int e = tsv::launch_merge_topk(sh->gather_s, sh->gather_i, G, B, k, B, k, scores_dev, ids_dev,
                                 st);
  if (e) return cuda_fail(static_cast<cudaError_t>(e), "merge launch");
  g_launches++;
  return TSV_OK;
}

int tsv_sharded_destroy(tsv_sharded* sh) {
  if (sh == nullptr) return TSV_OK;
  for (auto& s : sh->shards) {
    if (s.idx == nullptr) continue;
    DeviceGuard g(s.idx->device);
    if (s.stream) {
      cudaStreamSynchronize(s.stream);
      cudaStreamDestroy(s.stream);
    }
    if (s.done) cudaEventDestroy(s.done);
    if (s.go) cudaEventDestroy(s.go);
    if (s.q) cudaFree(s.q);
    if (s.part_s) cudaFree(s.part_s);
    if (s.part_i) cudaFree(s.part_i);
  }
  {
    DeviceGuard g(sh->root);
    if (sh->gather_s) cudaFree(sh->gather_s);
    if (sh->gather_i) cudaFree(sh->gather_i);
  }
  delete sh;
  return TSV_OK;
}

int tsv_stream_create(int device, void** out) {
  if (out == nullptr) return fail(TSV_ERR_ARGUMENT, "out is null");
  *out = nullptr;
  DeviceGuard g(device);
  cudaStream_t st = nullptr;
  TSV_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking), "cudaStreamCreate");
  *out = st;
  return TSV_OK;
}

int tsv_stream_destroy(void* stream) {
  if (stream == nullptr) return TSV_OK;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  TSV_CUDA(cudaStreamSynchronize(st), "cudaStreamSynchronize");
  {  // drop every index's workspace bound to this stream (see register_index)
    std::lock_guard<std::mutex> lock(g_index_mu);
    for (tsv_index* idx : g_indexes) {
      auto it = idx->ws.find(st);
      if (it == idx->ws.end()) continue;
      DeviceGuard g(idx->device);
      it->second.release();
      idx->ws.erase(it);
    }
  }
  TSV_CUDA(cudaStreamDestroy(st), "cudaStreamDestroy");
  return TSV_OK;
}

int tsv_normalize_rows(const void* src_dev, int src_dtype, int64_t n, int dim, int normalize,
                       void* dst_bf16_dev, void* stream) {
  int rc = check_dtype(src_dtype);
  if (rc) return rc;
  rc = check_dim(dim);
  if (rc) return rc;
  if (n < 0) return fail(TSV_ERR_CAPACITY, "negative row count");
  if (n == 0) return TSV_OK;
  if (!src_dev || !dst_bf16_dev) return fail(TSV_ERR_ARGUMENT, "null buffer");
  int e = tsv::launch_normalize(src_dev, src_dtype == TSV_F32, n, dim, normalize, dst_bf16_dev,
                                reinterpret_cast<cudaStream_t>(stream));
  if (e) return cuda_fail(static_cast<cudaError_t>(e), "normalize launch");
  g_launches++;
  return TSV_OK;
}

}  // extern "C"
