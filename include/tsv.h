/*
 * tsv.h - C ABI of the B200 retrieval backend (Teola vector-search / rerank primitives).
 *
 * This is the drop-in boundary behind Teola's primitive executor. In the reference the
 * Searching and Reranking primitives are executed by `Simulator._execute`
 * (reference: pkg/src/teola_sim/runtime.py:625-656), which only looks up a latency from
 * the engine profile (pkg/src/teola_sim/engines.py:105-109). Each entry point below names
 * the reference interface it replaces. All compute entry points are asynchronous on the
 * caller's CUDA stream, take caller-owned device buffers as plain pointers, and return a
 * status code (0 = OK). Handles are thread-compatible, not thread-safe; scratch space is
 * kept per (index, stream) so concurrent streams on one index do not collide.
 *
 * Ordering convention of every result list: (score desc, id asc). Lists shorter than k are
 * padded with (score = -inf, id = -1).
 */
#ifndef TSV_H_
#define TSV_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TSV_ABI_VERSION 1

#if defined(__GNUC__)
#define TSV_API __attribute__((visibility("default")))
#else
#define TSV_API
#endif

/* Status codes. Nonzero values map onto the reference's TeolaError hierarchy
 * (pkg/src/teola_sim/errors.py:7-67) in the Python host layer:
 *   TSV_ERR_CAPACITY -> CapacityExceeded (empty / oversize batch, errors.py:34-35)
 *   TSV_ERR_CONFIG   -> ConfigParse      (bad dim / dtype / metric, errors.py:54-55)
 *   TSV_ERR_DEVICE   -> DeviceError      (CUDA failure; new subclass)
 *   TSV_ERR_ARGUMENT -> ConfigParse      (null / misaligned pointers)                     */
enum {
  TSV_OK = 0,
  TSV_ERR_CAPACITY = 1,
  TSV_ERR_CONFIG = 2,
  TSV_ERR_DEVICE = 3,
  TSV_ERR_ARGUMENT = 4
};

enum { TSV_BF16 = 0, TSV_F32 = 1 };               /* element types */
/* arena storage: TSV_BF16 (row-major), TSV_F32 (fp32 mode), TSV_BF16_TILED (row-major within
 * contiguous 16 KB [128 rows x 64 elements] k-block tiles: the scan streams whole tiles; row
 * ranges passed to the search calls must start at multiples of 128) */
enum { TSV_BF16_TILED = 2 };
enum { TSV_METRIC_IP = 0, TSV_METRIC_COSINE = 1 }; /* cosine = IP over L2-normalised rows */

typedef struct tsv_index tsv_index;

TSV_API int tsv_abi_version(void);
/* Message of the last failing call on this thread ("" if none). */
TSV_API const char* tsv_last_error(void);
/* Kernel launches issued by this library since load (for launch accounting). */
TSV_API int64_t tsv_launch_count(void);

/* ---- corpus arena (Ingestion side; reference: optimizer.py:125-156 Ingestion node,
 *      executed through runtime.py:653-655 from profiles/default.json:27-46 vdb-ingest0) ---- */

/* Device-resident bf16 arena of up to cap_rows rows of `dim` elements (dim % 8 == 0). */
TSV_API int tsv_index_create(int device, int dim, int metric, int64_t cap_rows, tsv_index** out);
/* storage = TSV_BF16 (default arena, 2 B/element) or TSV_F32 (fp32 mode: each row is kept as a
 * tf32 "hi" plane plus an fp32 residual "lo" plane, 8 B/element; search runs 3xTF32 on the
 * tensor cores, scores within 1e-5 relative; k <= 64). */
TSV_API int tsv_index_create2(int device, int dim, int metric, int storage, int64_t cap_rows,
                              tsv_index** out);
/* Wrap an existing device matrix [n_rows, dim] bf16 (already normalised for cosine) without
 * copying; the caller keeps it alive. Appends are rejected on a view. */
TSV_API int tsv_index_create_view(int device, int dim, int metric, const void* rows_dev, int64_t n_rows,
                          tsv_index** out);
TSV_API int tsv_index_destroy(tsv_index* idx);
/* Append n rows (bf16 or f32, normalised when metric is cosine); *first_row receives the arena
 * row of the first appended row. Returns TSV_ERR_CAPACITY when the arena would overflow. */
TSV_API int tsv_index_append(tsv_index* idx, const void* rows_dev, int src_dtype, int64_t n,
                     int64_t* first_row, void* stream);
/* Claim n rows at the end of the arena without writing them (their content is undefined until
 * the caller writes them, e.g. through tsv_index_data: the ingest stages of a per-query index
 * fill their slices of one reserved segment); *first_row receives the first claimed row. */
TSV_API int tsv_index_reserve(tsv_index* idx, int64_t n, int64_t* first_row);
/* Drop rows >= n (n <= current row count). */
TSV_API int tsv_index_truncate(tsv_index* idx, int64_t n);
TSV_API int64_t tsv_index_rows(const tsv_index* idx);
TSV_API int tsv_index_dim(const tsv_index* idx);
TSV_API int tsv_index_metric(const tsv_index* idx);
TSV_API const void* tsv_index_data(const tsv_index* idx);     /* bf16 rows, or the fp32 hi plane */
TSV_API const void* tsv_index_data_lo(const tsv_index* idx);  /* fp32 residual plane (TSV_F32) */
TSV_API int tsv_index_storage(const tsv_index* idx);

/* Accumulated device time of the fused scan kernel (K1) launches issued while timing is on.
 * Reading synchronises on the recorded events. */
TSV_API int tsv_index_set_timing(tsv_index* idx, int enable);
TSV_API int tsv_index_scan_time(tsv_index* idx, double* total_ms, int64_t* launches);

/* ---- K1: Searching primitive over one contiguous row range (global corpus / shard).
 * Replaces the PHASE_GENERAL latency lookup of runtime.py:653-655 for engine category
 * "search" (engines.py:21, graph.py:47-59). q_dev: [B, dim] (bf16 or f32). Emitted id =
 * arena row + id_offset. Outputs scores/ids [B, k]. k <= 128. k <= 32 keeps the top-k lists in
 * registers (CTA-pair kernel for B > 128; 256-row corpus tiles for 96 < B <= 128 on long
 * scans). Larger k (B <= 32768): scans of <= 8192 rows append every row as a candidate and
 * select exactly; longer scans run a sample pass (1/32 of every range; 1/16 for k > 100) for a
 * per-query floor, then a candidate pass appending every row above the floor plus an exact
 * select, with a device-gated shared-memory-list pass if a candidate row overflows. Exact in
 * all cases. ---- */
TSV_API int tsv_search(tsv_index* idx, const void* q_dev, int q_dtype, int B, int k, int64_t row_beg,
               int64_t row_end, int32_t id_offset, float* scores_dev, int32_t* ids_dev,
               void* stream);

/* ---- K2: segmented Searching: queries [seg_q_beg[s], seg_q_beg[s+1]) search only arena rows
 * [seg_row_beg[s], seg_row_end[s]) (per-query indexes built by each query's own Ingestion;
 * workloads.py:95-97). Segment arrays are host memory. local_ids != 0 emits ids relative to
 * the segment's first row. ---- */
TSV_API int tsv_search_segmented(tsv_index* idx, const void* q_dev, int q_dtype, int nseg,
                         const int32_t* seg_q_beg, const int64_t* seg_row_beg,
                         const int64_t* seg_row_end, int k, int local_ids, float* scores_dev,
                         int32_t* ids_dev, void* stream);

/* ---- K3: Reranking primitive (optimizer.py:199-218): for each of B questions score the C
 * candidate arena rows cand_ids_dev[b, :] (id < 0 ignored), drop duplicate ids, keep k. ---- */
TSV_API int tsv_rerank(tsv_index* idx, const void* q_dev, int q_dtype, int B, const int32_t* cand_ids_dev,
               int C, int k, float* scores_dev, int32_t* ids_dev, void* stream);
/* K3 over per-query indexes: question b's candidate ids are rows of its own index segment,
 * i.e. arena row = row_offsets_dev[b] + id (device int32 [B]); the returned ids stay
 * segment-local, as the Searching stages that produced the candidates emitted them. A batch of
 * Reranking requests from different queries is one launch. */
TSV_API int tsv_rerank_segmented(tsv_index* idx, const void* q_dev, int q_dtype, int B,
                                 const int32_t* cand_ids_dev, int C, const int32_t* row_offsets_dev,
                                 int k, float* scores_dev, int32_t* ids_dev, void* stream);
/* The same with the row offsets in host memory (int32 [B]): uploaded on the stream through the
 * library's pinned slots (no device table for the caller to build per batch). */
TSV_API int tsv_rerank_segmented_host(tsv_index* idx, const void* q_dev, int q_dtype, int B,
                                      const int32_t* cand_ids_dev, int C,
                                      const int32_t* row_offsets_host, int k, float* scores_dev,
                                      int32_t* ids_dev, void* stream);

/* ---- K3s: contextual retrieval's Searching -> Reranking chain in ONE launch (BASELINE C5;
 * reference workloads.py:247-257 builds a per-query index, searches it, reranks the hits; the
 * stage pair is optimizer.py:178-218). Query b searches ITS OWN index segment, arena rows
 * [q_rows_dev[2b], q_rows_dev[2b+1]) (device int64 [B][2]; at most max_rows <= 1024 rows each,
 * longer segments are cut at max_rows), keeps the top k_search (written to search_*, [B, k_search],
 * ids segment-local when local_ids, else arena rows), and reranks those rows against
 * q_rerank_dev[b] (NULL: the query itself), keeping the top k_rerank <= k_search (rerank_*).
 * Cosine indexes normalise both vectors in the kernel. bf16 / tiled arenas, dim <= 2048.
 * Equivalent to tsv_search_segmented + tsv_rerank(_segmented): the rerank scores are
 * bit-identical to tsv_rerank's for the same rows; the search scores differ from the tensor-core
 * scan's by summation order only. No workspace, no host round trip: capture-safe. ---- */
TSV_API int tsv_search_rerank_segmented(tsv_index* idx, const void* q_search_dev,
                                        const void* q_rerank_dev, int q_dtype, int B,
                                        const int64_t* q_rows_dev, int max_rows, int k_search,
                                        int k_rerank, int local_ids, float* search_scores_dev,
                                        int32_t* search_ids_dev, float* rerank_scores_dev,
                                        int32_t* rerank_ids_dev, void* stream);

/* The same chain with the per-query row ranges as a HOST array (int64 [B][2]), uploaded
 * through the library's pinned staging slots on `stream` (stream-ordered, no pageable copy;
 * under CUDA-graph capture the table is baked into the graph): the executor's per-batch call,
 * which has the segment table on the host (reference runtime.py:625-656 builds the batch there). */
TSV_API int tsv_search_rerank_segmented_host(tsv_index* idx, const void* q_search_dev,
                                             const void* q_rerank_dev, int q_dtype, int B,
                                             const int64_t* q_rows_host, int max_rows,
                                             int k_search, int k_rerank, int local_ids,
                                             float* search_scores_dev, int32_t* search_ids_dev,
                                             float* rerank_scores_dev, int32_t* rerank_ids_dev,
                                             void* stream);

/* ---- K4: merge `lists` sorted lists per query. Input layout [lists][B][kin]; output [B][kout].
 * This is the Aggregate join of split Searching stages (optimizer.py:620-661,
 * runtime.py:544-549) and the cross-shard merge after the all-gather. dedup != 0 keeps one
 * entry per id (partial rerank lists of one question over overlapping candidates). ---- */
TSV_API int tsv_merge_topk(const float* in_scores, const int32_t* in_ids, int lists, int B, int kin,
                   int kout, int dedup, float* out_scores, int32_t* out_ids, void* stream);

/* ---- Sharded mode over NVLink: all-gather of the per-rank [B, k] lists fused with the
 * cross-shard merge (replaces ncclAllGather + tsv_merge_topk). One process per GPU; each
 * rank creates a symmetric buffer, exports its IPC handle, opens every peer's handle (handles
 * travel over any side channel, e.g. torch.distributed), then calls allgather_merge with the
 * same call sequence on every rank (B <= max_b and k <= max_k may vary from call to call). Ranks
 * push their lists into peers' memory, stamp each (source, query) slot with the call's epoch
 * and merge on arrival. ---- */
typedef struct tsv_peer_group tsv_peer_group;
TSV_API int tsv_peer_create(int device, int world, int rank, int max_b, int max_k,
                            tsv_peer_group** out);
TSV_API int tsv_peer_handle(tsv_peer_group* g, void* handle_out /* 64 bytes */, int* handle_bytes);
TSV_API int tsv_peer_open(tsv_peer_group* g, int peer, const void* handle);
/* In-process peer: map rank `peer`'s buffer from its group `other` (created in this process,
 * same world / max_b / max_k) without IPC — ranks driven by one process on one device or on
 * peer-accessible devices (enables peer access). Lets one process measure and test the
 * exchange with every rank's kernel in flight at once. */
TSV_API int tsv_peer_attach(tsv_peer_group* g, int peer, tsv_peer_group* other);
TSV_API int tsv_peer_allgather_merge(tsv_peer_group* g, const float* local_scores,
                                     const int32_t* local_ids, int B, int k, float* out_scores,
                                     int32_t* out_ids, void* stream);
/* A wait longer than the timeout (default 60 s; TSV_PEER_TIMEOUT_MS) aborts: every rank's
 * kernel ends with padded outputs, the group is marked dead and the next call (or
 * tsv_peer_status after a stream sync) returns TSV_ERR_DEVICE. */
TSV_API int tsv_peer_set_timeout_ms(tsv_peer_group* g, int64_t ms);
/* *aborted = 1 (and TSV_ERR_DEVICE) once an exchange of this group gave up waiting. Reads a
 * host-mapped word; synchronise the stream of the last call first. */
TSV_API int tsv_peer_status(tsv_peer_group* g, int* aborted);
TSV_API int tsv_peer_destroy(tsv_peer_group* g);

/* ---- Corpus-sharded search inside one process (several devices, or one device twice):
 * shard g is an index on its own device holding global rows [id_offsets[g], ...). A search
 * copies the queries (on device `root`, caller's stream) to every shard's device, runs K1 on
 * each shard on the shard's own stream with global ids, writes the per-shard [B, k] lists
 * straight into a gather buffer on the root over NVLink (peer access; staged copies where
 * peers cannot map each other) and merges them there (K4) on the caller's stream. Buffers are
 * sized at create time for B <= max_b, k <= max_k: the call allocates nothing.
 * Replaces the reference executor's single "search" engine call (runtime.py:625-656 ->
 * engines.py:105-109) for a corpus too large for one GPU; SURVEY.md §8(b) `tsv_sharded_search`.
 * The shard indexes must outlive the handle. ---- */
typedef struct tsv_sharded tsv_sharded;
TSV_API int tsv_sharded_create(tsv_index* const* shards, const int64_t* id_offsets, int nshards,
                               int root, int max_b, int max_k, tsv_sharded** out);
TSV_API int tsv_sharded_search(tsv_sharded* sh, const void* q_dev, int q_dtype, int B, int k,
                               float* scores_dev, int32_t* ids_dev, void* stream);
TSV_API int tsv_sharded_destroy(tsv_sharded* sh);

/* ---- A private (non-blocking) stream of the caller's own, outside any framework's stream
 * pool: scratch space is kept per (index, stream), so a stream that captures a CUDA graph of
 * searches must never be handed to another caller (the graph keeps the scratch addresses;
 * once a stream captured, its scratch is pinned and a call needing more fails with
 * TSV_ERR_CAPACITY instead of moving it). ---- */
TSV_API int tsv_stream_create(int device, void** out);
TSV_API int tsv_stream_destroy(void* stream);

/* ---- K5: L2-normalise (normalize != 0) and cast rows to bf16. ---- */
TSV_API int tsv_normalize_rows(const void* src_dev, int src_dtype, int64_t n, int dim, int normalize,
                       void* dst_bf16_dev, void* stream);

/* ---- Host scheduler: the engine queue of the topology-aware batch scheduler in native
 * memory (replaces the per-call rebuild in form_batch_topo, pkg/src/teola_sim/runtime.py:189-268,
 * and the dispatch-time queue filter, runtime.py:603-606). Host-only: no CUDA calls, no GPU
 * needed. A task is pushed once with its static fields (query id, node id, graph depth, phase
 * code, arrival time) and its request loads; tsv_topo_form forms one batch with the
 * reference's decisions (per-query buckets in order of earliest arrival, deepest nodes first
 * in node-id order, passes until the cap is reached) and writes (task handle, request count)
 * pairs; tsv_topo_commit consumes a dispatched batch's requests and drops drained tasks.
 * tsv_topo_form returns TSV_ERR_CAPACITY with *n_entries set when cap_entries is too small. */
typedef struct tsv_topo_queue tsv_topo_queue;
TSV_API int tsv_topo_create(double eps, tsv_topo_queue** out);
TSV_API int tsv_topo_destroy(tsv_topo_queue* q);
TSV_API int64_t tsv_topo_size(const tsv_topo_queue* q);
TSV_API int tsv_topo_push(tsv_topo_queue* q, int64_t handle, const char* query_id,
                          const char* node_id, int depth, int phase, double arrival_ms,
                          const double* loads, int64_t n_loads, int64_t next);
TSV_API int tsv_topo_form(tsv_topo_queue* q, double max_slots, int64_t cap_entries,
                          int64_t* handles, int64_t* counts, int64_t* n_entries, double* load,
                          int* phase);
TSV_API int tsv_topo_commit(tsv_topo_queue* q, const int64_t* handles, const int64_t* counts,
                            int64_t n);

#ifdef __cplusplus
}
#endif

#endif /* TSV_H_ */
