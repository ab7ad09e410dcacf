/*
 * rbe_cuda.h -- C ABI of the B200 exhaustive RBE retrieval path.
 *
 * This is the drop-in boundary: plain C types, caller-owned buffers, integer
 * status codes.  Everything above it (the C++ rbe:: API in include/rbe/*.hpp
 * and the Python module paper_1802_06466_b200._core) calls only these entry
 * points; everything below it is hand-written sm_100a CUDA.
 *
 * Reference interfaces replaced (paths relative to the reference's proj/):
 *   rbe_cuda_index_*          KeywordIndex / Partition held in host RAM
 *                             (include/rbe/index.hpp:16-34) -> an HBM-resident,
 *                             bit-plane-major device store.
 *   rbe_cuda_search           rbe::search (include/rbe/search.hpp:68-70,
 *                             src/search.cpp:130-168) incl. local_select
 *                             (search.cpp:57-113), global_select
 *                             (search.cpp:115-128) and the partition merge
 *                             (search.cpp:160-167), batched over Q queries.
 *   rbe_cuda_search_device    same, outputs left in device memory for the
 *                             multi-GPU gather (replaces the std::async
 *                             partition fan-out, search.cpp:148-157).
 *   rbe_cuda_merge_device     the final merge under entry_less
 *                             (search.cpp:50-53, 160-167) over gathered lists.
 *
 *   rbe_cuda_local_select     local_select (search.hpp:53-57, search.cpp:57-113):
 *                             per-logical-thread candidate lists of one partition.
 *   rbe_cuda_select_topn      global_select's sort + truncate (search.cpp:115-128).
 *
 * Streams and lifetime: every call may be issued on any stream; an index orders
 * its batches across streams itself (the next batch waits for the previous one),
 * and all scratch is owned by the index (or, for merge/select, by a per-device
 * context) and reused across calls -- no per-call device allocation in steady
 * state.  The tensor kernel's internal-consistency flag is sticky per index: a
 * batch enqueued asynchronously (search_device without stats) that trips it is
 * reported by the next synchronous call on that index (rbe_cuda_search,
 * search_device with stats, last_batch_ms, rbe_cuda_index_check, search_multi).
 *
 * Error model (mirrors the reference's exceptions):
 *   RBE_CUDA_EINVAL   -> std::invalid_argument / ValueError
 *   RBE_CUDA_ERANGE   -> std::out_of_range     / IndexError
 *   RBE_CUDA_ERUNTIME -> std::runtime_error    / RuntimeError (CUDA, I/O)
 * rbe_cuda_last_error() returns the thread-local message of the last failure.
 * There is no CPU fallback: without a usable CUDA device every compute entry
 * point fails with RBE_CUDA_ERUNTIME.
 */
#ifndef RBE_CUDA_H
#define RBE_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RBE_CUDA_OK 0
#define RBE_CUDA_EINVAL 1
#define RBE_CUDA_ERANGE 2
#define RBE_CUDA_ERUNTIME 3

/* Scan kernel variants.  AUTO = TENSOR when the shape is supported by the
 * tensor-core kernel, else EXACT.  Both are GPU kernels
 * with identical results; the variant that ran is reported in
 * rbe_search_stats.variant. */
#define RBE_VARIANT_AUTO 0
#define RBE_VARIANT_EXACT 1  /* CUDA-core XOR+popc, FP64 score per pair      */
#define RBE_VARIANT_TENSOR 2 /* int8 tensor-core scan + threshold filter     */

typedef struct rbe_cuda_index rbe_cuda_index;

/* rbe::ScanGeometry, include/rbe/search.hpp:12-21. */
typedef struct {
    uint32_t blocks;
    uint32_t threads_per_block;
    uint32_t items_per_thread;
    uint32_t queue_length;
} rbe_scan_geometry;

/* KeywordIndex header fields, include/rbe/index.hpp:23-27. */
typedef struct {
    uint32_t dim;
    uint32_t keyword_planes;
    uint32_t residual_weights;
} rbe_index_shape;

typedef struct {
    uint32_t variant;      /* RBE_VARIANT_*                                       */
    uint32_t probe_tiles;  /* TENSOR: tiles per logical block sampled for the
                              threshold probe (0 = default)                       */
    uint32_t reserved[6];
} rbe_search_options;

typedef struct {
    uint64_t scored;        /* SearchStats::scored (search.hpp:45-47): Q * keywords */
    uint32_t variant;       /* kernel that ran                                    */
    uint32_t fallback;      /* 1 if TENSOR overflowed its candidate buffer and the
                               batch was re-run with EXACT                        */
    uint64_t candidates;    /* TENSOR: pairs that passed the threshold filter     */
    uint64_t survivors;     /* per-logical-thread survivors fed to selection      */
    double scan_ms;         /* device time of the scan kernel(s)                  */
    double total_ms;        /* device time of the whole batch                     */
    uint32_t launches;      /* kernels launched for the batch                     */
    uint32_t reserved[3];
} rbe_search_stats;

/* Create an empty device index on CUDA device `device` holding
 * `n_partitions` partitions whose global ordinals (the `partition` field of
 * results, search.hpp:34-38) are `ordinals[i]` and sizes `counts[i]`.
 * Device memory for all partitions is reserved here. */
int rbe_cuda_index_create(const rbe_index_shape* shape, uint32_t n_partitions, const uint32_t* ordinals,
                          const uint64_t* counts, int device, rbe_cuda_index** out);

/* Upload local partition `i` from the reference's host layout
 * (Partition, index.hpp:16-21): planes = plane_blocks concatenated in plane
 * order, [keyword_planes][count * words_per_plane] u64; mags f32[count];
 * ids u64[count].  Magnitudes must be finite and > 0 (EINVAL otherwise; the
 * reference's load_index does not validate). */
int rbe_cuda_index_upload_partition(rbe_cuda_index* index, uint32_t i, const uint64_t* planes,
                                    const float* mags, const uint64_t* ids);
/* (Streamed in chunks through page-locked staging buffers filled by several host
 * threads; each chunk is re-packed into the store layout on the device.) */

/* RBEI v1 ingest.  Replaces the reference's load_index
 * (src/index.cpp:170-208) followed by an upload: the file is read once, straight
 * into HBM.  Same errors as load_index (ERUNTIME): "cannot open index: <path>",
 * "not an RBEI index file: <path>", "unsupported index version", "truncated index
 * file: <path>". */
typedef struct {
    uint64_t file_bytes_read; /* partition bytes read from the file            */
    double seconds;           /* wall time of the call                         */
} rbe_load_stats;

/* Header only: shape, partition count and (up to counts_cap) partition sizes.
 * Host-only (no GPU needed). */
int rbe_cuda_rbei_header(const char* path, rbe_index_shape* shape, uint32_t* n_partitions,
                         uint64_t* counts, uint32_t counts_cap);

/* A handle on `device` holding the file's partitions `partitions[0..n)` (n = 0:
 * all of them, in order) as its local partitions 0..n-1 with their file ordinals.
 * The partition blocks are read with pread by `io_threads` host threads (0 =
 * min(16, hardware threads)) into two alternating page-locked staging buffers
 * (64 MB chunks of documents), copied to the device and re-packed there.
 * Magnitudes must be finite and > 0 (EINVAL). `stats` may be NULL. */
int rbe_cuda_index_open_rbei(const char* path, const uint32_t* partitions, uint32_t n_partitions,
                             int device, uint32_t io_threads, rbe_cuda_index** out,
                             rbe_load_stats* stats);

/* RBEE v1 bulk embeddings -> index build on the device.  Replaces
 * the reference's EmbeddingReader + IndexBuilder loop of `rbe build`
 * (src/embedding_io.cpp:48-95, src/index.cpp:36-78, tools/rbe_main.cpp:109-123):
 * record k goes to partition k % n_partitions_total, slot k / n_partitions_total;
 * a record magnitude that is not > 0 is recomputed on the device exactly as
 * make_embedding does.  Errors as the reference (header: ERUNTIME "cannot open
 * embeddings file", "not an RBEE embeddings file", "unsupported embeddings version",
 * "embeddings file has empty shape", "embeddings file has truncated records"; EINVAL
 * "IndexBuilder: need at least one partition", "IndexBuilder: keyword has zero
 * magnitude", "IndexBuilder: duplicate keyword id" among this handle's keywords;
 * non-finite magnitudes are rejected as well).  The handle holds partitions
 * `partitions[0..n)` (n = 0: all).  Host-only header reader: rbe_cuda_rbee_header. */
int rbe_cuda_rbee_header(const char* path, rbe_index_shape* shape, uint64_t* count);
int rbe_cuda_index_build_rbee(const char* path, uint32_t n_partitions_total, const uint32_t* partitions,
                              uint32_t n_partitions, int device, uint32_t io_threads,
                              rbe_cuda_index** out, rbe_load_stats* stats);
/* Every id of the handle's partitions, ascending, into ids[total] (duplicate checks
 * across handles). */
int rbe_cuda_index_sorted_ids(const rbe_cuda_index* index, uint64_t* ids);

/* Fill every local partition on the device with the synthetic corpus of
 * global doc g of n_total, bits from counter-based
 * splitmix64(seed) in plane-major stream order, partition g % n_partitions_total,
 * slot g / n_partitions_total, id g, magnitude float(sqrt(sum refined^2)). */
int rbe_cuda_index_fill_synthetic(rbe_cuda_index* index, uint64_t seed, uint64_t n_total,
                                  uint32_t n_partitions_total);

/* Copy local partition `i` back in the reference's host layout (test path). */
int rbe_cuda_index_download_partition(const rbe_cuda_index* index, uint32_t i, uint64_t* planes,
                                      float* mags, uint64_t* ids);

int rbe_cuda_index_destroy(rbe_cuda_index* index);

/* Bytes of device memory held by the index, and the algorithmic bytes one
 * scan reads per batch (plane words + f32 magnitudes). */
int rbe_cuda_index_bytes(const rbe_cuda_index* index, uint64_t* device_bytes, uint64_t* scan_bytes);

/* Batched rbe::search.  query_words: [n_queries][query_planes][words_per_plane]
 * u64 in the reference's PackedBinaryVector layout (binary_vector.hpp:14-21).
 * Outputs (caller-owned host buffers, n entries per query):
 *   scores[q*n + k], ids[q*n + k], partitions[q*n + k], accs[q*n + k]
 *   (accs = exact integer accumulator, score = ldexp(acc, -L) / mag)
 *   counts[q] = number of valid entries for query q (<= n).
 * Entries are ordered by (score desc, id asc) (search.cpp:50-53).  Any of
 * accs / stats may be NULL.  Blocking; one batch in flight per index. */
int rbe_cuda_search(rbe_cuda_index* index, const uint64_t* query_words, uint32_t n_queries,
                    uint32_t query_planes, const rbe_scan_geometry* geometry, uint64_t n,
                    const rbe_search_options* options, double* scores, uint64_t* ids,
                    uint32_t* partitions, int64_t* accs, uint64_t* counts, rbe_search_stats* stats);

/* Result record in device memory (32 bytes). */
typedef struct {
    double score;
    uint64_t id;
    int64_t acc;
    uint32_t partition;
    uint32_t valid;
} rbe_result;

/* Same search with the query batch and outputs in DEVICE memory on the
 * index's device: out = rbe_result[n_queries][n] (invalid tail entries have
 * valid = 0).  `stream` is a cudaStream_t (NULL = the index's own stream).
 * With `stats` non-NULL the call returns after the batch completes on that
 * stream; with `stats` NULL (and the tensor variant) it only enqueues the
 * batch on the stream (no host synchronisation), so back-to-back batches keep
 * the GPU busy. */
int rbe_cuda_search_device(rbe_cuda_index* index, const uint64_t* d_query_words, uint32_t n_queries,
                           uint32_t query_planes, const rbe_scan_geometry* geometry, uint64_t n,
                           const rbe_search_options* options, rbe_result* d_out, void* stream,
                           rbe_search_stats* stats);

/* Device times (ms) of the index's last batch: the scan kernels and the whole
 * batch (CUDA events on the batch's stream); waits for that batch. */
int rbe_cuda_index_last_batch_ms(rbe_cuda_index* index, double* scan_ms, double* total_ms);

/* Page-locked host buffers (cudaMallocHost).  rbe_cuda_search detects output buffers in
 * page-locked memory and copies the results straight into them (DMA, no host-side
 * staging); pageable buffers work too, through a staging copy. */
int rbe_cuda_host_alloc(size_t bytes, void** out);
int rbe_cuda_host_free(void* ptr);

/* Merge `n_lists` result lists per query (d_in = rbe_result[n_lists][n_queries][n],
 * device memory on `device`) into the top n per query under (score desc,
 * id asc): d_out = rbe_result[n_queries][n].  Asynchronous: enqueued on `stream`
 * (NULL = a per-device stream) with persistent per-device scratch. */
int rbe_cuda_merge_device(int device, const rbe_result* d_in, uint32_t n_lists, uint32_t n_queries,
                          uint64_t n, rbe_result* d_out, void* stream);

/* local_select (search.hpp:53-57) of local partition `i` for one query
 * (query_words = [query_planes][words_per_plane] u64): for every logical thread
 * t = block * threads_per_block + thread, its best min(queue_length,
 * items_per_thread) candidates under (score desc, slot asc) in
 * scores/slots[t * ql .. t * ql + counts[t]) (ql = min(queue_length,
 * items_per_thread); buffers hold blocks * threads_per_block * ql entries and
 * counts blocks * threads_per_block).  *scored += keywords scored. */
int rbe_cuda_local_select(rbe_cuda_index* index, uint32_t i, const uint64_t* query_words, uint32_t query_planes,
                          const rbe_scan_geometry* geometry, double* scores, uint64_t* slots, uint32_t* counts,
                          uint64_t* scored);

/* global_select's selection (search.cpp:115-128) on device `device`: the top n of
 * `count` (score, id) candidates under (score desc, id asc); host buffers in and
 * out, *out_count = min(n, count). */
int rbe_cuda_select_topn(int device, const double* scores, const uint64_t* ids, uint64_t count, uint32_t partition,
                         uint64_t n, double* out_scores, uint64_t* out_ids, uint64_t* out_count);

/* Waits for the index's last batch and reports its sticky internal-consistency
 * flag (RBE_CUDA_ERUNTIME if any batch since the last report tripped it). */
int rbe_cuda_index_check(rbe_cuda_index* index);

/* Test hook: sets the index's sticky internal-consistency flag, as a failed
 * accumulator recovery in the tensor kernel would. */
int rbe_cuda_index_inject_error(rbe_cuda_index* index);

/* Single-process multi-GPU rbe::search: every handle (one per device) scans its
 * partitions into a device-resident top n -- all devices concurrently, each on
 * its own stream -- then the lists are copied peer-to-peer to the first
 * non-empty handle's device and merged there; host outputs as in
 * rbe_cuda_search.  Handles without documents take no part; only an index
 * whose handles are all empty is rejected (search.cpp:133-135).
 * stats->scored sums over handles. */
int rbe_cuda_search_multi(rbe_cuda_index* const* handles, uint32_t n_handles, const uint64_t* query_words,
                          uint32_t n_queries, uint32_t query_planes, const rbe_scan_geometry* geometry, uint64_t n,
                          const rbe_search_options* options, double* scores, uint64_t* ids, uint32_t* partitions,
                          int64_t* accs, uint64_t* counts, rbe_search_stats* stats);

const char* rbe_cuda_last_error(void);

/* Library/ABI version and the compiled device architecture, for loaders. */
const char* rbe_cuda_version(void);

#ifdef __cplusplus
}
#endif

#endif /* RBE_CUDA_H */
