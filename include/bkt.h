/*
 * bkt.h -- C ABI of the B200-native bigger-buffer k-d tree k-NN engine
 * (libbkt.so, built from paper_1512_02831_b200/csrc/).
 *
 * Plain pointers and sizes only.  Every entry point replaces one reference
 * interface of the `bufferknn` package's hot path (arXiv 1512.02831 re-
 * implementation at /root/reference/pkg); the Python host layer
 * (paper_1512_02831_b200/) mirrors the reference API on top of it and maps
 * the negative return codes to the reference's exception types.
 *
 * Threading: a context is bound to one CUDA device.  Calls on one context
 * must not overlap; distinct contexts (one per GPU) may be driven from
 * distinct host threads concurrently (reference scheduler.py:211-220).
 */
#ifndef BKT_H
#define BKT_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* return codes */
#define BKT_OK 0
#define BKT_EINVAL (-1)   /* ValueError  (shape / k / height validation)          */
#define BKT_ECONFIG (-2)  /* DeviceConfigError (memory budget, chunk capacity)      */
#define BKT_ECUDA (-3)    /* RuntimeError (CUDA failure; message has the cause)    */
#define BKT_ENOMEM (-4)   /* RuntimeError (host or device allocation failed)       */
#define BKT_ESTATE (-5)   /* RuntimeError (no tree loaded / context misuse)        */

typedef struct bkt_ctx bkt_ctx;

/* Search options.  Mirrors lazy_search's keyword surface
 * (buffer_tree.py:523-526, BufferConfig buffer_tree.py:61-92) plus the
 * B200-specific knobs.  Buffer capacity / fetch count / threshold only
 * schedule work in the reference (results are independent of them,
 * buffer_tree.py:263-284); the device engine schedules every active query
 * each round and accepts them for validation only. */
typedef struct bkt_search_opts {
  int32_t exact;            /* 1: bit-exact reference arithmetic (two roundings per dim); 0: FMA */
  int32_t queries_on_device;/* 1: `queries` is a device pointer (m x d, row-major, this ctx's GPU) */
  int32_t keys_on_device;   /* 1: `out_keys` is a device pointer                                   */
  int32_t record_timing;    /* 1: time leafscan launches with CUDA events (stats->leafscan_ms)     */
  int64_t batch_queries;    /* queries resident per batch (0 = auto from free memory)            */
  int32_t* visited_out;     /* optional (m,) host int32: leaves visited per query                  */
  int32_t* seq_log;         /* optional host int32 triples (query, visit#, leaf), capacity seq_cap */
  int64_t seq_cap;
  int64_t* seq_count_out;   /* number of triples written (may exceed seq_cap: truncated)         */
  int32_t kernel;           /* leaf scan: 0 auto (tensor-core filter when available), 1 CUDA-core
                               direct scan, 2 tensor-core filter (error if unavailable)           */
} bkt_search_opts;

typedef struct bkt_stats {
  int64_t rounds;           /* ProcessAllBuffers rounds (SearchStats.process_rounds)   */
  int64_t leaf_visits;      /* (query, leaf) scans (SearchStats.leaf_scan_events)       */
  int64_t pairs;            /* algorithmic distance pairs = sum over visits of |leaf|  */
  int64_t kernel_launches;  /* engine kernels launched by this call                   */
  int64_t leafscan_launches;
  double leafscan_ms;       /* CUDA-event time of leafscan launches (record_timing)    */
  double search_ms;         /* CUDA-event time of the whole device search             */
  double h2d_ms, d2h_ms;
  int64_t h2d_bytes, d2h_bytes;
  int64_t stream_bytes;     /* host-resident leaf structure: bytes streamed H2D into the chunk slots */
  int64_t stream_copies;    /* chunk copies issued (each a pinned -> device cudaMemcpyAsync pair)   */
} bkt_stats;

/* Context on one CUDA device (replaces device.py:361-364 device_init /
 * SimulatedDevice's buffers, queues and events: device.py:181-358). */
int bkt_open(int cuda_device, bkt_ctx** out);
void bkt_close(bkt_ctx* ctx);
/* Last error message of this context, or of the calling thread when ctx is NULL. */
const char* bkt_last_error(const bkt_ctx* ctx);
int bkt_device_info(bkt_ctx* ctx, int32_t* sm_count, int32_t* sm_clock_khz, int64_t* free_bytes,
                    int64_t* total_bytes);

/* Host build of the top tree + leaf order (replaces build_buffer_tree's
 * median splits, buffer_tree.py:149-197 and kdtree.py:55-70).  Writes
 * split values (2^h - 1, level order), the leaf-sorted order
 * (original_index, n) and leaf_starts (2^h + 1).  Native, multithreaded. */
int bkt_build_tree(const float* refs, int64_t n, int32_t d, int32_t h, float* split_out,
                   int64_t* order_out, int64_t* leaf_starts_out, int32_t nthreads);

/* The same build on a GPU (replaces the same reference code): per level a
 * radix selection of every subset's positional median key and a scan-based
 * partition.  Writes what bkt_build_tree writes plus, when points_out is not
 * NULL, the leaf-sorted (n, d) points.  On failure the message is in
 * bkt_build_tree_device_error(). */
int bkt_build_tree_device(int cuda_device, const float* refs, int64_t n, int32_t d, int32_t h, float* split_out,
                          int64_t* order_out, int64_t* leaf_starts_out, float* points_out);
const char* bkt_build_tree_device_error(void);

/* Upload a built tree (replaces ChunkPipeline's staging of the leaf
 * structure, device.py:380-420).  leaf_points is the leaf-sorted (n, d)
 * float32 matrix, original_index its (n,) row ids, leaf_starts (2^h + 1).
 * residency 0: leaf structure resident in HBM.  residency 1: host-resident
 * in pinned memory, streamed through two device chunk buffers per round
 * (sec. 3.2); chunk_bounds (num_chunks + 1 row offsets, the
 * reference ChunkPlan.bounds, scheduler.py:35-72) define the chunks. */
int bkt_load_tree(bkt_ctx* ctx, int32_t h, int32_t d, int64_t n, const float* split_values,
                  const float* leaf_points, const int64_t* original_index, const int64_t* leaf_starts,
                  int32_t residency, int32_t num_chunks, const int64_t* chunk_bounds);

/* Host-resident structures (residency 1) loaded after this call live in
 * file-backed pages under `dir` (unlinked files mapped MAP_SHARED) instead of
 * page-locked memory, so the structure may exceed host RAM: the drain
 * streams each unit disk -> host -> device (sec. 3.2).  NULL or ""
 * restores page-locked memory.  The general-domain path (k > 64, d > 32,
 * h > 16) needs a page-locked structure and fails with BKT_EINVAL on a
 * spilled one. */
int bkt_set_spill_dir(bkt_ctx* ctx, const char* dir);

/* k-NN search of m queries (replaces lazy_search, buffer_tree.py:523-646).
 * out_keys: (m, k) uint64 ascending packed keys (f32 bits << 32 | index),
 * exactly NeighborBatch.keys (core.py:230-262).  Domain: the reference's --
 * any 1 <= k <= n (core.py:92-102), any d, any height with 2^h <= n up to
 * h = 30 (buffer_tree.py:159-163).  k > 64, d > 32 or h > 16 run on the
 * general-domain path (one CTA per query, wide_search.cuh) with the same
 * results, visit counts and leaf sequences. */
int bkt_search(bkt_ctx* ctx, const float* queries, int64_t m, int32_t k, const bkt_search_opts* opts,
               uint64_t* out_keys, bkt_stats* stats);

/* Brute-force scan of one resident chunk for groups of query rows
 * (replaces SimulatedDevice.enqueue_brute_kernel, device.py:283-337, the
 * reference's device plugin seam).  points (L, d) + ids (L,) are the chunk;
 * group g covers rows group_rows[group_ptr[g] .. group_ptr[g+1]) scanned
 * against chunk rows [group_lo[g], group_hi[g]) (chunk-relative).  keys
 * (m, k) host array is merged in place (NeighborBatch.update_rows). */
int bkt_scan_groups(bkt_ctx* ctx, const float* points, const int64_t* ids, int64_t L, int32_t d,
                    const float* queries, int64_t m, int32_t k, uint64_t* keys, int32_t ngroups,
                    const int64_t* group_ptr, const int64_t* group_rows, const int64_t* group_lo,
                    const int64_t* group_hi, int32_t exact);

/* The same seam with device-resident chunk slots (SimulatedDevice
 * enqueue_copy / enqueue_brute_kernel, device.py:256-337, as driven by
 * ChunkPipeline, device.py:367-457).  bkt_seam_copy uploads a chunk (L
 * points of d coordinates + ids) into slot 0 or 1 on the context's copy
 * stream and returns at once when `points` is page-locked (an event marks
 * the copy's completion; bkt_seam_sync waits for it).  bkt_seam_scan runs the
 * group scan against a resident slot on the compute stream after that copy,
 * moving only the query rows and top-k rows the groups name, one warp per
 * distinct row (all of a row's ranges merged in one pass); keys (m, k) host
 * array is merged in place.  Same arguments and errors as bkt_scan_groups. */
int bkt_seam_copy(bkt_ctx* ctx, int32_t slot, const float* points, const int64_t* ids, int64_t L, int32_t d);
int bkt_seam_sync(bkt_ctx* ctx, int32_t slot);
int bkt_seam_scan(bkt_ctx* ctx, int32_t slot, const float* queries, int64_t m, int32_t k, uint64_t* keys,
                  int32_t ngroups, const int64_t* group_ptr, const int64_t* group_rows, const int64_t* group_lo,
                  const int64_t* group_hi, int32_t exact);

/* FP32 pipe probe: FFMA throughput of this device (TFLOP/s) measured with
 * CUDA events; used as the measured roofline denominator. */
int bkt_fp32_peak(bkt_ctx* ctx, double* tflops);

/* Page-locked host memory for result arrays (cudaHostAlloc, portable): a
 * search whose out_keys lie in it copies results straight from the device
 * instead of through the pinned staging slots.  NULL on failure. */
void* bkt_host_alloc(int64_t bytes);
void bkt_host_free(void* p);

#ifdef __cplusplus
}
#endif
#endif /* BKT_H */
