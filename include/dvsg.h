/*
 * dvsg.h -- C-ABI of the B200-native batched graph search (libdvsg.so).
 *
 * This is the drop-in boundary for the reference's hot path.  The reference
 * exposes the path as C++ free functions (paths relative to
 * /root/reference/proj):
 *
 *   beam_search_stats / beam_search / visited_count   include/dvs/graph_index.hpp:58-65
 *   combine_results                                   include/dvs/simulator.hpp:66-67
 *   run_pipeline (functional part)                    include/dvs/simulator.hpp:98-102
 *   assign_top_c / partition_database                 include/dvs/kmeans.hpp:41-46
 *   place_clusters / route                            include/dvs/router.hpp:53-57
 *   compute_entry_order / build_graph                 include/dvs/graph_index.hpp:40-45
 *   load_index / save_index (FNSY v1)                 include/dvs/index_file.hpp:13-14
 *
 * Every entry point below replaces one of those (cited per function), with
 * plain pointers and sizes, caller-owned buffers, and no C++/torch types.
 * INTEGRATION.md shows the C++ shim a maintainer binds in their place.
 *
 * Errors: status codes mirror the reference CLI's exit-code map
 * (src/commands.cpp:355-361): DVSG_EINVAL <-> std::invalid_argument /
 * config_error (2), DVSG_EFORMAT <-> format_error (3), DVSG_EINTERNAL <->
 * internal_error and every CUDA error (4).  dvsg_last_error() returns the
 * message of the last failing call on the calling thread.
 *
 * Threading: one host thread per context.  A context owns one CUDA device,
 * its device-resident index and two streams (compute, comm).
 */
#ifndef DVSG_H
#define DVSG_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef int dvsg_status;
#define DVSG_OK 0
#define DVSG_EINVAL 2
#define DVSG_EFORMAT 3
#define DVSG_EINTERNAL 4

#define DVSG_METRIC_L2 0 /* squared_l2, distance.cpp:19-27 */
#define DVSG_METRIC_IP 1 /* -dot (distance.cpp:35-42); extension, parity unpinned */

#define DVSG_ACCUM_F64 0 /* fp64 lane partials + fp64 tree, rounded once to f32 (parity mode; L2:
                          a distance near an f32 rounding boundary is redone in distance.cpp's
                          sequential order, so every key equals squared_l2's) */
#define DVSG_ACCUM_F32 1 /* fp32 lane partials + fp32 tree (fast mode); exact on integer-valued
                          data, upgraded to F64 (L2) / F32C (IP) on anything else (dvsg_index_integral) */
#define DVSG_ACCUM_F32C 2 /* compensated fp32 (TwoSum / FMA TwoProd pairs): ~48-bit sums */

typedef struct dvsg_ctx dvsg_ctx;

/* SearchParams, include/dvs/graph_index.hpp:27-32, plus the metric and
 * accumulation mode of the B200 kernel. */
typedef struct {
  int iterations;  /* I */
  int beam_width;  /* w */
  int k;
  int entry_count; /* entry nodes; the reference CLI defaults it to w (config.cpp:226) */
  int metric;      /* DVSG_METRIC_* */
  int accum;       /* DVSG_ACCUM_* */
} dvsg_search_params;

const char *dvsg_last_error(void);
const char *dvsg_version(void);

/* ---- context ------------------------------------------------------------ */
dvsg_status dvsg_create(int device, dvsg_ctx **out);
dvsg_status dvsg_destroy(dvsg_ctx *ctx);
/* the compute stream (cudaStream_t) so callers can time on it */
void *dvsg_stream(dvsg_ctx *ctx);
dvsg_status dvsg_synchronize(dvsg_ctx *ctx);

/* ---- index load / partition  (load_index index_file.cpp:149-296,
 *      BuiltIndex index.hpp:14-23, GraphIndex graph_index.hpp:13-25) ------- */

/* Drops every partition and the centroids held by the context. */
dvsg_status dvsg_index_reset(dvsg_ctx *ctx);
/* Sets the routing table: centroids (clusters x dim) and placement
 * (cluster_to_rank, router.cpp:28-43) for `ranks` ranks. */
dvsg_status dvsg_set_centroids(dvsg_ctx *ctx, const float *centroids, int clusters, int dim,
                               const uint32_t *cluster_to_rank, int ranks);
/* Uploads one partition (a GraphIndex).  Host arrays are copied; the caller
 * keeps ownership.  entry_order may be NULL, in which case it is computed
 * exactly as compute_entry_order (graph_index.cpp:21-44).  adjacency rows hold
 * local ids (n x out_degree); global_ids may be NULL (iota). */
dvsg_status dvsg_load_partition(dvsg_ctx *ctx, uint32_t cluster, uint64_t n, int dim,
                                int out_degree, const float *vectors,
                                const uint32_t *adjacency, const uint32_t *global_ids,
                                const uint32_t *entry_order);
/* FNSY v1 (index_file.cpp:16-25, :149-296): loads the routing table and the
 * partitions owned by `rank` (all partitions when rank < 0). */
dvsg_status dvsg_load_index_file(dvsg_ctx *ctx, const char *path, int rank);
/* FNSY v1 writer (index_file.cpp:88-147) over caller arrays: cluster c owns
 * rows [offsets[c], offsets[c+1]) of vectors / adjacency / global_ids. */
dvsg_status dvsg_save_index_file(const char *path, int clusters, int dim, int out_degree,
                                 const float *centroids, const uint32_t *cluster_to_rank,
                                 int ranks, const uint64_t *offsets, const float *vectors,
                                 const uint32_t *adjacency, const uint32_t *global_ids);
/* Shape of the loaded index: number of partitions resident on this context,
 * dims, and the partition -> cluster id map (array of nparts, may be NULL). */
dvsg_status dvsg_index_info(dvsg_ctx *ctx, int *nparts, int *dim, int *out_degree,
                            int *clusters, uint32_t *cluster_ids, uint64_t *sizes);
/* Downloads one resident partition's entry order (n u32) for checking. */
dvsg_status dvsg_get_entry_order(dvsg_ctx *ctx, uint32_t cluster, uint32_t *out);

/* compute_entry_order, graph_index.cpp:21-44 (host, exact) */
dvsg_status dvsg_compute_entry_order(const float *vectors, uint64_t n, int dim, uint32_t *out);

/* ---- the search (beam_search_stats, graph_index.cpp:105-187) ------------ */

/* Batched beam_search_stats of nq queries against one resident partition.
 * Host buffers.  out_ids/out_dists: nq x k, ascending (dist, global id);
 * out_count[q] <= k (ragged); out_visited[q] = the reference's scored count. */
dvsg_status dvsg_beam_search(dvsg_ctx *ctx, uint32_t cluster, const float *queries,
                             uint64_t nq, int dim, const dvsg_search_params *p,
                             uint32_t *out_ids, float *out_dists, uint32_t *out_count,
                             uint64_t *out_visited);

/* Device-pointer variant over an explicit unit list: unit u searches query
 * unit_query[u] (row of d_queries, nq x dim) in partition unit_cluster[u].
 * All pointers are device pointers on this context's device; runs on the
 * compute stream, asynchronous. */
dvsg_status dvsg_search_units_device(dvsg_ctx *ctx, const float *d_queries, uint64_t nq,
                                     int dim, const uint32_t *d_unit_query,
                                     const uint32_t *d_unit_cluster, uint64_t nunits,
                                     const dvsg_search_params *p, uint32_t *d_out_ids,
                                     float *d_out_dists, uint32_t *d_out_count,
                                     uint64_t *d_out_visited);

/* ---- node-sharded search (north-star frontier exchange) -----------------
 * The graph's vectors are split across ranks (node v on rank v / ceil(n/R));
 * adjacency, global ids and entry order are replicated.  One fused kernel per
 * GPU: the origin keeps pool + visited set, pushes remote candidate ids (and
 * the query) to their owners by NVLink peer stores, owners score against
 * their rows and push keys back; results are identical to the unsharded
 * beam_search_stats (graph_index.cpp:105-187). */

/* All R ranks emulated in one launch on this device over the resident
 * whole-graph partition (for parity tests without R GPUs).  Host buffers. */
dvsg_status dvsg_beam_search_sharded_emulated(dvsg_ctx *ctx, int nranks, const float *queries,
                                              uint64_t nq, int dim, const dvsg_search_params *p,
                                              uint32_t *out_ids, float *out_dists,
                                              uint32_t *out_count, uint64_t *out_visited);
/* Multi-GPU, one process per GPU: load this rank's shard rows
 * [rank*S, min(n,(rank+1)*S)) with S = ceil(n_total/nranks) plus the
 * replicated adjacency / global ids (NULL = iota) / entry order (required,
 * graph_index.cpp:21-44 over the whole graph); allocates the comm arena. */
dvsg_status dvsg_shard_init(dvsg_ctx *ctx, int nranks, int rank, uint64_t n_total, int dim,
                            int out_degree, const float *shard_vectors, const uint32_t *adjacency,
                            const uint32_t *global_ids, const uint32_t *entry_order);
/* Same, from the context's one resident partition (e.g. built on the
 * device with dvsg_partition_alloc_device): every rank builds or loads the
 * whole graph, then keeps only its shard rows of the vectors -- no host copy
 * of a 50 GB index. */
dvsg_status dvsg_shard_init_resident(dvsg_ctx *ctx, int nranks, int rank);
/* 64-byte IPC handle of this rank's comm arena (exchange it across ranks). */
dvsg_status dvsg_shard_export(dvsg_ctx *ctx, void *handle_out);
/* Open every rank's arena (handles: nranks x 64 bytes, in rank order). */
dvsg_status dvsg_shard_connect(dvsg_ctx *ctx, const void *handles);
/* Reset this rank's arena before a search; all ranks must finish it (host
 * barrier) before any rank launches. */
dvsg_status dvsg_shard_prepare(dvsg_ctx *ctx);
/* Sharded search of this rank's nq queries (device pointers, async on the
 * compute stream); every rank must launch it concurrently. */
dvsg_status dvsg_search_sharded_device(dvsg_ctx *ctx, const float *d_queries, uint64_t nq, int dim,
                                       const dvsg_search_params *p, uint32_t *d_out_ids,
                                       float *d_out_dists, uint32_t *d_out_count,
                                       uint64_t *d_out_visited);

/* Exchange algorithm of the node-sharded search (both exact):
 *   0  bulk-synchronous (default): per phase, xg_expand pushes every query's
 *      new candidates into the owners' inboxes, a peer-flag barrier, xg_score
 *      scores them and pushes the keys back, a barrier (xchg_kernel.cu);
 *   1  fused: one persistent kernel, per-CTA request/reply round trips
 *      (shard_kernel.cu);
 *   2  nccl: see below.
 * Default from the environment (DVSG_SHARD_EXCHANGE=fused|nccl), else 0.  With the
 * bulk exchange, dvsg_search_sharded_device is collective: every rank must
 * call it with the same nq and params; dvsg_synchronize reports a rank that
 * never reached a barrier (DVSG_EINTERNAL after 20 s). */
dvsg_status dvsg_set_shard_exchange(dvsg_ctx *ctx, int mode);
/* Mode 2 -- the NCCL baseline of the bulk exchange (north_star: "an NCCL
 * all-to-all variant kept only as the measured baseline"): the same
 * xg_step kernels over local send/receive slabs, with host-driven
 * ncclSend/ncclRecv of the requests and replies after each half-phase (their
 * sizes go through the host, two stream syncs per phase).  libnccl.so.2 is
 * loaded at run time.  Rank 0 creates the id, every rank connects with it. */
dvsg_status dvsg_nccl_unique_id(dvsg_ctx *ctx, void *id_out128);
dvsg_status dvsg_nccl_connect(dvsg_ctx *ctx, const void *id128);

/* ---- cluster-sharded run_pipeline, device-initiated exchange ------------
 * SURVEY 8e design A: cluster i lives on rank placement[i] (router.cpp:28-43),
 * every rank holds the centroids + placement (dvsg_set_centroids) and its own
 * partitions, and is the origin of its own query batch.  One call per step on
 * every rank (collective, asynchronous on the compute stream): K5 assign ->
 * K3 dispatch (each routed unit's query + header stored into the owner's
 * inbox over NVLink, route router.cpp:52-79) -> peer-flag barrier -> K1 over
 * the units this rank owns -> results (+ hit vectors) stored into each
 * origin's reply slots -> barrier -> K4 combine_results (simulator.cpp:219-243)
 * and the hit vectors (:329-333).  Results equal run_pipeline over the whole
 * index on one GPU.  Replaces the NCCL all-to-alls of the Python driver. */
dvsg_status dvsg_cluster_comm_init(dvsg_ctx *ctx, int nranks, int rank, uint64_t max_queries,
                                   int max_fanout, int k, int with_vectors);
/* 64-byte IPC handle of this rank's arena; connect with every rank's (rank order). */
dvsg_status dvsg_cluster_comm_export(dvsg_ctx *ctx, void *handle_out);
dvsg_status dvsg_cluster_comm_connect(dvsg_ctx *ctx, const void *handles);
/* Same process, same device (tests): the arenas' device pointers directly. */
void *dvsg_cluster_comm_arena(dvsg_ctx *ctx);
dvsg_status dvsg_cluster_comm_connect_local(dvsg_ctx *ctx, void *const *arenas);
dvsg_status dvsg_run_pipeline_cluster_device(dvsg_ctx *ctx, const float *d_queries, uint64_t nq,
                                             int dim, const dvsg_search_params *p, int fanout,
                                             uint32_t *d_out_ids, float *d_out_dists,
                                             uint32_t *d_out_count, float *d_out_vectors,
                                             uint64_t *d_visited_total);
/* Synchronizes and reports an error of the last step (overflow, routing,
 * barrier timeout, unsorted partial). */
dvsg_status dvsg_cluster_comm_check(dvsg_ctx *ctx);

/* ---- routing and merge -------------------------------------------------- */

/* assign_top_c, kmeans.cpp:243-280, on the GPU against the context's
 * centroids.  Host buffers; out is nq x c cluster ids. */
dvsg_status dvsg_assign_top_c(dvsg_ctx *ctx, const float *queries, uint64_t nq, int dim,
                              int c, uint32_t *out);

/* combine_results, simulator.cpp:219-243, on the GPU.  nq queries, each with
 * nparts partial lists of <= stride entries (counts nq x nparts); out nq x k. */
dvsg_status dvsg_combine_results(dvsg_ctx *ctx, uint64_t nq, int nparts, const uint32_t *ids,
                                 const float *dists, const uint32_t *counts, int stride, int k,
                                 uint32_t *out_ids, float *out_dists, uint32_t *out_count);

/* Device-pointer variants (asynchronous on the compute stream; combine
 * synchronizes to report an unsorted partial), used by the multi-GPU
 * cluster-sharded pipeline (paper_2512_02278_b200/dist.py,
 * run_pipeline_distributed).  gather_vectors: hit vectors of n result lists
 * (k ids each, counts[i] valid) from the resident partitions, n x k x dim. */
dvsg_status dvsg_assign_top_c_device(dvsg_ctx *ctx, const float *d_queries, uint64_t nq, int dim,
                                     int c, uint32_t *d_out);
dvsg_status dvsg_combine_results_device(dvsg_ctx *ctx, uint64_t nq, int nparts, const uint32_t *d_ids,
                                        const float *d_dists, const uint32_t *d_counts, int stride,
                                        int k, uint32_t *d_out_ids, float *d_out_dists,
                                        uint32_t *d_out_count);
dvsg_status dvsg_gather_vectors_device(dvsg_ctx *ctx, const uint32_t *d_ids, const uint32_t *d_counts,
                                       uint64_t n, int k, float *d_out);

/* ---- run_pipeline functional part (simulator.cpp:245-337), one GPU ------
 * assign (K5) -> route -> search (K1) -> combine (K4) -> attach hit vectors.
 * All clusters must be resident on this context.  Host buffers;
 * out_vectors (nq x k x dim) may be NULL; visited_total may be NULL. */
dvsg_status dvsg_run_pipeline(dvsg_ctx *ctx, const float *queries, uint64_t nq, int dim,
                              const dvsg_search_params *p, int fanout, int ranks,
                              int batch_index, uint32_t *out_ids, float *out_dists,
                              uint32_t *out_count, float *out_vectors, uint64_t *visited_total);
/* Same, device pointers, asynchronous on the compute stream.  d_visited is
 * per (query, fanout slot) (nq x fanout) and may be NULL. */
dvsg_status dvsg_run_pipeline_device(dvsg_ctx *ctx, const float *d_queries, uint64_t nq,
                                     int dim, const dvsg_search_params *p, int fanout,
                                     uint32_t *d_out_ids, float *d_out_dists,
                                     uint32_t *d_out_count, float *d_out_vectors,
                                     uint64_t *d_visited);

/* ---- graph build (build_graph, graph_index.cpp:46-97) -------------------
 * Exact kNN rows (ties by lower id) on the GPU over a host partition; the
 * distance is fp32 over (x-y)^2, exact for integer-valued data (SIFT-like
 * bytes), within fp32 rounding otherwise.  adjacency_out: n x out_degree. */
dvsg_status dvsg_build_graph(dvsg_ctx *ctx, const float *vectors, uint64_t n, int dim,
                             int out_degree, uint32_t *adjacency_out);

/* ---- partitioning (kmeans_train kmeans.cpp:189-241, partition_database
 *      :282-300; build_index index.cpp:43-72 composes them) ---------------- */

/* kmeans_train on the GPU with the reference's control flow and rounding:
 * k-means++ seeding from std::mt19937_64(seed), Lloyd iterations with
 * repair_empty_clusters and the fixed-point test, the final non-empty check.
 * db: n x dim host rows; centroids_out: clusters x dim; iterations_out and
 * wcss_out (max_iters doubles) may be NULL (KmeansStats, kmeans.hpp:27-30).
 * Bit-identical to the reference on integer-valued data (kmeans++ prefix sums
 * exact); errors as the reference (DVSG_EINVAL). */
dvsg_status dvsg_kmeans_train(dvsg_ctx *ctx, const float *db, uint64_t n, int dim, int clusters,
                              int max_iters, uint64_t seed, float *centroids_out,
                              int *iterations_out, double *wcss_out);
/* partition_database: the nearest centroid of every row (expanded_dist,
 * ties to the lower id) -> labels_out[n]; the reference's per-cluster id
 * lists are the rows of each label in row order. */
dvsg_status dvsg_partition_database(dvsg_ctx *ctx, const float *db, uint64_t n, int dim,
                                    const float *centroids, int clusters, uint32_t *labels_out);

/* ---- ground truth (brute_force_topk, topk.cpp:12-30) ---------------------
 * Exact top-k by (dist, id) of nq queries over the n x dim database (host
 * buffers), k <= 32; fp32 distances over (x - y)^2, exact for integer-valued
 * data.  Used for recall@k at sizes the CPU oracle cannot reach. */
dvsg_status dvsg_brute_force_topk(dvsg_ctx *ctx, const float *db, uint64_t n, int dim,
                                  const float *queries, uint64_t nq, int k, uint32_t *out_ids,
                                  float *out_dists);

/* ---- large-index construction on the device (csrc/ivf_build.cu) ----------
 * The pieces a 10M-100M-row index is built from without leaving HBM.  All
 * pointers are device pointers on the context's device; every call is
 * synchronous (it returns after its kernels finished).
 *
 * K7 range top-m: for each block, the rows [row0, row0+nrows) (nrows <= 128)
 * of d_rows against the column ranges ranges[list_off[list] ..
 * list_off[list+1]) (pairs {begin, end} of d_cols rows, disjoint): the m <= 32
 * smallest (squared L2, column id) keys -- the ordering of scored_less
 * (dataset.hpp:33-46) -- written to rows out_row0 + i of d_out_ids /
 * d_out_dists (nullable), out_stride entries per row.  Distances use the dot
 * form over precomputed fp32 norms (dvsg_row_norms_device): exact on
 * integer-valued data below 2^24 per term.  Serves the cluster-restricted
 * graph build that stands in for build_graph (graph_index.cpp:46-97) at
 * 10^16-pair sizes, nearest-centroid assignment, and brute-force ground truth
 * (topk.cpp:12-30) split over column ranges.  Missing entries (fewer than m
 * candidates) are id 0xFFFFFFFF / +inf, or with DVSG_RANGE_BUILD_PAD the
 * valid ones repeated cyclically (graph_index.cpp:86-92).  d_row_map
 * (nullable): block row i reads physical row d_row_map[row0 + i] of d_rows
 * (and its norm), so a permuted view needs no gathered copy. */
typedef struct {
  uint32_t row0, nrows, list, out_row0;
} dvsg_range_block;
#define DVSG_RANGE_EXCLUDE_SELF 1 /* skip column == row (d_rows == d_cols) */
#define DVSG_RANGE_BUILD_PAD 2
#define DVSG_RANGE_MERGE 4 /* start from the lists already in d_out_ids / d_out_dists (ids
                              0xFFFFFFFF = empty): several passes over disjoint ranges give
                              the top-m of their union */
#define DVSG_RANGE_OUT_PHYSICAL 8 /* outputs (and merge inputs) at row d_row_map[row0 + i] */
dvsg_status dvsg_range_topk_device(dvsg_ctx *ctx, const float *d_rows, const float *d_row_norms,
                                   const float *d_cols, const float *d_col_norms, int dpad,
                                   const uint32_t *d_row_map, const dvsg_range_block *d_blocks,
                                   uint64_t nblocks,
                                   const uint32_t *d_list_off, const uint32_t *d_ranges, int m,
                                   int flags, uint32_t *d_out_ids, float *d_out_dists,
                                   uint64_t out_stride);
/* K7 on the tensor cores (csrc/ivf_tc.cu): the same contract over bf16 rows /
 * columns (n x kpad, kpad a multiple of 16 <= 256, zero pad), one
 * tcgen05.mma (M=128, N=128, K=16) per K slice into TMEM, top-m epilogue
 * from tcgen05.ld.  Exact (== dvsg_range_topk_device) when the data are
 * integers in [-256, 256] (bf16-exact, every fp32 partial sum exact). */
dvsg_status dvsg_range_topk_bf16_device(dvsg_ctx *ctx, const uint16_t *d_rows, const float *d_row_norms,
                                        const uint16_t *d_cols, const float *d_col_norms, int kpad,
                                        const uint32_t *d_row_map, const dvsg_range_block *d_blocks,
                                        uint64_t nblocks, const uint32_t *d_list_off,
                                        const uint32_t *d_ranges, int m, int flags, uint32_t *d_out_ids,
                                        float *d_out_dists, uint64_t out_stride);
/* n rows of dpad floats -> n rows of kpad bf16 (round to nearest even, zero pad) */
dvsg_status dvsg_to_bf16_device(dvsg_ctx *ctx, const float *d_x, uint64_t n, int dpad, int kpad,
                                uint16_t *d_out);
/* fp32 squared norms of n rows of dpad floats */
dvsg_status dvsg_row_norms_device(dvsg_ctx *ctx, const float *d_x, uint64_t n, int dpad,
                                  float *d_out);
/* Segment means for the clustering: d_cents[s] = f32(fp64 in-order sum of
 * rows d_idx[d_off[s] .. d_off[s+1]) / count) (d_idx NULL: rows d_off[s]..);
 * empty segments keep their centroid.  Deterministic (no atomics). */
dvsg_status dvsg_segment_means_device(dvsg_ctx *ctx, const float *d_x, int dpad,
                                      const uint32_t *d_idx, const uint64_t *d_off, uint32_t nseg,
                                      float *d_cents);
/* compute_entry_order (graph_index.cpp:21-44) on the device, bit-exact: fp64
 * column sums in row order, f32 mean, fp64 sequential squared_l2 per row,
 * sort by (f32 dist, id).  dim <= 1024. */
dvsg_status dvsg_compute_entry_order_device(dvsg_ctx *ctx, const float *d_x, uint64_t n, int dim,
                                            int dpad, uint32_t *d_out);
/* Build a partition in place: reserves n rows in the context's index arrays
 * and returns device pointers to them (vectors n x dpad with dpad = dim
 * rounded up to 4, pad columns zeroed; adjacency n x out_degree local ids;
 * global ids; entry order), which the caller fills; then commit validates it
 * on the device (ids in range, finite, pad zero) and makes it resident, like
 * dvsg_load_partition without a host copy of a 50 GB index. */
dvsg_status dvsg_partition_alloc_device(dvsg_ctx *ctx, uint32_t cluster, uint64_t n, int dim,
                                        int out_degree, float **d_vectors, uint32_t **d_adjacency,
                                        uint32_t **d_global_ids, uint32_t **d_entry_order);
#define DVSG_COMMIT_ENTRY_ORDER 1 /* compute the entry order on the device */
#define DVSG_COMMIT_IOTA_IDS 2    /* global ids = 0..n-1 */
dvsg_status dvsg_partition_commit_device(dvsg_ctx *ctx, int flags);
/* CAGRA-style optimisation of a kNN graph (rows sorted by distance), in
 * place on device adjacency (n x out_degree local ids, n < 2^27, degree
 * <= 32): rank-based detour pruning keeps `keep` forward edges per row, the
 * rest of each row becomes reverse edges (in-edges closest in forward rank
 * first), then the remaining forward edges; no duplicates.  Deterministic.
 * The search (graph_index.cpp:105-187) is unchanged; only its graph is. */
dvsg_status dvsg_optimize_graph_device(dvsg_ctx *ctx, uint32_t *d_adjacency, uint64_t n,
                                       int out_degree, int keep);
/* Read-only device pointers to a resident partition's arrays (vectors
 * n x dpad, adjacency n x out_degree, global ids, entry order), valid until
 * the next index change. */
dvsg_status dvsg_partition_view_device(dvsg_ctx *ctx, uint32_t cluster, const float **d_vectors,
                                       const uint32_t **d_adjacency, const uint32_t **d_global_ids,
                                       const uint32_t **d_entry_order, uint64_t *n);
/* 1 when every resident row is integer-valued below 2^24, i.e. the fp32 fast
 * mode is exact; otherwise DVSG_ACCUM_F32 searches run in DVSG_ACCUM_F32C
 * (inner product or dim >= 384) or DVSG_ACCUM_F64. */
dvsg_status dvsg_index_integral(dvsg_ctx *ctx, int *out);

/* ---- instrumentation ---------------------------------------------------- */
/* Device time (ms) of the last search kernel launch (K1) and of the whole
 * last pipeline call, measured with CUDA events on the compute stream;
 * enable with dvsg_set_timing(ctx, 1). */
dvsg_status dvsg_set_timing(dvsg_ctx *ctx, int enabled);
/* Measured timeline of the last dvsg_run_pipeline with timing on (SURVEY
 * 8f-4; the reference models one in replay_schedule, simulator.cpp:71-168):
 * per microbatch 6 times in ms from the pipeline start -- H2D start/end
 * (copy stream), compute start/end (compute stream: finiteness check,
 * assign, route, K1, combine, hit vectors), D2H start/end (copy stream).
 * out holds 6 x max_microbatches doubles; *n_out = microbatches written. */
dvsg_status dvsg_last_pipeline_timeline(dvsg_ctx *ctx, double *out, int max_microbatches, int *n_out);
/* Measured timeline of the last node-sharded bulk / NCCL search with timing
 * on: per interval {kind (0 step kernel, 1 peer barrier or NCCL exchange),
 * start ms, end ms} from the search start; out holds 3 x max_intervals. */
dvsg_status dvsg_last_sharded_timeline(dvsg_ctx *ctx, double *out, int max_intervals, int *n_out);
dvsg_status dvsg_last_timings(dvsg_ctx *ctx, float *search_ms, float *assign_ms,
                              float *combine_ms, float *total_ms);
/* Number of library kernels launched by this context since creation. */
uint64_t dvsg_kernel_launches(dvsg_ctx *ctx);
/* Which K5 variant served the last assign_top_c / run_pipeline assign of
 * this context: 0 warp kernel (C < 8), 1 exact fp64 tiles, 2 tensor cores
 * (TF32 tcgen05 candidates + exact fp64 re-rank + certificate; *fallbacks =
 * queries whose certificate failed and were finished by the exact kernel).
 * -1 before any assign.  Results are identical on every path. */
dvsg_status dvsg_last_assign_info(dvsg_ctx *ctx, int *path, uint64_t *fallbacks);
/* Vector storage K1 reads (whole-graph searches: dvsg_beam_search*,
 * dvsg_search_units*, dvsg_run_pipeline*).  DVSG_STORAGE_U8 keeps a byte copy
 * of the resident rows and gathers a quarter of the bytes; results are
 * bit-identical because every coordinate must be an integer in [0, 255]
 * (checked here: DVSG_EINVAL otherwise; dim <= 256).  The copy is dropped
 * automatically when the rows change (call again after loading).  An
 * extension (the reference stores fp32 only); DVSG_STORAGE_F32 is the default. */
#define DVSG_STORAGE_F32 0
#define DVSG_STORAGE_U8 1
dvsg_status dvsg_set_vector_storage(dvsg_ctx *ctx, int mode);
/* How the last dvsg_build_graph / dvsg_brute_force_topk of this context ran:
 * *exact_mode 0 = fp32 tiles (byte-like data: every squared distance an exact
 * fp32 integer), 1 = fp32 candidates + fp64 re-rank + certificate (any float
 * data); *fallbacks = rows the certificate sent to the fp64 full scan.  -1
 * before any call.  Results equal the reference's either way. */
dvsg_status dvsg_last_knn_info(dvsg_ctx *ctx, int *exact_mode, uint64_t *fallbacks);
/* Totals of the last K1 launch: units searched, vectors scored (the
 * reference's visited counter) and frontier nodes expanded -- the inputs of
 * the algorithmic byte count visited*4d + expanded*4*d_g + 4d per unit. */
dvsg_status dvsg_last_search_stats(dvsg_ctx *ctx, uint64_t *units, uint64_t *visited,
                                   uint64_t *expanded);
/* Raw K1 counters of the last launch (16 u64; [0] work counter, [1..3] the
 * stats above, [3..] kernel-variant debug counters, zero in release builds). */
dvsg_status dvsg_debug_counters(dvsg_ctx *ctx, uint64_t *out16);

#ifdef __cplusplus
}
#endif
#endif
