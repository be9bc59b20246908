// dvsg_internal.h -- shared device-side definitions of libdvsg (not public API).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

// Race stress build (-DDVSG_STRESS=1; scripts/stress_check.sh): after every
// block / warp barrier a pseudo-random 1/8 of the threads sleep up to ~4 us,
// so code that relies on timing instead of a barrier (a missing
// __syncthreads / __syncwarp, a read racing a write) sees its other
// interleavings.  compute-sanitizer is not available on this pool; the parity
// suite run against this build is the substitute.  Never in release builds.
#if defined(__CUDACC__) && defined(DVSG_STRESS) && DVSG_STRESS
__device__ __forceinline__ void dvsg_jitter() {
  unsigned t = (unsigned)clock() * 2654435761u ^ (threadIdx.x * 40503u) ^ (blockIdx.x * 9973u);
  t ^= t >> 15;
  t *= 2246822519u;
  if ((t >> 29) == 0) __nanosleep((t >> 6) & 4095u);
}
#define __syncthreads() (__syncthreads(), dvsg_jitter())
#define __syncwarp(...) (__syncwarp(__VA_ARGS__), dvsg_jitter())
#endif

namespace dvsg {

#ifndef DVSG_K1_THREADS
#define DVSG_K1_THREADS 256
#endif
constexpr int kThreads = DVSG_K1_THREADS;  // K1 CTA size (8 warps; build variants may change it)
constexpr int kWarps = kThreads / 32;
constexpr uint32_t kEmpty = 0xFFFFFFFFu;

// One resident partition (a GraphIndex, graph_index.hpp:13-25) inside the
// context's concatenated device arrays: rows [row_off, row_off + n) of
// vectors (dpad floats per row, 16-B aligned), adjacency (dg local ids per
// row), global ids and entry order.
struct PartDesc {
  uint64_t row_off;
  uint32_t n;
  uint32_t cluster;
};

struct SearchArgs {
  const float* vectors;       // rows x dpad
  const uint8_t* vectors8;    // nullable: the same rows as bytes (dvsg_set_vector_storage U8; dpad <= 256)
  const uint32_t* adjacency;  // rows x dg
  const uint32_t* gids;       // rows
  const uint32_t* entry;      // rows (per-partition entry order)
  const PartDesc* parts;      // partition slots
  const float* queries;       // nq x dim (unpadded)
  uint64_t nq;
  const uint32_t* unit_query;  // nunits
  const uint32_t* unit_part;   // nunits (partition slot)
  const uint32_t* unit_order;  // nullable: CTAs claim units in this order (locality); outputs stay per unit
  uint64_t nunits;
  int dim, dpad, dg;
  int iters, beam, k, entry_count, cap;
  int chp;      // survivor buffer entries (pow2 >= max(chunk, cap))
  int hsize;    // visited hash slots (pow2)
  int hsmall;   // K1, global hash: > 0 -> start each unit in a hsmall-slot table and
                // move to the full hsize one only when the load could pass 3/4
                // (per-CTA region = hsmall + hsize slots); 0 -> full table
  uint32_t* hash_global;  // nullptr -> visited hash in shared memory
  uint32_t* out_ids;      // nunits x k
  float* out_dists;       // nunits x k
  uint32_t* out_count;    // nunits
  uint64_t* out_visited;  // nunits
  unsigned long long* work_counter;
  unsigned long long* stats;  // [0] units, [1] visited, [2] expanded (frontier nodes); nullable
  const unsigned long long* nunits_dev;  // nullable: unit count produced on the device (<= nunits)
};

// ---- node-sharded K1 (shard_kernel.cu) ------------------------------------
// Vectors of node v live on rank v / shard_rows; adjacency, global ids and
// entry order are replicated.  Each rank's comm arena holds its doorbell ring,
// the mailboxes peers push candidate ids + query into, the reply boxes peers
// push scored keys into, and counters.  `views` gives every rank's arena (peer
// pointers over NVLink, or slices of one device when emulating ranks).
struct ShardView {
  const float* vec;              // this rank's shard rows (dpad floats each)
  uint32_t* ring;                // doorbell ring [ring_mask + 1], entries (origin<<16 | cta) + 1
  unsigned* ring_tail;           // producers reserve slots (peer atomics)
  unsigned* ring_head;           // local consumers claim slots
  unsigned char* mail;           // [nranks * gpr] mailboxes, mail_stride bytes each
  unsigned char* reply;          // [gpr * nranks] reply boxes, reply_stride bytes each
  unsigned* done;                // ranks that finished all their units
  unsigned* finished;            // CTAs of this rank that finished their units
  unsigned long long* work;      // this rank's unit counter
};

struct ShardArgs {
  const ShardView* views;        // device array [nranks]
  int nranks;
  int rank_self;                 // >= 0: one rank per launch (multi-GPU); -1: emulate all ranks
  int gpr;                       // CTAs per rank
  uint64_t shard_rows;           // S
  uint32_t ring_mask;
  uint32_t mail_stride;
  uint32_t reply_stride;
  uint64_t units_per_rank;       // emulation: rank r owns units [r*upr, (r+1)*upr)
  int origin_ctas;               // CTAs [0, origin_ctas) of a rank search; the rest only serve
};

// Comm-arena layout helpers (bytes), shared by host and device.
__host__ __device__ inline uint32_t shard_mail_stride(int dpad) {
  return (uint32_t)(16 + 4 * dpad + 4 * 2048 + 15) & ~15u;
}
__host__ __device__ inline uint32_t shard_reply_stride() { return 16 + 8 * 2048; }

cudaError_t launch_search_sharded(const SearchArgs& a, const ShardArgs& sh, int metric, int accum,
                                  int num_sms, cudaStream_t stream, int* grid_out,
                                  int* gpr_out);
// CTAs per rank the sharded kernel can keep resident for these args.
int search_sharded_blocks_per_sm(const SearchArgs& a, int metric, int accum);

// ---- node-sharded, bulk-synchronous frontier exchange (xchg_kernel.cu) ----
// Same shard rule as above (node v on rank v / shard_rows).  Per phase every
// rank's origins push their new candidate ids into the owners' inboxes, the
// owners score them and push the keys back; a peer-flag barrier separates the
// phases.  Each rank's comm arena (IPC-exported) holds:
struct XgView {
  const float* vec;    // this rank's shard rows: node v at vec + (v - lo) * dpad (owner side)
  uint64_t lo;
  unsigned* cursor;    // [2][nranks] inbox fill per origin, slot = phase & 1
  unsigned* flags;     // [nranks] barrier epoch last published by each rank
  float* qall;         // [nranks][wcap][dpad] every origin's queries (this wave)
  uint64_t* inbox;     // [nranks][rstride] requests (qid << 32 | node) from each origin
  uint64_t* reply;     // [nranks][rstride] keys scored by each owner, same index as its inbox
};

constexpr int kXgMaxRanks = 8;

struct XgArgs {
  const XgView* views;  // device array [nranks]
  int nranks;
  int rank_lo, rank_n;  // ranks this launch acts for (multi-GPU: self, 1; emulation: 0, R)
  uint32_t wave_n[kXgMaxRanks];  // queries of each acting rank in this wave
  uint32_t wcap;        // per-rank query capacity (state / qall stride)
  uint32_t maxraw;      // max new candidates per query per phase
  uint64_t rstride;     // wcap * maxraw
  uint32_t shard_rows;  // S
  int phase;            // 0: entry nodes, 1..iters: expansions, iters + 1: finalize
  // origin state, [rank_n][wcap] (acting-rank relative)
  uint64_t* pool;       // x cap
  uint32_t* psize;
  uint64_t* visited;
  uint32_t* expd;
  uint32_t* hash;       // x hsize
  uint2* meta;          // x nranks: (inbox position, count) at each owner, last phase
  // replicated graph
  const uint32_t* adjacency;
  const uint32_t* gids;
  const uint32_t* entry;
  uint32_t n;
  int dim, dpad, dg, iters, beam, k, entry_count, cap, chp, hsize;
  // outputs: acting rank rr's wave query j at [rr * out_stride + j]
  uint32_t* out_ids;
  float* out_dists;
  uint32_t* out_count;
  uint64_t* out_visited;
  uint64_t out_stride;
  unsigned long long* stats;  // [0] units, [1] visited, [2] expanded
  int* err;
};

size_t xg_expand_smem_bytes(int cap, int chp, int beam, int maxraw);
// One phase step (xg_step): expand items of lane ea (do_e) and score items of
// lane sa (do_s), claimed interleaved from *counter (zeroed by the caller).
cudaError_t launch_xg_step(const XgArgs& ea, const XgArgs& sa, int do_e, int do_s,
                           unsigned long long* counter, int metric, int accum, int num_sms,
                           cudaStream_t stream);
// Peer-flag barrier over all ranks (one thread); sets bit 3 of *err after a 20 s timeout.
cudaError_t launch_xg_barrier(const XgView* views, int nranks, int me, unsigned epoch, int* err,
                              cudaStream_t stream);

// Launch K1 (search_kernel.cu).  Returns a cudaError_t.
// max_grid > 0 caps the persistent grid (one global hash region per CTA).
cudaError_t launch_search(const SearchArgs& a, int metric, int accum, int num_sms,
                          int max_grid, cudaStream_t stream, int* grid_out);
// Byte copy of float rows for the U8 vector storage: out[i] = x[i] when every
// element is an integer in [0, 255]; otherwise bit 0 of *bad is set.
cudaError_t launch_to_u8(const float* x, uint64_t n, uint8_t* out, int* bad, cudaStream_t stream);
// Shared-memory bytes K1 needs for these args (hash in smem when hash_global==nullptr).
size_t search_smem_bytes(int cap, int chp, int beam, int hsize, bool hash_in_smem);
constexpr int kChunk = 8 * kThreads;  // raw candidates per dedup/score/merge chunk (8 per thread)

// K5 assign (route_kernels.cu): nq x c cluster ids, exact fp64 expanded form.
// scratch: assign_scratch_words(...) u64.  *path (nullable) = 0 warp kernel,
// 1 fp64 tiles, 2 tensor cores (TF32 candidates + exact re-rank; word 0 of
// the scratch then holds the number of queries the certificate sent to the
// exact kernel).
size_t assign_scratch_words(uint64_t nq, int dim, int clusters, int c);
cudaError_t launch_assign(const float* queries, uint64_t nq, int dim, const float* cents,
                          const double* cent_norms, int clusters, int c, uint32_t* out,
                          uint64_t* scratch, cudaStream_t stream, int* path = nullptr);
// K4 combine: per query merge nparts sorted partial lists (stride entries each).
cudaError_t launch_combine(uint64_t nq, int nparts, const uint32_t* ids, const float* dists,
                           const uint32_t* counts, int stride, int k, uint32_t* out_ids,
                           float* out_dists, uint32_t* out_count, int* err_flag,
                           cudaStream_t stream);
// Route: build (unit_query, unit_part) from the assignment and the cluster->slot map
// (nmap entries); an id >= nmap or a non-resident cluster sets bit 0 of *err_flag.
cudaError_t launch_route(const uint32_t* assign, uint64_t nq, int fanout,
                         const int32_t* cluster_to_slot, uint32_t nmap, uint32_t* unit_query,
                         uint32_t* unit_part, int* err_flag, cudaStream_t stream);
// Attach hit vectors (simulator.cpp:329-333): gid -> (slot row) locator.
cudaError_t launch_gather_vectors(const uint32_t* ids, const uint32_t* counts, uint64_t nq,
                                  int k, const uint64_t* locator, const float* vectors,
                                  int dim, int dpad, float* out, cudaStream_t stream);
// Locality order of units: bucket each unit's query by its nearest anchor
// (fp32; any order gives identical results), then a counting sort over the
// buckets.  anchors: na x dpad; scratch: nunits + na + 1 u32.
cudaError_t launch_locality_order(const float* queries, int dim, const uint32_t* unit_query,
                                  uint64_t nunits, const float* anchors, int na, int dpad,
                                  uint32_t* scratch, uint32_t* order, cudaStream_t stream);
// Flag bit 2 of *flag when any of x[0..n) is non-finite.
cudaError_t launch_check_finite(const float* x, uint64_t n, int* flag, cudaStream_t stream);
// Sum of per-unit visited counters.
cudaError_t launch_reduce_u64(const uint64_t* in, uint64_t n, unsigned long long* out,
                              cudaStream_t stream);

// Exact brute-force top-k (topk.cpp:12-30) of nq queries over n rows (k <= 32).
cudaError_t launch_brute_force(const float* queries, uint64_t nq, const float* db, uint64_t n,
                               int dpad, int k, uint32_t* out_ids, float* out_dists,
                               cudaStream_t stream);
// ---- large-index construction (ivf_build.cu) -------------------------------
// One K7 work item: rows [row0, row0 + nrows) (nrows <= 128) against the
// column ranges ranges[list_off[list] .. list_off[list + 1]); outputs go to
// rows out_row0 + i of out_ids / out_dists (out_stride entries per row).
struct RangeBlock {
  uint32_t row0, nrows, list, out_row0;
};
// flags: bit 0 exclude column == row (rows and cols are the same array);
// bit 1 build_graph padding (cyclic repeat of short lists); bit 2 merge into the
// lists already in out_ids / out_dists (multi-pass); bit 3 output row = the
// physical row (row_map[row0 + r]) instead of out_row0 + r.  row_map (nullable):
// block row r reads physical row row_map[row0 + r] of `rows` (norms likewise).
cudaError_t launch_range_topk(const float* rows, const float* rnorm, const float* cols,
                              const float* cnorm, int dpad, const uint32_t* row_map, const RangeBlock* blocks,
                              uint64_t nblocks, const uint32_t* list_off, const uint2* ranges,
                              int m, int flags, uint32_t* out_ids, float* out_dists,
                              uint64_t out_stride, cudaStream_t stream);
size_t range_topk_smem_bytes();
// K7 on the tensor cores (ivf_tc.cu): rows / cols as bf16 (n x kpad, kpad % 16 == 0, <= 256)
cudaError_t launch_range_topk_tc(const uint16_t* rows, const float* rnorm, const uint16_t* cols, const float* cnorm,
                                 int kpad, const uint32_t* row_map, const RangeBlock* blocks, uint64_t nblocks,
                                 const uint32_t* list_off, const uint2* ranges, int m, int flags, uint32_t* out_ids,
                                 float* out_dists, uint64_t out_stride, cudaStream_t stream);
size_t range_topk_tc_smem_bytes(int kpad);
// same over fp32 rows / cols read as tf32 (kind::tf32; kpad % 8 == 0, <= 128)
cudaError_t launch_range_topk_tf32(const float* rows, const float* rnorm, const float* cols, const float* cnorm,
                                   int kpad, const uint32_t* row_map, const RangeBlock* blocks, uint64_t nblocks,
                                   const uint32_t* list_off, const uint2* ranges, int m, int flags, uint32_t* out_ids,
                                   float* out_dists, uint64_t out_stride, cudaStream_t stream);
cudaError_t launch_to_bf16(const float* x, uint64_t n, int dpad, int kpad, uint16_t* out, cudaStream_t stream);
cudaError_t launch_row_norms(const float* x, uint64_t n, int dpad, float* out, cudaStream_t stream);
// Exact compute_entry_order on the device (dim <= 1024).
size_t entry_order_scratch_bytes(uint64_t n);
cudaError_t launch_entry_order(const float* x, uint64_t n, int dim, int dpad, void* scratch,
                               size_t scratch_bytes, uint32_t* out, cudaStream_t stream);
// Partition validators: *flag |= 1 (adjacency id >= n), 4 (non-finite),
// 16 (not integer-valued below 2^24), 32 (non-zero pad column), 64 (gids not
// strictly increasing; gids may be null).
cudaError_t launch_check_partition(const float* x, uint64_t n, int dim, int dpad, const uint32_t* adj,
                                   int dg, const uint32_t* gids, int* flag, cudaStream_t stream);
cudaError_t launch_iota(uint32_t* out, uint64_t n, cudaStream_t stream);
cudaError_t launch_segment_means(const float* x, int dpad, const uint32_t* idx, const uint64_t* off,
                                 uint32_t nseg, float* cents, cudaStream_t stream);

// CAGRA-style rank-based pruning + reverse edges of a kNN graph, in place
// (graph_opt.cu); n < 2^27, 2 <= d <= 32.
size_t graph_opt_scratch_bytes(uint64_t n, int d, int keep);
cudaError_t launch_graph_optimize(uint32_t* adj, uint64_t n, int d, int keep, void* scratch,
                                  size_t scratch_bytes, cudaStream_t stream);

// kmeans_train device parts (kmeans.cu)
cudaError_t launch_kpp_d2(const float* x, uint64_t n, int dim, const float* center, double* d2, int first,
                          cudaStream_t s);
size_t kmeans_scan_bytes(uint64_t n);
cudaError_t launch_kpp_scan(const double* d2, double* scan, uint64_t n, void* temp, size_t temp_bytes,
                            cudaStream_t s);
cudaError_t launch_first_gt(const double* scan, uint64_t n, double r, unsigned long long* out, cudaStream_t s);
cudaError_t launch_own_dist(const float* x, uint64_t n, int dim, const float* cents, const uint32_t* labels,
                            float* out, cudaStream_t s);
cudaError_t launch_cluster_means(const float* x, uint64_t n, int dim, const uint32_t* labels, int clusters,
                                 float* cents, uint32_t* keys_tmp, uint32_t* order, uint32_t* iota,
                                 void* temp, size_t temp_bytes, cudaStream_t s);

// ---- cluster-sharded run_pipeline exchange (cluster_xchg.cu) ---------------
// Each rank's IPC-exported arena: header (barrier flags, per-origin inbox
// cursors by step parity), its inbox (queries + {cluster, origin unit} of the
// units other ranks route to it) and its reply region (per own unit: k ids,
// k dists, count, visited, optional k hit vectors).
struct ClArena {
  unsigned* flags;        // [kXgMaxRanks] barrier epochs published by each rank
  unsigned* cursor;       // [2][kXgMaxRanks] units written into this inbox by each origin, per parity
  float* inbox_q;         // [R][cap][dim]
  uint2* inbox_meta;      // [R][cap] {cluster, origin unit}
  uint32_t* r_ids;        // [ucap][k]
  float* r_dists;         // [ucap][k]
  uint32_t* r_count;      // [ucap]
  uint64_t* r_visited;    // [ucap]
  float* r_vec;           // [ucap][k][dim] or null
};
cudaError_t launch_cl_dispatch(const ClArena* peers, int nranks, int me, int parity, const float* q, uint64_t nq,
                               int dim, int fanout, const uint32_t* assign, const uint32_t* placement,
                               uint32_t nclusters, uint64_t cap, int* err, cudaStream_t s);
cudaError_t launch_cl_units(const ClArena* peers, int nranks, int me, int parity, uint64_t cap,
                            const int32_t* cluster_to_slot, uint32_t nmap, uint32_t* unit_query,
                            uint32_t* unit_part, unsigned long long* nunits, int* err, cudaStream_t s);
cudaError_t launch_cl_reply(const ClArena* peers, int me, uint64_t cap, const uint32_t* unit_query,
                            const unsigned long long* nunits, uint64_t max_units, int k, const uint32_t* ids,
                            const float* dists, const uint32_t* counts, const uint64_t* visited,
                            const uint64_t* locator, const float* vectors, int dim, int dpad, int with_vectors,
                            cudaStream_t s);
cudaError_t launch_cl_reset(const ClArena* peers, int me, int parity, cudaStream_t s);
cudaError_t launch_cl_pick_vectors(const uint32_t* ids, const uint32_t* counts, uint64_t nq, int k, int fanout,
                                   const uint32_t* r_ids, const uint32_t* r_count, const float* r_vec, int dim,
                                   float* out, cudaStream_t s);
cudaError_t launch_cl_barrier(const ClArena* peers, int nranks, int me, unsigned epoch, int* err, cudaStream_t s);

// K6 exact kNN graph rows (knn_build.cu)
cudaError_t launch_knn_build(const float* vectors, uint64_t n, int dim, int dpad,
                             int out_degree, uint32_t* adjacency, cudaStream_t stream);
// K6 exact on any float data: fp32 tiles keep 32 candidates + a lower bound of
// the rest, fp64 re-rank + certificate, fp64 full scan of rejected rows.
// build: rows == cols (graph rows, self excluded, cyclic padding); else brute
// force (ids + dists, deg <= n).  scratch: knn_exact_scratch_bytes(nrows).
size_t knn_exact_scratch_bytes(uint64_t nrows);
cudaError_t launch_knn_exact(const float* rowv, uint64_t nrows, const float* vec, uint64_t n, int dim, int dpad,
                             int deg, bool build, uint32_t* out_ids, float* out_dists, void* scratch,
                             cudaStream_t stream);

}  // namespace dvsg
