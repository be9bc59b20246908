// host.cpp -- C++ host layer + C-ABI of libdvsg.so (declared in include/dvsg.h).
//
// Keeps the reference's index-load / partition / search API
// (/root/reference/proj/include/dvs/{graph_index,index,index_file,kmeans,
// router,simulator}.hpp) and drives the sm_100a kernels in
// search_kernel.cu (K1), route_kernels.cu (K4/K5) and knn_build.cu (K6).
//
// Device layout per context (one CUDA device):
//   vectors   rows x dpad f32 (dpad = dim rounded up to 4: 16-B aligned rows,
//             zero padded -- padding adds exact zeros to every distance)
//   adjacency rows x out_degree u32 (partition-local ids)
//   gids      rows u32, entry rows u32 (per-partition entry order)
//   parts     PartDesc per resident partition (row offset, n, cluster id)
// Partitions are appended; a partition never moves once uploaded except
// when the arrays grow (one device-to-device copy).
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <numeric>
#include <random>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include "../../include/dvsg.h"
#include "dvsg_internal.h"

namespace {

thread_local std::string g_err;

struct Fail {
  int code;
  std::string msg;
};

[[noreturn]] void fail(int code, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  throw Fail{code, buf};
}

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) fail(DVSG_EINTERNAL, "%s: CUDA error %s (%s)", what, cudaGetErrorName(e), cudaGetErrorString(e));
}

template <class F>
dvsg_status guarded(F&& f) {
  try {
    f();
    return DVSG_OK;
  } catch (const Fail& e) {
    g_err = e.msg;
    return e.code;
  } catch (const std::bad_alloc&) {
    g_err = "out of host memory";
    return DVSG_EINTERNAL;
  } catch (const std::exception& e) {
    g_err = e.what();
    return DVSG_EINTERNAL;
  }
}

// Growable device array.
template <class T>
struct DevBuf {
  T* p = nullptr;
  size_t cap = 0;  // elements
  int device = 0;
  ~DevBuf() {
    if (p) cudaFree(p);
  }
  void reserve(size_t n, cudaStream_t s, bool keep = false, size_t keep_n = 0) {
    if (n <= cap) return;
    size_t nc = std::max(n, cap + cap / 2);
    T* np = nullptr;
    cuda_check(cudaMalloc(&np, nc * sizeof(T)), "cudaMalloc");
    if (keep && p && keep_n) {
      cuda_check(cudaMemcpyAsync(np, p, keep_n * sizeof(T), cudaMemcpyDeviceToDevice, s), "grow copy");
      cuda_check(cudaStreamSynchronize(s), "grow sync");
    }
    if (p) cudaFree(p);
    p = np;
    cap = nc;
  }
};

uint64_t env_u64(const char* name, uint64_t dflt) {
  const char* e = std::getenv(name);
  return e && *e ? std::strtoull(e, nullptr, 10) : dflt;
}

bool ids_increasing(const uint32_t* g, uint64_t n) {
  for (uint64_t i = 1; i < n; ++i)
    if (g[i] <= g[i - 1]) return false;
  return true;
}

bool finite_all(const float* x, uint64_t n) {
  for (uint64_t i = 0; i < n; ++i)
    if (!std::isfinite(x[i])) return false;
  return true;
}

// integer-valued with |x| < 2^24: every fp32 squared-L2 / dot sum the fast
// mode forms is then exact (at the dims the bench uses), i.e. equal to the
// reference's fp64-then-round arithmetic (distance.cpp:19-27)
bool integral_all(const float* x, uint64_t n) {
  for (uint64_t i = 0; i < n; ++i)
    if (!(x[i] == std::nearbyint(x[i]) && std::fabs(x[i]) < 16777216.f)) return false;
  return true;
}

// K6's fp32 tile distances equal the reference's fp64-then-rounded ones when
// every coordinate is an integer and every squared distance stays below 2^24
// (each partial sum an exact fp32 integer); otherwise the exact mode runs.
bool k6_fp32_exact(const float* x, uint64_t rows, int dim, float* lo_out = nullptr, float* hi_out = nullptr) {
  float lo = INFINITY, hi = -INFINITY;
  const uint64_t n = rows * (uint64_t)dim;
  for (uint64_t i = 0; i < n; ++i) {
    if (x[i] != std::nearbyint(x[i])) return false;
    lo = std::min(lo, x[i]);
    hi = std::max(hi, x[i]);
  }
  if (lo_out) *lo_out = lo;
  if (hi_out) *hi_out = hi;
  const double span = n ? (double)hi - (double)lo : 0.0;  // |x_i - y_i| <= span
  return span * span * (double)dim < 16777216.0;
}

// both operands of a brute-force search: the span covers the union of their ranges
bool k6_fp32_exact2(const float* a, uint64_t na, const float* b, uint64_t nb, int dim) {
  float la, ha, lb, hb;
  if (!k6_fp32_exact(a, na, dim, &la, &ha) || !k6_fp32_exact(b, nb, dim, &lb, &hb)) return false;
  const double span = (double)std::max(ha, hb) - (double)std::min(la, lb);
  return span * span * (double)dim < 16777216.0;
}

}  // namespace

struct dvsg_ctx {
  int device = 0;
  int num_sms = 148;
  size_t smem_optin = 227 * 1024;
  cudaStream_t stream = nullptr;  // compute
  cudaStream_t comm = nullptr;    // exchange
  // index
  int dim = 0, dpad = 0, dg = 0;
  uint64_t rows = 0;
  DevBuf<float> vec;
  DevBuf<uint32_t> adj, gids, entry;
  std::vector<dvsg::PartDesc> parts;
  std::vector<char> part_mono;     // global ids strictly increasing in local id (per part)
  bool all_integral = true;        // every resident row integer-valued below 2^24 (fp32 sums exact)
  struct Pending {                 // dvsg_partition_alloc_device .. commit
    bool active = false;
    uint32_t cluster = 0;
    uint64_t n = 0, r0 = 0;
  } pend;
  DevBuf<dvsg::PartDesc> d_parts;
  bool parts_dirty = true;
  // routing table
  int clusters = 0, ranks = 1;
  std::vector<float> cents;
  std::vector<uint32_t> placement;
  DevBuf<float> d_cents;
  DevBuf<double> d_cent_norms;
  DevBuf<int32_t> d_cluster_slot;
  uint32_t slot_map_n = 0;
  bool slot_dirty = true;
  DevBuf<uint64_t> d_locator;
  uint64_t locator_n = 0;
  bool locator_dirty = true;
  // scratch
  DevBuf<uint32_t> unit_q, unit_p, assign;
  DevBuf<uint32_t> u_ids, u_count;
  DevBuf<float> u_dists;
  DevBuf<uint64_t> u_visited;
  DevBuf<uint32_t> hash;
  DevBuf<unsigned long long> counter;  // [0] work counter, [1..3] stats
  DevBuf<uint64_t> assign_scratch;
  unsigned long long last_stats[3] = {0, 0, 0};
  bool stats_pending = false;
  DevBuf<int> err_flag;
  DevBuf<float> io_f, io_dists, io_vecs;
  DevBuf<uint32_t> io_u;
  DevBuf<uint64_t> io_u64;
  // node-sharded mode (shard_kernel.cu)
  struct Shard {
    bool active = false;     // ctx holds one rank's shard (multi-GPU)
    int nranks = 0, rank = 0;
    uint64_t n_total = 0, shard_rows = 0;
    int gpr_max = 0;
    uint32_t ring_cap = 0;
    size_t arena_bytes = 0;
    unsigned char* arena = nullptr;            // own comm arena (IPC-exported)
    std::vector<unsigned char*> peers;         // every rank's arena (own included)
    bool connected = false;
    size_t xg_off = 0, xg_bytes = 0;           // bulk-exchange region of the arena
  } sh;
  // bulk-synchronous exchange (xchg_kernel.cu): origin state + emulation arenas
  struct Xg {
    DevBuf<uint64_t> pool, visited;
    DevBuf<uint32_t> psize, expd, hash;
    DevBuf<uint2> meta;
    DevBuf<unsigned char> emu_arena;
    DevBuf<float> emu_q;
    DevBuf<dvsg::XgView> d_views;
    DevBuf<unsigned long long> counters;
    DevBuf<int> err;
    std::vector<size_t> nccl_send, nccl_recv;  // this phase's request counts per peer
    unsigned epoch[4] = {0, 0, 0, 0};
    bool issued = false;
  } xg;

  // cluster-sharded run_pipeline exchange (cluster_xchg.cu): this rank's arena
  struct Cl {
    bool active = false, connected = false, with_vectors = false, own_peers = false;
    int nranks = 0, rank = 0, k = 0, max_fanout = 0, dim = 0;
    uint64_t max_queries = 0, cap = 0, ucap = 0;
    size_t bytes = 0;
    size_t off_q = 0, off_meta = 0, off_ids = 0, off_dists = 0, off_count = 0, off_vis = 0, off_vec = 0;
    unsigned char* arena = nullptr;
    std::vector<unsigned char*> peers;
    unsigned epoch = 0;
    int parity = 0;
  } cl;
  DevBuf<dvsg::ClArena> cl_peers;
  DevBuf<uint32_t> cl_uq, cl_up, cl_ids, cl_count, cl_place;
  DevBuf<float> cl_dists;
  DevBuf<uint64_t> cl_vis;
  DevBuf<unsigned long long> cl_nunits;
  DevBuf<int> cl_err;

  // measured timeline of the last bulk-exchange search (timing on)
  std::vector<int> xg_tl;                      // 0: step kernel, 1: barrier / NCCL exchange
  std::vector<cudaEvent_t> xg_tl_ev;
  int shard_exchange = -1;                     // 0 bulk (default), 1 fused, 2 nccl; -1: env DVSG_SHARD_EXCHANGE
  // NCCL baseline of the bulk exchange (host-driven send/recv per phase)
  ncclComm_t nccl = nullptr;
  DevBuf<unsigned char> nccl_buf;
  DevBuf<unsigned char> emu_arena;             // emulation: all virtual ranks' arenas
  DevBuf<dvsg::ShardView> d_views;
  DevBuf<uint32_t> iota_q, zero_p;
  // locality ordering of units (anchors = evenly spaced resident rows)
  DevBuf<float> anchors;
  int n_anchors = 0;
  bool anchors_dirty = true;
  DevBuf<uint32_t> order_scratch, unit_order;
  uint64_t iota_n = 0;
  // timing
  bool timing = false;
  cudaEvent_t ev[8] = {};
  cudaEvent_t mb_ev[2 * 16] = {};  // microbatch pipeline (H2D done, compute done)
  // measured timeline of the last run_pipeline (timing on): base + per
  // microbatch {h2d start, h2d end, compute start, compute end, d2h start, d2h end}
  cudaEvent_t tl_ev[1 + 6 * 16] = {};
  int tl_mb = 0;
  float t_search = 0, t_assign = 0, t_combine = 0, t_total = 0;
  int timing_pending = 0;  // 1: search only, 2: pipeline
  std::atomic<uint64_t> launches{0};
  int assign_path = -1;  // K5 variant of the last context assign (launch_assign's *path)
  bool pipeline_pageable = false;  // last dvsg_run_pipeline saw pageable host buffers
  // U8 vector storage (dvsg_set_vector_storage): a byte copy of the resident
  // rows, valid while vec_gen (bumped on every change of the rows) matches
  DevBuf<uint8_t> vec8;
  uint64_t vec_gen = 0, u8_gen = ~0ull;
  bool want_u8 = false;
  int knn_exact = -1;          // last build_graph / brute_force_topk: 0 fp32 tiles, 1 exact mode
  uint64_t knn_fallbacks = 0;  // exact mode: rows the certificate sent to the fp64 scan
};

namespace {

// kernels one launch_assign issues on each path (warp / fp64 tiles / tensor cores)
uint64_t assign_launches(int path) { return path == 2 ? 7 : path == 1 ? 3 : 1; }

void set_device(dvsg_ctx* c) { cuda_check(cudaSetDevice(c->device), "cudaSetDevice"); }

// Synchronous-API copies and memsets run on the legacy default stream, which
// is not ordered with the context's non-blocking streams (and a pageable
// cudaMemcpy H2D may return before its DMA has landed): drain it before any
// kernel on c->stream reads what they wrote.
void legacy_fence() { cuda_check(cudaStreamSynchronize(cudaStreamLegacy), "legacy stream"); }

int32_t slot_of(const dvsg_ctx* c, uint32_t cluster) {
  for (size_t i = 0; i < c->parts.size(); ++i)
    if (c->parts[i].cluster == cluster) return (int32_t)i;
  return -1;
}

void sync_parts(dvsg_ctx* c) {
  if (!c->parts_dirty) return;
  c->d_parts.reserve(std::max<size_t>(c->parts.size(), 1), c->stream);
  if (!c->parts.empty())
    cuda_check(cudaMemcpyAsync(c->d_parts.p, c->parts.data(), c->parts.size() * sizeof(dvsg::PartDesc),
                               cudaMemcpyHostToDevice, c->stream), "upload parts");
  cuda_check(cudaStreamSynchronize(c->stream), "sync parts");
  c->parts_dirty = false;
}

void sync_slots(dvsg_ctx* c) {
  if (!c->slot_dirty) return;
  int n = c->clusters;
  for (auto& p : c->parts) n = std::max<int>(n, (int)p.cluster + 1);
  std::vector<int32_t> m((size_t)std::max(n, 1), -1);
  for (size_t i = 0; i < c->parts.size(); ++i) m[c->parts[i].cluster] = (int32_t)i;
  c->d_cluster_slot.reserve(m.size(), c->stream);
  cuda_check(cudaMemcpyAsync(c->d_cluster_slot.p, m.data(), m.size() * 4, cudaMemcpyHostToDevice, c->stream), "slots");
  c->slot_map_n = (uint32_t)m.size();
  cuda_check(cudaStreamSynchronize(c->stream), "sync slots");
  c->slot_dirty = false;
}

// compute_entry_order, graph_index.cpp:21-44: fp64 column sums, f32 mean,
// fp64 sequential squared_l2 to the mean rounded to f32, sort (dist, id).
void entry_order_host(const float* v, uint64_t n, int dim, uint32_t* out) {
  std::vector<double> sums((size_t)dim, 0.0);
  for (uint64_t i = 0; i < n; ++i) {
    const float* r = v + i * (uint64_t)dim;
    for (int j = 0; j < dim; ++j) sums[(size_t)j] += r[j];
  }
  std::vector<float> mean((size_t)dim);
  for (int j = 0; j < dim; ++j) mean[(size_t)j] = (float)(sums[(size_t)j] / (double)n);
  std::vector<uint64_t> key(n);
  auto body = [&](uint64_t b, uint64_t e) {
    for (uint64_t i = b; i < e; ++i) {
      const float* r = v + i * (uint64_t)dim;
      double acc = 0.0;
      for (int j = 0; j < dim; ++j) {
        const double d = (double)r[j] - (double)mean[(size_t)j];
        acc += d * d;
      }
      const float f = (float)acc;  // >= 0, so the raw bits order like the value
      uint32_t bits;
      std::memcpy(&bits, &f, 4);
      key[i] = ((uint64_t)bits << 32) | (uint32_t)i;
    }
  };
  const unsigned nt = std::min<unsigned>(std::max(1u, std::thread::hardware_concurrency()), 32u);
  if (n < 65536 || nt == 1) {
    body(0, n);
  } else {
    std::vector<std::thread> th;
    for (unsigned t = 0; t < nt; ++t) th.emplace_back(body, n * t / nt, n * (t + 1) / nt);
    for (auto& x : th) x.join();
  }
  std::sort(key.begin(), key.end());
  for (uint64_t i = 0; i < n; ++i) out[i] = (uint32_t)key[i];
}

void validate_params(const dvsg_search_params* p) {
  if (!p) fail(DVSG_EINVAL, "SearchParams: null");
  if (p->iterations < 1 || p->beam_width < 1 || p->k < 1 || p->entry_count < 1)
    fail(DVSG_EINVAL, "SearchParams: iterations, beam_width, k and entry_count must all be >= 1");
  if (p->metric != DVSG_METRIC_L2 && p->metric != DVSG_METRIC_IP) fail(DVSG_EINVAL, "SearchParams: unknown metric %d", p->metric);
  if (p->accum != DVSG_ACCUM_F64 && p->accum != DVSG_ACCUM_F32 && p->accum != DVSG_ACCUM_F32C)
    fail(DVSG_EINVAL, "SearchParams: unknown accum %d", p->accum);
}

// The fp32 fast mode (DVSG_ACCUM_F32) is exact only when every sum it forms
// is exact, i.e. on integer-valued data (checked at upload, all_integral).  On
// anything else it is upgraded to a mode that meets the parity bar:
// compensated f32 for inner product / wide rows (faster than f64 there), f64
// otherwise.  DVSG_ALLOW_F32_FLOAT=1 keeps plain f32 (measurements only).
dvsg_search_params effective_params(const dvsg_ctx* c, const dvsg_search_params* p) {
  dvsg_search_params e = *p;
  static const bool allow = env_u64("DVSG_ALLOW_F32_FLOAT", 0) != 0;
  // L2 -> f64 (exact by construction, finish_dist; with the wide-row K1 it is
  // also the faster mode at 768-d), inner product -> f32c (no reference to match)
  if (e.accum == DVSG_ACCUM_F32 && !c->all_integral && !allow)
    e.accum = e.metric == DVSG_METRIC_IP ? DVSG_ACCUM_F32C : DVSG_ACCUM_F64;
  return e;
}

uint64_t pow2_at_least(uint64_t x) {
  uint64_t p = 1;
  while (p < x) p <<= 1;
  return p;
}

// Shapes of a K1 launch for these params (cap, survivor buffer, hash size).
struct K1Shape {
  uint64_t cap, chp, hsize;
  bool hash_in_smem;
  size_t smem;
};

K1Shape k1_shape(dvsg_ctx* c, const dvsg_search_params* p, uint64_t nmax, bool allow_smem_hash) {
  K1Shape k{};
  k.cap = std::max<uint64_t>(4ull * (uint64_t)p->k, 2ull * (uint64_t)p->iterations * (uint64_t)p->beam_width);
  if (k.cap > (1ull << 20)) fail(DVSG_EINVAL, "beam_search: candidate pool capacity %llu exceeds the device limit", (unsigned long long)k.cap);
  // Exact pool truncation.  The frontier of iteration t is the first w
  // unexpanded entries, and at most t*w entries are expanded, so every pick
  // sits at a position < I*w; entries only ever move down.  Hence keeping
  // the first max(I*w, k) entries instead of cap = max(4k, 2*I*w)
  // (graph_index.cpp:127-129) picks the same frontiers, scores the same
  // vectors (same visited counter) and holds the same first k -- and when
  // global ids increase with local ids the final (dist, gid) order equals the
  // pool's (dist, local) order, so no tie beyond position k can enter the
  // top k either.  Halves the pool, the survivors to sort and the merges.
  static const bool trunc_env = env_u64("DVSG_POOL_TRUNC", 1) != 0;
  bool mono = trunc_env && !c->part_mono.empty();
  for (char m : c->part_mono) mono = mono && m;
  if (mono) k.cap = std::max<uint64_t>((uint64_t)p->k, (uint64_t)p->iterations * (uint64_t)p->beam_width);
  // visited never exceeds min(n_max, entries + I*w*dg)
  const uint64_t entries = std::min<uint64_t>((uint64_t)p->entry_count, nmax);
  const uint64_t bound = std::min<uint64_t>(nmax, entries + (uint64_t)p->iterations * (uint64_t)p->beam_width * (uint64_t)c->dg);
  k.hsize = std::max<uint64_t>(64, pow2_at_least(bound + 1));
  // linear probing near 100% load costs hundreds of probes per insert.  When
  // the partition size is the bound (a small partition can be explored
  // completely) keep the worst case at <= 3/4 load.  The I*w*dg bound is
  // never reached in practice (duplicate neighbours), and doubling those
  // tables would push the per-CTA regions out of L2.
  if (bound == nmax && 4 * (bound + 1) > 3 * k.hsize) k.hsize *= 2;
  k.chp = std::max<uint64_t>(pow2_at_least((uint64_t)dvsg::kChunk), pow2_at_least(k.cap));
  static const uint64_t hash_smem_max = [] {
    const char* e = std::getenv("DVSG_HASH_SMEM_MAX");
    // default: visited hash in global memory (L2-resident, one 4*hsize-byte
    // region per persistent CTA).  Measured faster than shared memory at
    // cfg1 because it frees 64 KB/CTA of smem for occupancy (profiles/).
    return e ? std::strtoull(e, nullptr, 10) : 0ull;
  }();
  k.hash_in_smem = allow_smem_hash && k.hsize <= hash_smem_max;
  k.smem = dvsg::search_smem_bytes((int)k.cap, (int)k.chp, p->beam_width, (int)k.hsize, k.hash_in_smem);
  if (k.hash_in_smem && k.smem > c->smem_optin) k.hash_in_smem = false;
  k.smem = dvsg::search_smem_bytes((int)k.cap, (int)k.chp, p->beam_width, (int)k.hsize, k.hash_in_smem);
  if (k.smem > c->smem_optin) fail(DVSG_EINVAL, "beam_search: pool (%llu) too large for shared memory", (unsigned long long)k.cap);
  return k;
}

dvsg::SearchArgs k1_args(dvsg_ctx* c, const dvsg_search_params* p, const K1Shape& k, const float* d_q,
                         uint64_t nq, int dim, const uint32_t* d_uq, const uint32_t* d_up,
                         uint64_t nunits, uint32_t* d_ids, float* d_dists, uint32_t* d_count,
                         uint64_t* d_visited) {
  dvsg::SearchArgs a{};
  a.vectors = c->vec.p;
  a.vectors8 = (c->want_u8 && c->u8_gen == c->vec_gen && !c->sh.active && c->dpad <= 256) ? c->vec8.p : nullptr;
  a.adjacency = c->adj.p;
  a.gids = c->gids.p;
  a.entry = c->entry.p;
  a.parts = c->d_parts.p;
  a.queries = d_q;
  a.nq = nq;
  a.unit_query = d_uq;
  a.unit_part = d_up;
  a.nunits = nunits;
  a.dim = dim;
  a.dpad = c->dpad;
  a.dg = c->dg;
  a.iters = p->iterations;
  a.beam = p->beam_width;
  a.k = p->k;
  a.entry_count = p->entry_count;
  a.cap = (int)k.cap;
  a.chp = (int)k.chp;
  a.hsize = (int)k.hsize;
  a.out_ids = d_ids;
  a.out_dists = d_dists;
  a.out_count = d_count;
  a.out_visited = d_visited;
  c->counter.reserve(16, c->stream);
  a.work_counter = c->counter.p;
  a.stats = c->counter.p + 1;
  cuda_check(cudaMemsetAsync(c->counter.p, 0, 16 * sizeof(unsigned long long), c->stream), "counter reset");
  c->stats_pending = true;
  return a;
}

// Core: K1 over a device unit list.  All pointers device.
void search_units(dvsg_ctx* c, const float* d_q, uint64_t nq, int dim, const uint32_t* d_uq,
                  const uint32_t* d_up, uint64_t nunits, const dvsg_search_params* p,
                  uint32_t* d_ids, float* d_dists, uint32_t* d_count, uint64_t* d_visited,
                  const unsigned long long* d_nunits = nullptr) {
  validate_params(p);
  const dvsg_search_params pe = effective_params(c, p);
  p = &pe;
  if (c->sh.active) fail(DVSG_EINVAL, "beam_search: this context holds one rank's shard; use dvsg_search_sharded_device");
  if (c->parts.empty()) fail(DVSG_EINVAL, "beam_search: empty graph");
  if (dim != c->dim) fail(DVSG_EINVAL, "beam_search: query dim %d != index dim %d", dim, c->dim);
  if (nunits == 0) return;
  if ((uint64_t)p->beam_width * (uint64_t)c->dg > (1ull << 24)) fail(DVSG_EINVAL, "beam_search: beam_width * out_degree above 2^24 candidates per iteration");
  sync_parts(c);
  uint64_t nmax = 0;
  for (auto& pd : c->parts) nmax = std::max<uint64_t>(nmax, pd.n);
  const K1Shape k = k1_shape(c, p, nmax, true);
  dvsg::SearchArgs a = k1_args(c, p, k, d_q, nq, dim, d_uq, d_up, nunits, d_ids, d_dists, d_count, d_visited);
  a.nunits_dev = d_nunits;  // unit count produced on the device (cluster exchange)
  // locality order: CTAs claim units grouped by the query's nearest anchor row,
  // so concurrent CTAs walk overlapping graph regions (L2 reuse).  Pure
  // scheduling: outputs are per unit, results are identical in any order.
  // measured at cfg1: K1 -1.8%, but the bucketing pass costs the same -> off by default
  static const bool locality = [] {
    const char* e = std::getenv("DVSG_LOCALITY");
    return e ? std::atoi(e) != 0 : false;
  }();
  if (locality && nunits >= 4096 && dim <= 256 && c->rows >= 1024) {
    if (c->anchors_dirty) {
      c->n_anchors = 256;
      c->anchors.reserve((size_t)c->n_anchors * c->dpad, c->stream);
      for (int i = 0; i < c->n_anchors; ++i) {
        const uint64_t row = c->rows * (uint64_t)i / (uint64_t)c->n_anchors;
        cuda_check(cudaMemcpyAsync(c->anchors.p + (size_t)i * c->dpad, c->vec.p + row * (uint64_t)c->dpad,
                                   (size_t)c->dpad * 4, cudaMemcpyDeviceToDevice, c->stream), "anchors");
      }
      c->anchors_dirty = false;
    }
    c->order_scratch.reserve(nunits + (uint64_t)c->n_anchors + 1, c->stream);
    c->unit_order.reserve(nunits, c->stream);
    cuda_check(dvsg::launch_locality_order(d_q, dim, d_uq, nunits, c->anchors.p, c->n_anchors, c->dpad,
                                           c->order_scratch.p, c->unit_order.p, c->stream), "locality order");
    c->launches += 3;
    a.unit_order = c->unit_order.p;
  }
  int max_grid = 0;
  if (!k.hash_in_smem) {
    // one L2-resident region per persistent CTA; optionally cap the grid so
    // the tables' total footprint stays within an L2 budget (large beams)
    max_grid = 8 * c->num_sms;
    static const uint64_t l2_budget = [] {
      const char* e = std::getenv("DVSG_HASH_L2_BUDGET_MB");
      return e ? std::strtoull(e, nullptr, 10) << 20 : 0ull;
    }();
    if (l2_budget) max_grid = (int)std::max<uint64_t>((uint64_t)c->num_sms, std::min<uint64_t>((uint64_t)max_grid, l2_budget / (4 * k.hsize)));
    // large beams: the worst-case tables (256 KB/CTA at w=256) stop fitting
    // in L2; start every unit in a half-size table and grow exactly on demand
    // (DVSG_HASH_SMALL_MIN: smallest full table that gets a small one; tests lower it)
    const uint64_t small_min = env_u64("DVSG_HASH_SMALL_MIN", 65536);
    a.hsmall = small_min && k.hsize >= small_min && k.hsize >= 128 ? (int)(k.hsize / 2) : 0;
    c->hash.reserve((uint64_t)max_grid * (k.hsize + (uint64_t)a.hsmall), c->stream);
    a.hash_global = c->hash.p;
  }
  if (c->timing) cudaEventRecord(c->ev[0], c->stream);
  int grid = 0;
  cuda_check(dvsg::launch_search(a, p->metric, p->accum, c->num_sms, max_grid, c->stream, &grid), "search kernel launch");
  if (c->timing) {
    cudaEventRecord(c->ev[1], c->stream);
    c->timing_pending = 1;
  }
  c->launches += 1;
}

// ---- node-sharded search --------------------------------------------------
constexpr size_t kArenaHeader = 256;  // work u64 @0, done @8, finished @12, ring_head @16, ring_tail @20

size_t shard_arena_bytes(int nranks, int gpr_max, uint32_t ring_cap, int dpad) {
  size_t b = kArenaHeader + (size_t)ring_cap * 4;
  b = (b + 255) & ~(size_t)255;
  b += (size_t)nranks * gpr_max * dvsg::shard_mail_stride(dpad);
  b = (b + 255) & ~(size_t)255;
  b += (size_t)gpr_max * nranks * dvsg::shard_reply_stride();
  return b;
}

dvsg::ShardView shard_view(unsigned char* arena, const float* vec, int nranks, int gpr_max,
                           uint32_t ring_cap, int dpad) {
  dvsg::ShardView v{};
  v.vec = vec;
  v.work = reinterpret_cast<unsigned long long*>(arena);
  v.done = reinterpret_cast<unsigned*>(arena + 8);
  v.finished = reinterpret_cast<unsigned*>(arena + 12);
  v.ring_head = reinterpret_cast<unsigned*>(arena + 16);
  v.ring_tail = reinterpret_cast<unsigned*>(arena + 20);
  v.ring = reinterpret_cast<uint32_t*>(arena + kArenaHeader);
  size_t off = (kArenaHeader + (size_t)ring_cap * 4 + 255) & ~(size_t)255;
  v.mail = arena + off;
  off += (size_t)nranks * gpr_max * dvsg::shard_mail_stride(dpad);
  off = (off + 255) & ~(size_t)255;
  v.reply = arena + off;
  return v;
}

const uint32_t* iota_units(dvsg_ctx* c, uint64_t n, const uint32_t** zero_parts) {
  if (c->iota_n < n) {
    std::vector<uint32_t> h(n);
    std::iota(h.begin(), h.end(), 0u);
    c->iota_q.reserve(n, c->stream);
    c->zero_p.reserve(n, c->stream);
    cuda_check(cudaMemcpyAsync(c->iota_q.p, h.data(), n * 4, cudaMemcpyHostToDevice, c->stream), "iota");
    cuda_check(cudaMemsetAsync(c->zero_p.p, 0, n * 4, c->stream), "zero");
    cuda_check(cudaStreamSynchronize(c->stream), "iota");
    c->iota_n = n;
  }
  *zero_parts = c->zero_p.p;
  return c->iota_q.p;
}

// Launch the sharded kernel.  emulate: all ranks in one launch on this device.
void search_sharded(dvsg_ctx* c, bool emulate, int nranks, const float* d_q, uint64_t nq, int dim,
                    const dvsg_search_params* p, uint32_t* d_ids, float* d_dists, uint32_t* d_count,
                    uint64_t* d_visited) {
  validate_params(p);
  const dvsg_search_params pe = effective_params(c, p);
  p = &pe;
  if (dim != c->dim) fail(DVSG_EINVAL, "beam_search: query dim %d != index dim %d", dim, c->dim);
  if (c->parts.size() != 1) fail(DVSG_EINVAL, "sharded search: the context must hold exactly one (whole-graph) partition");
  if (nranks < 1 || nranks > 8) fail(DVSG_EINVAL, "sharded search: nranks %d outside 1..8", nranks);
  if (c->dpad > 768) fail(DVSG_EINVAL, "sharded search: dim above 768 not supported");
  if (nq == 0) return;
  sync_parts(c);
  const uint64_t n = c->sh.active ? c->sh.n_total : c->parts[0].n;
  const K1Shape k = k1_shape(c, p, n, false);
  const uint32_t* zp = nullptr;
  const uint32_t* uq = iota_units(c, nq, &zp);
  dvsg::SearchArgs a = k1_args(c, p, k, d_q, nq, dim, uq, zp, nq, d_ids, d_dists, d_count, d_visited);
  const int per_sm = dvsg::search_sharded_blocks_per_sm(a, p->metric, p->accum);
  if (per_sm < 1) fail(DVSG_EINTERNAL, "sharded search: kernel does not fit on an SM");
  const int resident = per_sm * c->num_sms;
  const int gpr_max = 8 * c->num_sms;
  const uint32_t ring_cap = (uint32_t)pow2_at_least((uint64_t)nranks * gpr_max);
  dvsg::ShardArgs sh{};
  sh.nranks = nranks;
  sh.ring_mask = ring_cap - 1;
  sh.mail_stride = dvsg::shard_mail_stride(c->dpad);
  sh.reply_stride = dvsg::shard_reply_stride();
  std::vector<dvsg::ShardView> views((size_t)nranks);
  if (emulate) {
    sh.rank_self = -1;
    sh.gpr = resident / nranks;
    sh.shard_rows = (n + (uint64_t)nranks - 1) / (uint64_t)nranks;
    sh.units_per_rank = (nq + (uint64_t)nranks - 1) / (uint64_t)nranks;
    const size_t ab = shard_arena_bytes(nranks, sh.gpr, ring_cap, c->dpad);
    c->emu_arena.reserve(ab * (size_t)nranks, c->stream);
    cuda_check(cudaMemsetAsync(c->emu_arena.p, 0, ab * (size_t)nranks, c->stream), "arena reset");
    for (int r = 0; r < nranks; ++r)
      views[(size_t)r] = shard_view(c->emu_arena.p + ab * (size_t)r,
                                    c->vec.p + (uint64_t)r * sh.shard_rows * (uint64_t)c->dpad,
                                    nranks, sh.gpr, ring_cap, c->dpad);
  } else {
    if (!c->sh.active || !c->sh.connected) fail(DVSG_EINVAL, "sharded search: call dvsg_shard_init and dvsg_shard_connect first");
    if (nranks != c->sh.nranks) fail(DVSG_EINVAL, "sharded search: nranks %d != %d", nranks, c->sh.nranks);
    sh.rank_self = c->sh.rank;
    sh.gpr = std::min(resident, c->sh.gpr_max);
    sh.shard_rows = c->sh.shard_rows;
    sh.units_per_rank = nq;
    for (int r = 0; r < nranks; ++r)
      views[(size_t)r] = shard_view(c->sh.peers[(size_t)r], r == c->sh.rank ? c->vec.p : nullptr,
                                    nranks, c->sh.gpr_max, c->sh.ring_cap, c->dpad);
    sh.ring_mask = c->sh.ring_cap - 1;
  }
  c->d_views.reserve((size_t)nranks, c->stream);
  cuda_check(cudaMemcpyAsync(c->d_views.p, views.data(), views.size() * sizeof(dvsg::ShardView), cudaMemcpyHostToDevice, c->stream), "views");
  sh.views = c->d_views.p;
  // dedicated server CTAs per rank (drain the doorbell ring promptly)
  static const int servers_env = [] {
    const char* e = std::getenv("DVSG_SHARD_SERVERS");
    return e ? std::atoi(e) : -1;
  }();
  int servers = servers_env >= 0 ? servers_env : 0;  // measured: dedicated servers do not pay
  if (servers >= sh.gpr) servers = sh.gpr - 1;
  sh.origin_ctas = sh.gpr - servers;
  const int grid_total = emulate ? sh.gpr * nranks : sh.gpr;
  c->hash.reserve((uint64_t)grid_total * k.hsize, c->stream);
  a.hash_global = c->hash.p;
  if (c->timing) cudaEventRecord(c->ev[0], c->stream);
  int grid = 0, gpr = 0;
  cuda_check(dvsg::launch_search_sharded(a, sh, p->metric, p->accum, c->num_sms, c->stream, &grid, &gpr), "sharded search launch");
  if (c->timing) {
    cudaEventRecord(c->ev[1], c->stream);
    c->timing_pending = 1;
  }
  c->launches += 1;
}

// ---- NCCL, loaded at run time (the process's libnccl.so.2, e.g. torch's) ---
struct NcclApi {
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  ncclResult_t (*send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*group_start)() = nullptr;
  ncclResult_t (*group_end)() = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
};

const NcclApi& nccl_api() {
  static NcclApi api = [] {
    NcclApi a;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW);
    if (!h) return a;
    a.get_unique_id = reinterpret_cast<decltype(a.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
    a.comm_init_rank = reinterpret_cast<decltype(a.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
    a.comm_destroy = reinterpret_cast<decltype(a.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
    a.send = reinterpret_cast<decltype(a.send)>(dlsym(h, "ncclSend"));
    a.recv = reinterpret_cast<decltype(a.recv)>(dlsym(h, "ncclRecv"));
    a.group_start = reinterpret_cast<decltype(a.group_start)>(dlsym(h, "ncclGroupStart"));
    a.group_end = reinterpret_cast<decltype(a.group_end)>(dlsym(h, "ncclGroupEnd"));
    a.error_string = reinterpret_cast<decltype(a.error_string)>(dlsym(h, "ncclGetErrorString"));
    return a;
  }();
  if (!api.send || !api.comm_init_rank) fail(DVSG_EINTERNAL, "NCCL exchange: libnccl.so.2 not loadable");
  return api;
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess)
    fail(DVSG_EINTERNAL, "%s: NCCL error %d (%s)", what, (int)r,
         nccl_api().error_string ? nccl_api().error_string(r) : "?");
}

// ---- node-sharded search, bulk-synchronous exchange (xchg_kernel.cu) -------
constexpr size_t kXgHeader = 256;  // cursor [2][8] u32 @0, flags [8] u32 @64
// Two query waves half a phase apart: every xg_step launch carries exactly one
// expand op and one score op, so more lanes would need several of each per
// launch (a third lane's op would collide with lane 0's parity) -- capped.
constexpr int kXgLanes = 2;
constexpr size_t kXgTlMax = 1024;  // timeline intervals kept per search

size_t xg_region_bytes(int nranks, uint64_t wcap, uint64_t maxraw, int dpad) {
  size_t b = kXgHeader;
  b += (size_t)nranks * wcap * (uint64_t)dpad * 4;
  b = (b + 255) & ~(size_t)255;
  b += 2 * (size_t)nranks * wcap * maxraw * 8;
  return b;
}

dvsg::XgView xg_view(unsigned char* region, const float* vec, uint64_t lo, int nranks, uint64_t wcap,
                     uint64_t maxraw, int dpad) {
  dvsg::XgView v{};
  v.vec = vec;
  v.lo = lo;
  v.cursor = reinterpret_cast<unsigned*>(region);
  v.flags = reinterpret_cast<unsigned*>(region + 64);
  size_t off = kXgHeader;
  v.qall = reinterpret_cast<float*>(region + off);
  off += (size_t)nranks * wcap * (uint64_t)dpad * 4;
  off = (off + 255) & ~(size_t)255;
  v.inbox = reinterpret_cast<uint64_t*>(region + off);
  off += (size_t)nranks * wcap * maxraw * 8;
  v.reply = reinterpret_cast<uint64_t*>(region + off);
  return v;
}

void xg_check(dvsg_ctx* c) {
  if (!c->xg.issued) return;
  int err = 0;
  cuda_check(cudaStreamSynchronize(c->stream), "sharded err");
  cuda_check(cudaMemcpy(&err, c->xg.err.p, sizeof err, cudaMemcpyDeviceToHost), "sharded err");
  c->xg.issued = false;
  if (err & 8) fail(DVSG_EINTERNAL, "sharded search: a peer rank did not reach the exchange barrier (20 s)");
}

// emulate: all R ranks on this device (queries split evenly, rank r origin of
// [r*upr, (r+1)*upr)); else this rank's nq queries, every rank concurrently.
// The rank's queries are processed in waves; L lanes (streams, each with its
// own comm region, state slice and barrier epoch) run waves concurrently,
// offset by half a phase so one lane's xg_expand (latency bound) overlaps the
// other lane's xg_score (HBM bound).
void search_xchg(dvsg_ctx* c, bool emulate, int nranks, const float* d_q, uint64_t nq, int dim,
                 const dvsg_search_params* p, uint32_t* d_ids, float* d_dists, uint32_t* d_count,
                 uint64_t* d_visited) {
  validate_params(p);
  const dvsg_search_params pe = effective_params(c, p);
  p = &pe;
  if (dim != c->dim) fail(DVSG_EINVAL, "beam_search: query dim %d != index dim %d", dim, c->dim);
  if (c->parts.size() != 1) fail(DVSG_EINVAL, "sharded search: the context must hold exactly one (whole-graph) partition");
  if (nranks < 1 || nranks > dvsg::kXgMaxRanks) fail(DVSG_EINVAL, "sharded search: nranks %d outside 1..8", nranks);
  if (c->dpad > 768) fail(DVSG_EINVAL, "sharded search: dim above 768 not supported");
  if (nq == 0) return;
  sync_parts(c);
  const int R = nranks;
  const uint64_t n = c->sh.active ? c->sh.n_total : c->parts[0].n;
  const K1Shape k = k1_shape(c, p, n, false);
  const uint64_t maxraw = std::max<uint64_t>(std::min<uint64_t>((uint64_t)p->entry_count, n),
                                             (uint64_t)p->beam_width * (uint64_t)c->dg);
  const size_t smem = dvsg::xg_expand_smem_bytes((int)k.cap, (int)k.chp, p->beam_width, (int)maxraw);
  if (smem > c->smem_optin) fail(DVSG_EINVAL, "sharded search: beam x degree / entry_count too large (%llu new candidates per phase)", (unsigned long long)maxraw);
  const uint64_t S = emulate ? (n + (uint64_t)R - 1) / (uint64_t)R : c->sh.shard_rows;
  const uint64_t upr = emulate ? (nq + (uint64_t)R - 1) / (uint64_t)R : nq;
  const int rank_n = emulate ? R : 1;
  const int me = emulate ? 0 : c->sh.rank;
  auto rank_count = [&](int r) -> uint64_t {
    if (!emulate) return nq;
    const uint64_t lo = std::min<uint64_t>(nq, (uint64_t)r * upr);
    return std::min<uint64_t>(nq, lo + upr) - lo;
  };
  if (!emulate) {
    if (!c->sh.connected) fail(DVSG_EINVAL, "sharded search: call dvsg_shard_init and dvsg_shard_connect first");
    if (nranks != c->sh.nranks) fail(DVSG_EINVAL, "sharded search: nranks %d != %d", nranks, c->sh.nranks);
  }
  // NCCL baseline: same kernels over local send/receive slabs, exchanged by
  // host-driven ncclSend/ncclRecv after each half-phase (counts via the host)
  const bool use_nccl = !emulate && c->shard_exchange == 2;
  if (use_nccl && !c->nccl) fail(DVSG_EINVAL, "NCCL exchange: call dvsg_nccl_connect first");
  // lanes and wave size (comm region + origin state budgets, split per lane)
  const int L = use_nccl ? 1 : (int)std::max<uint64_t>(1, std::min<uint64_t>(kXgLanes, env_u64("DVSG_XG_LANES", 2)));
  const uint64_t comm_q = (uint64_t)R * ((uint64_t)c->dpad * 4 + 16 * maxraw);
  const uint64_t state_q = k.cap * 8 + k.hsize * 4 + 16 + 8 * (uint64_t)R;
  const size_t lane_bytes = emulate ? 0 : ((c->sh.xg_bytes / (size_t)L) & ~(size_t)4095);
  uint64_t wmax = upr;
  if (emulate) {
    wmax = std::min<uint64_t>(wmax, std::max<uint64_t>(1, (env_u64("DVSG_XG_EMU_MB", 2048) << 20) / ((uint64_t)L * R * comm_q)));
  } else if (use_nccl) {
    const uint64_t per_q = (uint64_t)R * R * maxraw * 16 + (uint64_t)R * c->dpad * 4;
    wmax = std::min<uint64_t>(wmax, std::max<uint64_t>(1, (env_u64("DVSG_XG_NCCL_MB", 16384) << 20) / per_q));
  } else {
    const uint64_t room = lane_bytes > kXgHeader + 512 ? (lane_bytes - kXgHeader - 512) / comm_q : 0;
    if (room < 1) fail(DVSG_EINVAL, "sharded search: comm arena too small for one query");
    wmax = std::min<uint64_t>(wmax, room);
  }
  wmax = std::min<uint64_t>(wmax, std::max<uint64_t>(1, (env_u64("DVSG_XG_STATE_MB", 16384) << 20) / ((uint64_t)L * rank_n * state_q)));
  const uint64_t wlim = env_u64("DVSG_XG_WAVE", 0);
  if (wlim) wmax = std::min<uint64_t>(wmax, wlim);
  wmax = std::min<uint64_t>(wmax, 1ull << 30);
  // equal waves, a multiple of L of them (every lane busy)
  uint64_t nwaves = (upr + wmax - 1) / wmax;
  if (L > 1) nwaves = (nwaves + L - 1) / (uint64_t)L * (uint64_t)L;
  const uint64_t wcap = (upr + nwaves - 1) / nwaves;
  const uint64_t rstride = wcap * maxraw;

  auto& x = c->xg;
  const uint64_t st_n = (uint64_t)L * rank_n * wcap;
  x.pool.reserve(st_n * k.cap, c->stream);
  x.visited.reserve(st_n, c->stream);
  x.psize.reserve(st_n, c->stream);
  x.expd.reserve(st_n, c->stream);
  x.hash.reserve(st_n * k.hsize, c->stream);
  x.meta.reserve(st_n * (uint64_t)R, c->stream);
  x.err.reserve(1, c->stream);
  cuda_check(cudaMemsetAsync(x.err.p, 0, sizeof(int), c->stream), "err reset");

  // views: [lane][rank]
  std::vector<dvsg::XgView> views((size_t)L * R);
  if (emulate) {
    const size_t rb = xg_region_bytes(R, wcap, maxraw, c->dpad);
    x.emu_arena.reserve(rb * (size_t)R * L, c->stream);
    x.emu_q.reserve((size_t)L * R * wcap * (uint64_t)c->dpad, c->stream);
    for (int l = 0; l < L; ++l)
      for (int r = 0; r < R; ++r) {
        unsigned char* reg = x.emu_arena.p + rb * ((size_t)l * R + r);
        cuda_check(cudaMemsetAsync(reg, 0, kXgHeader, c->stream), "xg header reset");
        auto& v = views[(size_t)l * R + r];
        v = xg_view(reg, c->vec.p + (uint64_t)r * S * (uint64_t)c->dpad, (uint64_t)r * S, R, wcap, maxraw, c->dpad);
        v.qall = x.emu_q.p + (size_t)l * R * wcap * (uint64_t)c->dpad;  // one copy stands in for every owner's
      }
  } else {
    for (int l = 0; l < L && !use_nccl; ++l)
      for (int r = 0; r < R; ++r)
        views[(size_t)l * R + r] = xg_view(c->sh.peers[(size_t)r] + c->sh.xg_off + (size_t)l * lane_bytes,
                                           r == me ? c->vec.p : nullptr, (uint64_t)r * S, R, wcap, maxraw, c->dpad);
  }
  // NCCL layout (all local): slab (o*R + s) of the request / reply arrays is
  // "from origin s to owner o" / "from owner s to origin o"; with
  // views[o].inbox = req + o*R*rstride the kernels' indexing (origin writes
  // views[o].inbox + me*rstride, owner reads views[me].inbox + o*rstride)
  // lands in send slab (o*R+me) and receive slab (me*R+o).  Cursors:
  // views[o].cursor = cur + o*2R, so origin counters and received counts
  // (written by ncclRecv) never collide.
  uint64_t* n_req = nullptr;
  uint64_t* n_rep = nullptr;
  unsigned* n_cur = nullptr;
  float* n_q = nullptr;
  if (use_nccl) {
    const size_t slabs = (size_t)R * R * rstride * 8;
    const size_t qb = (size_t)R * wcap * (uint64_t)c->dpad * 4;
    const size_t cb = (size_t)R * 2 * R * 4;
    c->nccl_buf.reserve(2 * slabs + qb + cb + 1024, c->stream);
    n_req = reinterpret_cast<uint64_t*>(c->nccl_buf.p);
    n_rep = reinterpret_cast<uint64_t*>(c->nccl_buf.p + slabs);
    n_q = reinterpret_cast<float*>(c->nccl_buf.p + 2 * slabs);
    n_cur = reinterpret_cast<unsigned*>(c->nccl_buf.p + 2 * slabs + qb);
    for (int o = 0; o < R; ++o) {
      auto& v = views[(size_t)o];
      v.vec = o == me ? c->vec.p : nullptr;
      v.lo = (uint64_t)o * S;
      v.cursor = n_cur + (size_t)o * 2 * R;
      v.flags = nullptr;
      v.qall = n_q;
      v.inbox = n_req + (size_t)o * R * rstride;
      v.reply = n_rep + (size_t)o * R * rstride;
    }
  }
  x.d_views.reserve(views.size(), c->stream);
  cuda_check(cudaMemcpyAsync(x.d_views.p, views.data(), views.size() * sizeof(dvsg::XgView), cudaMemcpyHostToDevice, c->stream), "views");

  dvsg::SearchArgs ka = k1_args(c, p, k, d_q, nq, dim, nullptr, nullptr, nq, d_ids, d_dists, d_count, d_visited);
  dvsg::XgArgs base{};
  base.nranks = R;
  base.rank_lo = me;
  base.rank_n = rank_n;
  base.wcap = (uint32_t)wcap;
  base.maxraw = (uint32_t)maxraw;
  base.rstride = rstride;
  base.shard_rows = (uint32_t)S;
  base.adjacency = c->adj.p;
  base.gids = c->gids.p;
  base.entry = c->entry.p;
  base.n = (uint32_t)n;
  base.dim = dim;
  base.dpad = c->dpad;
  base.dg = c->dg;
  base.iters = p->iterations;
  base.beam = p->beam_width;
  base.k = p->k;
  base.entry_count = p->entry_count;
  base.cap = (int)k.cap;
  base.chp = (int)k.chp;
  base.hsize = (int)k.hsize;
  base.out_stride = emulate ? upr : 0;
  base.stats = ka.stats;
  base.err = x.err.p;
  dvsg::XgArgs la[kXgLanes];
  for (int l = 0; l < L; ++l) {
    la[l] = base;
    la[l].views = x.d_views.p + (size_t)l * R;
    const uint64_t so = (uint64_t)l * rank_n * wcap;
    la[l].pool = x.pool.p + so * k.cap;
    la[l].psize = x.psize.p + so;
    la[l].visited = x.visited.p + so;
    la[l].expd = x.expd.p + so;
    la[l].hash = x.hash.p + so * k.hsize;
    la[l].meta = x.meta.p + so * (uint64_t)R;
  }
  // measured timeline of this search (timing on): an event pair around every
  // step kernel (compute lane) and every barrier / NCCL exchange (comm lane)
  c->xg_tl.clear();
  auto tl_mark = [&](int kind) -> int {
    if (!c->timing || c->xg_tl.size() >= kXgTlMax) return -1;
    const int i = (int)c->xg_tl.size();
    c->xg_tl.push_back(kind);
    cuda_check(cudaEventRecord(c->xg_tl_ev[2 * i], c->stream), "event");
    return i;
  };
  auto tl_end = [&](int i) {
    if (i >= 0) cuda_check(cudaEventRecord(c->xg_tl_ev[2 * i + 1], c->stream), "event");
  };
  auto barrier = [&](int l) {
    if (emulate || use_nccl) return;  // stream order (+ NCCL) is the barrier
    x.epoch[l] += 1;
    const int m = tl_mark(1);
    cuda_check(dvsg::launch_xg_barrier(la[l].views, R, me, x.epoch[l], x.err.p, c->stream), "xg barrier");
    tl_end(m);
    c->launches += 1;
  };
  // Per lane the ops are E0 S0 E1 S1 ... E_I S_I E_{I+1} (E_{I+1}: finalize).
  // Launch t runs lane 0's op t and lane 1's op t-1: one expand and one score
  // per launch, co-resident in one xg_step grid.
  const int nops = 2 * (p->iterations + 1) + 1;
  const int nlaunch = nops + L - 1;
  x.counters.reserve(2 * (size_t)nlaunch, c->stream);
  if (c->timing) cudaEventRecord(c->ev[0], c->stream);
  for (uint64_t w0 = 0; w0 < nwaves; w0 += (uint64_t)L) {
    for (int l = 0; l < L; ++l) {
      auto& a = la[l];
      const uint64_t off = (w0 + (uint64_t)l) * wcap;
      for (int rr = 0; rr < rank_n; ++rr) {
        const uint64_t cnt = rank_count(me + rr);
        a.wave_n[rr] = (uint32_t)(cnt > off ? std::min<uint64_t>(wcap, cnt - off) : 0);
      }
      // each origin's wave queries into every owner's qall[origin] (padded rows)
      for (int rr = 0; rr < rank_n; ++rr) {
        if (!a.wave_n[rr]) continue;
        const int o = me + rr;
        const float* src = d_q + ((emulate ? (uint64_t)o * upr : 0) + off) * (uint64_t)dim;
        for (int r = 0; r < (emulate || use_nccl ? 1 : R); ++r) {
          float* dst = views[(size_t)l * R + r].qall + (uint64_t)o * wcap * (uint64_t)c->dpad;
          cuda_check(cudaMemcpy2DAsync(dst, (size_t)c->dpad * 4, src, (size_t)dim * 4, (size_t)dim * 4,
                                       a.wave_n[rr], cudaMemcpyDefault, c->stream), "push queries");
        }
      }
      a.out_ids = d_ids + off * (uint64_t)p->k;
      a.out_dists = d_dists + off * (uint64_t)p->k;
      a.out_count = d_count + off;
      a.out_visited = d_visited + off;
      if (use_nccl) {  // all-gather of the wave's queries (every rank has the same wave size)
        const NcclApi& nc = nccl_api();
        const size_t qn = (size_t)a.wave_n[0] * (uint64_t)c->dpad;
        nccl_check(nc.group_start(), "ncclGroupStart");
        for (int o = 0; o < R; ++o) {
          if (o == me) continue;
          nccl_check(nc.send(n_q + (size_t)me * wcap * c->dpad, qn, ncclFloat32, o, c->nccl, c->stream), "ncclSend");
          nccl_check(nc.recv(n_q + (size_t)o * wcap * c->dpad, qn, ncclFloat32, o, c->nccl, c->stream), "ncclRecv");
        }
        nccl_check(nc.group_end(), "ncclGroupEnd");
      }
      barrier(l);  // every owner holds this wave's queries
    }
    cuda_check(cudaMemsetAsync(x.counters.p, 0, 2 * (size_t)nlaunch * sizeof(unsigned long long), c->stream), "counters");
    for (int t = 0; t < nlaunch; ++t) {
      int le = -1, ls = -1;  // lanes doing an expand / a score op in this launch
      for (int l = 0; l < L; ++l) {
        const int op = t - l;
        if (op < 0 || op >= nops) continue;
        if (op & 1) {
          ls = l;
          la[l].phase = op >> 1;
        } else {
          le = l;
          la[l].phase = op >> 1;
        }
      }
      const dvsg::XgArgs& ea = la[std::max(0, le >= 0 ? le : ls)];
      const dvsg::XgArgs& sa = la[std::max(0, ls >= 0 ? ls : le)];
      if (use_nccl && le >= 0)
        cuda_check(cudaMemsetAsync(n_cur, 0, (size_t)R * 2 * R * 4, c->stream), "cursor reset");
      const int mk = tl_mark(0);
      cuda_check(dvsg::launch_xg_step(ea, sa, le >= 0, ls >= 0, x.counters.p + 2 * t, p->metric, p->accum,
                                      c->num_sms, c->stream), "xg step");
      tl_end(mk);
      c->launches += 1;
      if (ls >= 0 && !use_nccl)  // that phase's inbox cursors are free again (next used two barriers later)
        for (int rr = 0; rr < rank_n; ++rr)
          cuda_check(cudaMemsetAsync(views[(size_t)ls * R + me + rr].cursor + (la[ls].phase & 1) * R, 0,
                                     (size_t)R * 4, c->stream), "cursor reset");
      // requests (after an expand) / replies (after a score) delivered
      if (le >= 0 && la[le].phase <= p->iterations) barrier(le);
      if (ls >= 0) barrier(ls);
      const int mx = use_nccl ? tl_mark(1) : -1;
      if (use_nccl && le >= 0 && la[le].phase <= p->iterations) {
        // requests: counts through the host (NCCL needs host-side sizes), then data
        const NcclApi& nc = nccl_api();
        const int slot = la[le].phase & 1;
        std::vector<unsigned> cur((size_t)R * 2 * R);
        cuda_check(cudaMemcpyAsync(cur.data(), n_cur, cur.size() * 4, cudaMemcpyDeviceToHost, c->stream), "counts");
        cuda_check(cudaStreamSynchronize(c->stream), "counts");
        nccl_check(nc.group_start(), "ncclGroupStart");
        for (int o = 0; o < R; ++o) {
          if (o == me) continue;
          nccl_check(nc.send(n_cur + (size_t)o * 2 * R + slot * R + me, 1, ncclUint32, o, c->nccl, c->stream), "ncclSend");
          nccl_check(nc.recv(n_cur + (size_t)me * 2 * R + slot * R + o, 1, ncclUint32, o, c->nccl, c->stream), "ncclRecv");
        }
        nccl_check(nc.group_end(), "ncclGroupEnd");
        cuda_check(cudaMemcpyAsync(cur.data(), n_cur, cur.size() * 4, cudaMemcpyDeviceToHost, c->stream), "counts");
        cuda_check(cudaStreamSynchronize(c->stream), "counts");
        x.nccl_send.assign((size_t)R, 0);
        x.nccl_recv.assign((size_t)R, 0);
        for (int o = 0; o < R; ++o) {
          x.nccl_send[(size_t)o] = cur[(size_t)o * 2 * R + slot * R + me];
          x.nccl_recv[(size_t)o] = cur[(size_t)me * 2 * R + slot * R + o];
        }
        nccl_check(nc.group_start(), "ncclGroupStart");
        for (int o = 0; o < R; ++o) {
          if (o == me) continue;
          if (x.nccl_send[(size_t)o])
            nccl_check(nc.send(n_req + ((size_t)o * R + me) * rstride, x.nccl_send[(size_t)o], ncclUint64, o, c->nccl, c->stream), "ncclSend");
          if (x.nccl_recv[(size_t)o])
            nccl_check(nc.recv(n_req + ((size_t)me * R + o) * rstride, x.nccl_recv[(size_t)o], ncclUint64, o, c->nccl, c->stream), "ncclRecv");
        }
        nccl_check(nc.group_end(), "ncclGroupEnd");
      }
      if (use_nccl && ls >= 0) {  // replies: the same counts, reversed
        const NcclApi& nc = nccl_api();
        nccl_check(nc.group_start(), "ncclGroupStart");
        for (int o = 0; o < R; ++o) {
          if (o == me) continue;
          if (x.nccl_recv[(size_t)o])
            nccl_check(nc.send(n_rep + ((size_t)o * R + me) * rstride, x.nccl_recv[(size_t)o], ncclUint64, o, c->nccl, c->stream), "ncclSend");
          if (x.nccl_send[(size_t)o])
            nccl_check(nc.recv(n_rep + ((size_t)me * R + o) * rstride, x.nccl_send[(size_t)o], ncclUint64, o, c->nccl, c->stream), "ncclRecv");
        }
        nccl_check(nc.group_end(), "ncclGroupEnd");
      }
      tl_end(mx);
    }
  }
  if (c->timing) {
    cudaEventRecord(c->ev[1], c->stream);
    c->timing_pending = 1;
  }
  x.issued = true;
}

bool use_bulk_exchange(dvsg_ctx* c) {
  if (c->shard_exchange < 0) {
    const char* e = std::getenv("DVSG_SHARD_EXCHANGE");
    c->shard_exchange = (e && std::strcmp(e, "fused") == 0) ? 1 : (e && std::strcmp(e, "nccl") == 0) ? 2 : 0;
  }
  return c->shard_exchange != 1;
}

template <class T>
T* stage(DevBuf<T>& b, const T* host, size_t n, cudaStream_t s) {
  b.reserve(std::max<size_t>(n, 1), s);
  if (n) cuda_check(cudaMemcpyAsync(b.p, host, n * sizeof(T), cudaMemcpyHostToDevice, s), "H2D");
  return b.p;
}

void build_locator(dvsg_ctx* c) {
  if (!c->locator_dirty) return;
  // gid -> device row, over the resident partitions (simulator.cpp:275-288)
  std::vector<uint32_t> g(c->rows);
  cuda_check(cudaStreamSynchronize(c->stream), "sync");
  if (c->rows) cuda_check(cudaMemcpy(g.data(), c->gids.p, c->rows * 4, cudaMemcpyDeviceToHost), "gids D2H");
  uint64_t total = 0;
  for (auto x : g) total = std::max<uint64_t>(total, (uint64_t)x + 1);
  std::vector<uint64_t> loc(std::max<uint64_t>(total, 1), ~0ull);
  for (uint64_t r = 0; r < c->rows; ++r) {
    if (loc[g[r]] != ~0ull) fail(DVSG_EINTERNAL, "run_pipeline: partitions do not form a dense id cover");
    loc[g[r]] = r;
  }
  c->d_locator.reserve(loc.size(), c->stream);
  cuda_check(cudaMemcpyAsync(c->d_locator.p, loc.data(), loc.size() * 8, cudaMemcpyHostToDevice, c->stream), "locator");
  cuda_check(cudaStreamSynchronize(c->stream), "locator sync");
  c->locator_n = total;
  c->locator_dirty = false;
}

void pipeline_device(dvsg_ctx* c, const float* d_q, uint64_t nq, int dim, const dvsg_search_params* p,
                     int fanout, uint32_t* d_ids, float* d_dists, uint32_t* d_count, float* d_vecs,
                     uint64_t* d_visited, bool reset_err = true) {
  validate_params(p);
  if (c->clusters < 1) fail(DVSG_EINVAL, "BuiltIndex: index is not built");
  if (dim != c->dim) fail(DVSG_EINVAL, "run_pipeline: query dim %d != index dim %d", dim, c->dim);
  if (fanout < 1 || fanout > c->clusters)
    fail(DVSG_EINVAL, "run_pipeline: fanout %d out of range for %d clusters", fanout, c->clusters);
  if (fanout > 32) fail(DVSG_EINVAL, "run_pipeline: fanout %d above the device merge width 32", fanout);
  if (nq == 0) return;
  sync_slots(c);
  const uint64_t nu = nq * (uint64_t)fanout;
  c->assign.reserve(nu, c->stream);
  c->unit_q.reserve(nu, c->stream);
  c->unit_p.reserve(nu, c->stream);
  c->u_ids.reserve(nu * (uint64_t)p->k, c->stream);
  c->u_dists.reserve(nu * (uint64_t)p->k, c->stream);
  c->u_count.reserve(nu, c->stream);
  uint64_t* vis = d_visited;
  if (!vis) {
    c->u_visited.reserve(nu, c->stream);
    vis = c->u_visited.p;
  }
  c->err_flag.reserve(1, c->stream);
  if (reset_err) cuda_check(cudaMemsetAsync(c->err_flag.p, 0, sizeof(int), c->stream), "err reset");
  if (c->timing) cudaEventRecord(c->ev[2], c->stream);
  c->assign_scratch.reserve(dvsg::assign_scratch_words(nq, dim, c->clusters, fanout), c->stream);
  cuda_check(dvsg::launch_assign(d_q, nq, dim, c->d_cents.p, c->d_cent_norms.p, c->clusters, fanout, c->assign.p, c->assign_scratch.p, c->stream, &c->assign_path), "assign");
  cuda_check(dvsg::launch_route(c->assign.p, nq, fanout, c->d_cluster_slot.p, c->slot_map_n, c->unit_q.p, c->unit_p.p, c->err_flag.p, c->stream), "route");
  if (c->timing) cudaEventRecord(c->ev[3], c->stream);
  c->launches += assign_launches(c->assign_path) + 1;
  search_units(c, d_q, nq, dim, c->unit_q.p, c->unit_p.p, nu, p, c->u_ids.p, c->u_dists.p, c->u_count.p, vis);
  if (c->timing) cudaEventRecord(c->ev[4], c->stream);
  cuda_check(dvsg::launch_combine(nq, fanout, c->u_ids.p, c->u_dists.p, c->u_count.p, p->k, p->k, d_ids, d_dists, d_count, c->err_flag.p, c->stream), "combine");
  c->launches += 1;
  if (d_vecs) {
    build_locator(c);
    cuda_check(dvsg::launch_gather_vectors(d_ids, d_count, nq, p->k, c->d_locator.p, c->vec.p, c->dim, c->dpad, d_vecs, c->stream), "gather vectors");
    c->launches += 1;
  }
  if (c->timing) {
    cudaEventRecord(c->ev[5], c->stream);
    c->timing_pending = 2;
  }
}

void check_err_flag(dvsg_ctx* c, const char* what) {
  int flag = 0;
  cuda_check(cudaMemcpyAsync(&flag, c->err_flag.p, sizeof(int), cudaMemcpyDeviceToHost, c->stream), "err flag");
  cuda_check(cudaStreamSynchronize(c->stream), "sync");
  if (flag) fail(DVSG_EINTERNAL, "%s", what);
}

void read_timings(dvsg_ctx* c, bool pipeline) {
  if (!c->timing) return;
  c->timing_pending = 0;
  cudaEventSynchronize(c->ev[pipeline ? 5 : 1]);
  cudaEventElapsedTime(&c->t_search, c->ev[0], c->ev[1]);
  if (pipeline) {
    cudaEventElapsedTime(&c->t_assign, c->ev[2], c->ev[3]);
    cudaEventElapsedTime(&c->t_combine, c->ev[4], c->ev[5]);
    cudaEventElapsedTime(&c->t_total, c->ev[2], c->ev[5]);
  } else {
    c->t_assign = c->t_combine = 0;
    c->t_total = c->t_search;
  }
}

// ---- FNSY v1 (index_file.cpp:16-25) -------------------------------------
struct Section {
  uint32_t id;
  uint64_t offset;  // payload offset in the file
  uint64_t length;
};

struct FileReader {
  FILE* f = nullptr;
  uint64_t pos = 0;
  explicit FileReader(const char* path) {
    f = std::fopen(path, "rb");
    if (!f) fail(DVSG_EFORMAT, "cannot open %s for reading (byte offset 0)", path);
  }
  ~FileReader() {
    if (f) std::fclose(f);
  }
  void seek(uint64_t off) {
    if (fseeko(f, (off_t)off, SEEK_SET) != 0) fail(DVSG_EFORMAT, "index file: seek failed (byte offset %llu)", (unsigned long long)off);
    pos = off;
  }
  bool read(void* dst, size_t n) {
    const size_t got = std::fread(dst, 1, n, f);
    pos += got;
    return got == n;
  }
};

struct SecCursor {
  FileReader& r;
  const char* name;
  uint64_t begin, end;
  SecCursor(FileReader& rr, const Section& s, const char* nm) : r(rr), name(nm), begin(s.offset), end(s.offset + s.length) { r.seek(begin); }
  uint64_t offset() const { return r.pos; }
  void need(uint64_t bytes) {
    if (r.pos + bytes > end) fail(DVSG_EFORMAT, "index file: truncated %s section (byte offset %llu)", name, (unsigned long long)r.pos);
  }
  uint32_t u32() {
    need(4);
    unsigned char b[4];
    if (!r.read(b, 4)) fail(DVSG_EFORMAT, "index file: truncated %s section (byte offset %llu)", name, (unsigned long long)r.pos);
    return (uint32_t)b[0] | ((uint32_t)b[1] << 8) | ((uint32_t)b[2] << 16) | ((uint32_t)b[3] << 24);
  }
  void bulk(void* dst, uint64_t bytes) {  // little-endian host assumed (x86-64)
    need(bytes);
    if (!r.read(dst, bytes)) fail(DVSG_EFORMAT, "index file: truncated %s section (byte offset %llu)", name, (unsigned long long)r.pos);
  }
  void skip(uint64_t bytes) {
    need(bytes);
    r.seek(r.pos + bytes);
  }
  void expect_consumed() {
    if (r.pos != end) fail(DVSG_EFORMAT, "index file: trailing bytes in %s section (byte offset %llu)", name, (unsigned long long)r.pos);
  }
};

void put_u32(std::vector<unsigned char>& b, uint32_t v) {
  for (int i = 0; i < 4; ++i) b.push_back((unsigned char)((v >> (8 * i)) & 0xff));
}

}  // namespace

// ===========================================================================
// C-ABI
// ===========================================================================
extern "C" {

const char* dvsg_last_error(void) { return g_err.c_str(); }
const char* dvsg_version(void) { return "dvsg 0.1 (sm_100a)"; }

dvsg_status dvsg_create(int device, dvsg_ctx** out) {
  return guarded([&] {
    if (!out) fail(DVSG_EINVAL, "dvsg_create: null out");
    int n = 0;
    cuda_check(cudaGetDeviceCount(&n), "cudaGetDeviceCount");
    if (device < 0 || device >= n) fail(DVSG_EINVAL, "dvsg_create: device %d out of range (%d devices)", device, n);
    auto c = std::make_unique<dvsg_ctx>();
    c->device = device;
    cuda_check(cudaSetDevice(device), "cudaSetDevice");
    cudaDeviceProp prop{};
    cuda_check(cudaGetDeviceProperties(&prop, device), "props");
    if (prop.major < 10) fail(DVSG_EINTERNAL, "dvsg: device %d is sm_%d%d; this library is built for sm_100a only", device, prop.major, prop.minor);
    c->num_sms = prop.multiProcessorCount;
    c->smem_optin = prop.sharedMemPerBlockOptin;
    cuda_check(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking), "stream");
    cuda_check(cudaStreamCreateWithFlags(&c->comm, cudaStreamNonBlocking), "stream");

    for (auto& e : c->ev) cuda_check(cudaEventCreate(&e), "event");
    for (auto& e : c->mb_ev) cuda_check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
    for (auto& e : c->tl_ev) cuda_check(cudaEventCreate(&e), "event");
    c->xg_tl_ev.resize(2 * kXgTlMax);
    for (auto& e : c->xg_tl_ev) cuda_check(cudaEventCreate(&e), "event");
    *out = c.release();
  });
}

dvsg_status dvsg_destroy(dvsg_ctx* c) {
  return guarded([&] {
    if (!c) return;
    cudaSetDevice(c->device);
    cudaStreamSynchronize(c->stream);
    for (size_t r = 0; r < c->sh.peers.size(); ++r)
      if ((int)r != c->sh.rank && c->sh.peers[r]) cudaIpcCloseMemHandle(c->sh.peers[r]);
    if (c->sh.arena) cudaFree(c->sh.arena);
    for (size_t r = 0; r < c->cl.peers.size(); ++r)
      if ((int)r != c->cl.rank && c->cl.peers[r] && !c->cl.own_peers) cudaIpcCloseMemHandle(c->cl.peers[r]);
    if (c->cl.arena) cudaFree(c->cl.arena);
    if (c->nccl) nccl_api().comm_destroy(c->nccl);
    for (auto& e : c->ev) cudaEventDestroy(e);
    for (auto& e : c->mb_ev) cudaEventDestroy(e);
    for (auto& e : c->tl_ev) cudaEventDestroy(e);
    for (auto& e : c->xg_tl_ev) cudaEventDestroy(e);
    cudaStreamDestroy(c->stream);
    cudaStreamDestroy(c->comm);

    delete c;
  });
}

void* dvsg_stream(dvsg_ctx* c) { return c ? (void*)c->stream : nullptr; }

dvsg_status dvsg_synchronize(dvsg_ctx* c) {
  return guarded([&] {
    set_device(c);
    cuda_check(cudaStreamSynchronize(c->stream), "synchronize");
    xg_check(c);
  });
}

dvsg_status dvsg_index_reset(dvsg_ctx* c) {
  return guarded([&] {
    set_device(c);
    cuda_check(cudaStreamSynchronize(c->stream), "sync");
    c->parts.clear();
    c->part_mono.clear();
    c->all_integral = true;
    c->pend = dvsg_ctx::Pending{};
    c->rows = 0;
    c->vec_gen += 1;
    c->dim = c->dpad = c->dg = 0;
    c->clusters = 0;
    c->sh.active = false;
    c->sh.connected = false;
    c->cents.clear();
    c->placement.clear();
    c->parts_dirty = c->slot_dirty = c->locator_dirty = true;
  });
}

dvsg_status dvsg_set_centroids(dvsg_ctx* c, const float* centroids, int clusters, int dim,
                               const uint32_t* cluster_to_rank, int ranks) {
  return guarded([&] {
    set_device(c);
    if (clusters < 1 || dim < 1 || !centroids) fail(DVSG_EINVAL, "assign_top_c: empty centroids");
    if (c->dim && dim != c->dim) fail(DVSG_EINVAL, "set_centroids: dim %d != index dim %d", dim, c->dim);
    if (ranks < 1) fail(DVSG_EINVAL, "ClusterTopology: ranks must be >= 1");
    if (!finite_all(centroids, (uint64_t)clusters * (uint64_t)dim)) fail(DVSG_EINVAL, "Dataset: non-finite centroid element");
    c->clusters = clusters;
    c->ranks = ranks;
    c->cents.assign(centroids, centroids + (size_t)clusters * dim);
    c->placement.resize((size_t)clusters);
    for (int i = 0; i < clusters; ++i) {
      const uint32_t r = cluster_to_rank ? cluster_to_rank[i] : (uint32_t)(i % ranks);  // router.cpp:38-41
      if ((int)r >= ranks) fail(DVSG_EINVAL, "placement rank %u out of range", r);
      c->placement[(size_t)i] = r;
    }
    std::vector<double> norms((size_t)clusters);
    for (int j = 0; j < clusters; ++j) {  // refresh_center_norms, kmeans.cpp:34-40
      double acc = 0.0;
      for (int i = 0; i < dim; ++i) acc += (double)centroids[(size_t)j * dim + i] * (double)centroids[(size_t)j * dim + i];
      norms[(size_t)j] = acc;
    }
    if (!c->dim) c->dim = dim;
    c->d_cents.reserve((size_t)clusters * dim, c->stream);
    c->d_cent_norms.reserve((size_t)clusters, c->stream);
    cuda_check(cudaMemcpyAsync(c->d_cents.p, centroids, (size_t)clusters * dim * 4, cudaMemcpyHostToDevice, c->stream), "cents");
    cuda_check(cudaMemcpyAsync(c->d_cent_norms.p, norms.data(), (size_t)clusters * 8, cudaMemcpyHostToDevice, c->stream), "norms");
    cuda_check(cudaStreamSynchronize(c->stream), "sync");
    c->slot_dirty = true;
  });
}

dvsg_status dvsg_load_partition(dvsg_ctx* c, uint32_t cluster, uint64_t n, int dim, int out_degree,
                                const float* vectors, const uint32_t* adjacency,
                                const uint32_t* global_ids, const uint32_t* entry_order) {
  return guarded([&] {
    set_device(c);
    if (n == 0) fail(DVSG_EINVAL, "BuiltIndex: empty partition");
    if (n >= (1ull << 31)) fail(DVSG_EINVAL, "load_partition: %llu rows exceed the 2^31 local-id limit", (unsigned long long)n);
    if (dim < 1) fail(DVSG_EINVAL, "Dataset: dim must be positive, got %d", dim);
    if (out_degree < 1) fail(DVSG_EINVAL, "build_graph: out_degree must be >= 1");
    if (!vectors || !adjacency) fail(DVSG_EINVAL, "load_partition: null vectors/adjacency");
    if (c->dim && c->dim != dim) fail(DVSG_EINVAL, "BuiltIndex: graph dim mismatch (%d vs %d)", dim, c->dim);
    if (c->dg && c->dg != out_degree) fail(DVSG_EINVAL, "BuiltIndex: graph out-degree mismatch (%d vs %d)", out_degree, c->dg);
    if (slot_of(c, cluster) >= 0) fail(DVSG_EINVAL, "load_partition: cluster %u already resident", cluster);
    if (!finite_all(vectors, n * (uint64_t)dim)) fail(DVSG_EINVAL, "Dataset: non-finite element in partition %u", cluster);
    for (uint64_t i = 0; i < n * (uint64_t)out_degree; ++i)
      if (adjacency[i] >= n) fail(DVSG_EFORMAT, "index file: neighbor id out of range in cluster %u", cluster);
    std::vector<uint32_t> eo;
    if (!entry_order) {
      eo.resize(n);
      entry_order_host(vectors, n, dim, eo.data());
      entry_order = eo.data();
    }
    std::vector<uint32_t> iota;
    if (!global_ids) {
      iota.resize(n);
      std::iota(iota.begin(), iota.end(), 0u);
      global_ids = iota.data();
    }
    c->dim = dim;
    c->dpad = (dim + 3) & ~3;
    c->dg = out_degree;
    const uint64_t r0 = c->rows, r1 = r0 + n;
    c->vec.reserve(r1 * (uint64_t)c->dpad, c->stream, true, r0 * (uint64_t)c->dpad);
    c->adj.reserve(r1 * (uint64_t)c->dg, c->stream, true, r0 * (uint64_t)c->dg);
    c->gids.reserve(r1, c->stream, true, r0);
    c->entry.reserve(r1, c->stream, true, r0);
    if (c->dpad == dim) {
      cuda_check(cudaMemcpy(c->vec.p + r0 * c->dpad, vectors, n * (uint64_t)dim * 4, cudaMemcpyHostToDevice), "vectors H2D");
    } else {
      cuda_check(cudaMemcpy2D(c->vec.p + r0 * c->dpad, (size_t)c->dpad * 4, vectors, (size_t)dim * 4, (size_t)dim * 4, n, cudaMemcpyHostToDevice), "vectors H2D");
      cuda_check(cudaMemset2D(reinterpret_cast<char*>(c->vec.p + r0 * c->dpad) + (size_t)dim * 4, (size_t)c->dpad * 4, 0, (size_t)(c->dpad - dim) * 4, n), "pad");
    }
    cuda_check(cudaMemcpy(c->adj.p + r0 * c->dg, adjacency, n * (uint64_t)c->dg * 4, cudaMemcpyHostToDevice), "adjacency H2D");
    cuda_check(cudaMemcpy(c->gids.p + r0, global_ids, n * 4, cudaMemcpyHostToDevice), "gids H2D");
    cuda_check(cudaMemcpy(c->entry.p + r0, entry_order, n * 4, cudaMemcpyHostToDevice), "entry H2D");
    legacy_fence();
    c->parts.push_back(dvsg::PartDesc{r0, (uint32_t)n, cluster});
    c->part_mono.push_back(ids_increasing(global_ids, n));
    c->all_integral = c->all_integral && integral_all(vectors, n * (uint64_t)dim);
    c->rows = r1;
    c->vec_gen += 1;
    c->parts_dirty = c->slot_dirty = c->locator_dirty = c->anchors_dirty = true;
  });
}

dvsg_status dvsg_index_info(dvsg_ctx* c, int* nparts, int* dim, int* out_degree, int* clusters,
                            uint32_t* cluster_ids, uint64_t* sizes) {
  return guarded([&] {
    if (nparts) *nparts = (int)c->parts.size();
    if (dim) *dim = c->dim;
    if (out_degree) *out_degree = c->dg;
    if (clusters) *clusters = c->clusters;
    for (size_t i = 0; i < c->parts.size(); ++i) {
      if (cluster_ids) cluster_ids[i] = c->parts[i].cluster;
      if (sizes) sizes[i] = c->parts[i].n;
    }
  });
}

dvsg_status dvsg_get_entry_order(dvsg_ctx* c, uint32_t cluster, uint32_t* out) {
  return guarded([&] {
    set_device(c);
    const int32_t s = slot_of(c, cluster);
    if (s < 0) fail(DVSG_EINVAL, "cluster %u not resident", cluster);
    const auto& pd = c->parts[(size_t)s];
    cuda_check(cudaStreamSynchronize(c->stream), "sync");
    cuda_check(cudaMemcpy(out, c->entry.p + pd.row_off, (size_t)pd.n * 4, cudaMemcpyDeviceToHost), "entry D2H");
  });
}

dvsg_status dvsg_compute_entry_order(const float* vectors, uint64_t n, int dim, uint32_t* out) {
  return guarded([&] {
    if (n == 0 || dim < 1) fail(DVSG_EINVAL, "compute_entry_order: empty partition");
    entry_order_host(vectors, n, dim, out);
  });
}

dvsg_status dvsg_beam_search(dvsg_ctx* c, uint32_t cluster, const float* queries, uint64_t nq, int dim,
                             const dvsg_search_params* p, uint32_t* out_ids, float* out_dists,
                             uint32_t* out_count, uint64_t* out_visited) {
  return guarded([&] {
    set_device(c);
    validate_params(p);
    const int32_t slot = slot_of(c, cluster);
    if (slot < 0) fail(DVSG_EINVAL, "beam_search: empty graph (cluster %u not resident)", cluster);
    if (dim != c->dim) fail(DVSG_EINVAL, "beam_search: query dim %d != index dim %d", dim, c->dim);
    if (nq == 0) return;
    if (!finite_all(queries, nq * (uint64_t)dim)) fail(DVSG_EINVAL, "Dataset: non-finite query element");
    const float* d_q = stage(c->io_f, queries, nq * (uint64_t)dim, c->stream);
    std::vector<uint32_t> uq(nq), up(nq, (uint32_t)slot);
    std::iota(uq.begin(), uq.end(), 0u);
    stage(c->unit_q, uq.data(), nq, c->stream);
    stage(c->unit_p, up.data(), nq, c->stream);
    const uint64_t k = (uint64_t)p->k;
    c->u_ids.reserve(nq * k, c->stream);
    c->u_dists.reserve(nq * k, c->stream);
    c->u_count.reserve(nq, c->stream);
    c->u_visited.reserve(nq, c->stream);
    search_units(c, d_q, nq, dim, c->unit_q.p, c->unit_p.p, nq, p, c->u_ids.p, c->u_dists.p, c->u_count.p, c->u_visited.p);
    cuda_check(cudaMemcpyAsync(out_ids, c->u_ids.p, nq * k * 4, cudaMemcpyDeviceToHost, c->stream), "D2H");
    cuda_check(cudaMemcpyAsync(out_dists, c->u_dists.p, nq * k * 4, cudaMemcpyDeviceToHost, c->stream), "D2H");
    cuda_check(cudaMemcpyAsync(out_count, c->u_count.p, nq * 4, cudaMemcpyDeviceToHost, c->stream), "D2H");
    cuda_check(cudaMemcpyAsync(out_visited, c->u_visited.p, nq * 8, cudaMemcpyDeviceToHost, c->stream), "D2H");
    cuda_check(cudaStreamSynchronize(c->stream), "beam_search");
    read_timings(c, false);
  });
}

dvsg_status dvsg_search_units_device(dvsg_ctx* c, const float* d_queries, uint64_t nq, int dim,
                                     const uint32_t* d_unit_query, const uint32_t* d_unit_cluster,
                                     uint64_t nunits, const dvsg_search_params* p, uint32_t* d_out_ids,
                                     float* d_out_dists, uint32_t* d_out_count, uint64_t* d_out_visited) {
  return guarded([&] {
    set_device(c);
    // unit_cluster holds cluster ids: translate to resident slots on device
    sync_slots(c);
    c->unit_p.reserve(std::max<uint64_t>(nunits, 1), c->stream);
    c->unit_q.reserve(std::max<uint64_t>(nunits, 1), c->stream);
    c->err_flag.reserve(1, c->stream);
    cuda_check(cudaMemsetAsync(c->err_flag.p, 0, sizeof(int), c->stream), "err reset");
    // route_kernel with fanout 1 maps cluster -> slot and writes unit_query = u;
    // the caller's unit_query is then used directly.
    cuda_check(dvsg::launch_route(d_unit_cluster, nunits, 1, c->d_cluster_slot.p, c->slot_map_n, c->unit_q.p, c->unit_p.p, c->err_flag.p, c->stream), "route");
    c->launches += 1;
    // a unit naming an unknown or non-resident cluster is the caller's error:
    // report it before launching the search (as the host-buffer entry points do)
    int flag = 0;
    cuda_check(cudaMemcpyAsync(&flag, c->err_flag.p, sizeof(int), cudaMemcpyDeviceToHost, c->stream), "err flag");
    cuda_check(cudaStreamSynchronize(c->stream), "sync");
    if (flag) fail(DVSG_EINVAL, "search_units: a unit names a cluster that is not resident on this context");
    search_units(c, d_queries, nq, dim, d_unit_query, c->unit_p.p, nunits, p, d_out_ids, d_out_dists, d_out_count, d_out_visited);
  });
}

dvsg_status dvsg_beam_search_sharded_emulated(dvsg_ctx* c, int nranks, const float* queries, uint64_t nq,
                                              int dim, const dvsg_search_params* p, uint32_t* out_ids,
                                              float* out_dists, uint32_t* out_count, uint64_t* out_visited) {
  return guarded([&] {
    set_device(c);
    validate_params(p);
    if (c->sh.active) fail(DVSG_EINVAL, "emulated sharded search needs the whole graph resident");
    if (dim != c->dim) fail(DVSG_EINVAL, "beam_search: query dim %d != index dim %d", dim, c->dim);
    if (nq == 0) return;
    if (!finite_all(queries, nq * (uint64_t)dim)) fail(DVSG_EINVAL, "Dataset: non-finite query element");
    const float* d_q = stage(c->io_f, queries, nq * (uint64_t)dim, c->stream);
    const uint64_t k = (uint64_t)p->k;
    c->u_ids.reserve(nq * k, c->stream);
    c->u_dists.reserve(nq * k, c->stream);
    c->u_count.reserve(nq, c->stream);
    c->u_visited.reserve(nq, c->stream);
    // diagnostic path: poison the outputs so a skipped query cannot pass as an
    // earlier search's result left in the shared staging buffers
    cuda_check(cudaMemsetAsync(c->u_ids.p, 0xFF, nq * k * 4, c->stream), "poison");
    cuda_check(cudaMemsetAsync(c->u_count.p, 0xFF, nq * 4, c->stream), "poison");
    cuda_check(cudaMemsetAsync(c->u_visited.p, 0xFF, nq * 8, c->stream), "poison");
    if (use_bulk_exchange(c)) search_xchg(c, true, nranks, d_q, nq, dim, p, c->u_ids.p, c->u_dists.p, c->u_count.p, c->u_visited.p);
    else search_sharded(c, true, nranks, d_q, nq, dim, p, c->u_ids.p, c->u_dists.p, c->u_count.p, c->u_visited.p);
    cuda_check(cudaMemcpyAsync(out_ids, c->u_ids.p, nq * k * 4, cudaMemcpyDeviceToHost, c->stream), "D2H");
    cuda_check(cudaMemcpyAsync(out_dists, c->u_dists.p, nq * k * 4, cudaMemcpyDeviceToHost, c->stream), "D2H");
    cuda_check(cudaMemcpyAsync(out_count, c->u_count.p, nq * 4, cudaMemcpyDeviceToHost, c->stream), "D2H");
    cuda_check(cudaMemcpyAsync(out_visited, c->u_visited.p, nq * 8, cudaMemcpyDeviceToHost, c->stream), "D2H");
    cuda_check(cudaStreamSynchronize(c->stream), "sharded search");
    xg_check(c);
    read_timings(c, false);
  });
}

namespace {
void shard_arena_setup(dvsg_ctx* c, int nranks, int rank, uint64_t n_total);
}

dvsg_status dvsg_shard_init(dvsg_ctx* c, int nranks, int rank, uint64_t n_total, int dim, int out_degree,
                            const float* shard_vectors, const uint32_t* adjacency,
                            const uint32_t* global_ids, const uint32_t* entry_order) {
  return guarded([&] {
    set_device(c);
    if (nranks < 1 || nranks > 8 || rank < 0 || rank >= nranks) fail(DVSG_EINVAL, "shard_init: rank %d of %d", rank, nranks);
    if (n_total == 0 || n_total >= (1ull << 31)) fail(DVSG_EINVAL, "shard_init: n %llu outside 1..2^31", (unsigned long long)n_total);
    if (dim < 1 || dim > 768) fail(DVSG_EINVAL, "shard_init: dim %d outside 1..768", dim);
    if (out_degree < 1) fail(DVSG_EINVAL, "build_graph: out_degree must be >= 1");
    if (!shard_vectors || !adjacency || !entry_order) fail(DVSG_EINVAL, "shard_init: null input");
    const uint64_t S = (n_total + (uint64_t)nranks - 1) / (uint64_t)nranks;
    const uint64_t lo = std::min<uint64_t>(n_total, S * (uint64_t)rank);
    const uint64_t hi = std::min<uint64_t>(n_total, lo + S);
    for (uint64_t i = 0; i < n_total * (uint64_t)out_degree; ++i)
      if (adjacency[i] >= n_total) fail(DVSG_EFORMAT, "index file: neighbor id out of range");
    cuda_check(cudaStreamSynchronize(c->stream), "sync");
    c->parts.clear();
    c->part_mono.clear();
    c->dim = dim;
    c->dpad = (dim + 3) & ~3;
    c->dg = out_degree;
    c->rows = n_total;
    c->vec_gen += 1;
    // own shard rows only (at least one row so the buffer exists)
    const uint64_t rows = std::max<uint64_t>(hi - lo, 1);
    c->vec.reserve(rows * (uint64_t)c->dpad, c->stream);
    cuda_check(cudaMemset(c->vec.p, 0, rows * (uint64_t)c->dpad * 4), "memset");
    if (hi > lo)
      cuda_check(cudaMemcpy2D(c->vec.p, (size_t)c->dpad * 4, shard_vectors, (size_t)dim * 4, (size_t)dim * 4, hi - lo, cudaMemcpyHostToDevice), "shard H2D");
    c->adj.reserve(n_total * (uint64_t)out_degree, c->stream);
    c->gids.reserve(n_total, c->stream);
    c->entry.reserve(n_total, c->stream);
    cuda_check(cudaMemcpy(c->adj.p, adjacency, n_total * (uint64_t)out_degree * 4, cudaMemcpyHostToDevice), "adjacency H2D");
    if (global_ids) {
      cuda_check(cudaMemcpy(c->gids.p, global_ids, n_total * 4, cudaMemcpyHostToDevice), "gids H2D");
    } else {
      std::vector<uint32_t> io(n_total);
      std::iota(io.begin(), io.end(), 0u);
      cuda_check(cudaMemcpy(c->gids.p, io.data(), n_total * 4, cudaMemcpyHostToDevice), "gids H2D");
    }
    cuda_check(cudaMemcpy(c->entry.p, entry_order, n_total * 4, cudaMemcpyHostToDevice), "entry H2D");
    legacy_fence();
    c->parts.push_back(dvsg::PartDesc{0, (uint32_t)n_total, 0});
    c->part_mono.push_back(global_ids ? ids_increasing(global_ids, n_total) : 1);
    c->all_integral = integral_all(shard_vectors, (hi - lo) * (uint64_t)dim);
    c->parts_dirty = c->slot_dirty = c->locator_dirty = true;
    shard_arena_setup(c, nranks, rank, n_total);
  });
}

dvsg_status dvsg_shard_init_resident(dvsg_ctx* c, int nranks, int rank) {
  return guarded([&] {
    set_device(c);
    if (nranks < 1 || nranks > 8 || rank < 0 || rank >= nranks) fail(DVSG_EINVAL, "shard_init: rank %d of %d", rank, nranks);
    if (c->sh.active) fail(DVSG_EINVAL, "shard_init_resident: already sharded");
    if (c->parts.size() != 1 || c->parts[0].row_off != 0) fail(DVSG_EINVAL, "shard_init_resident: needs exactly one resident partition");
    if (c->dim > 768) fail(DVSG_EINVAL, "shard_init: dim %d outside 1..768", c->dim);
    const uint64_t n_total = c->parts[0].n;
    const uint64_t S = (n_total + (uint64_t)nranks - 1) / (uint64_t)nranks;
    const uint64_t lo = std::min<uint64_t>(n_total, S * (uint64_t)rank);
    const uint64_t hi = std::min<uint64_t>(n_total, lo + S);
    cuda_check(cudaStreamSynchronize(c->stream), "sync");
    // keep only this rank's rows of the vectors; adjacency, global ids and
    // entry order stay whole (replicated)
    const uint64_t rows = std::max<uint64_t>(hi - lo, 1);
    DevBuf<float> own;
    own.reserve(rows * (uint64_t)c->dpad, c->stream);
    cuda_check(cudaStreamSynchronize(c->stream), "sync");
    cuda_check(cudaMemset(own.p, 0, rows * (uint64_t)c->dpad * 4), "memset");
    if (hi > lo)
      cuda_check(cudaMemcpy(own.p, c->vec.p + lo * c->dpad, (hi - lo) * (uint64_t)c->dpad * 4, cudaMemcpyDeviceToDevice), "shard rows");
    legacy_fence();
    std::swap(c->vec.p, own.p);
    std::swap(c->vec.cap, own.cap);
    c->parts[0].cluster = 0;
    c->rows = n_total;
    c->vec_gen += 1;
    c->parts_dirty = c->slot_dirty = c->locator_dirty = true;
    shard_arena_setup(c, nranks, rank, n_total);
  });
}

namespace {
void shard_arena_setup(dvsg_ctx* c, int nranks, int rank, uint64_t n_total) {
  const uint64_t S = (n_total + (uint64_t)nranks - 1) / (uint64_t)nranks;
  auto& sh = c->sh;
  if (sh.arena) cudaFree(sh.arena);
  sh = dvsg_ctx::Shard{};
  sh.active = true;
  sh.nranks = nranks;
  sh.rank = rank;
  sh.n_total = n_total;
  sh.shard_rows = S;
  sh.gpr_max = 8 * c->num_sms;
  sh.ring_cap = (uint32_t)pow2_at_least((uint64_t)nranks * sh.gpr_max);
  sh.arena_bytes = shard_arena_bytes(nranks, sh.gpr_max, sh.ring_cap, c->dpad);
  // + the bulk-exchange region (queries, inboxes, replies of one wave)
  sh.xg_off = (sh.arena_bytes + 4095) & ~(size_t)4095;
  sh.xg_bytes = (size_t)env_u64("DVSG_XG_ARENA_MB", 16384) << 20;
  sh.arena_bytes = sh.xg_off + sh.xg_bytes;
  cuda_check(cudaMalloc(&sh.arena, sh.arena_bytes), "arena");
  cuda_check(cudaMemset(sh.arena, 0, sh.xg_off + kXgHeader), "arena reset");
  legacy_fence();
  for (auto& e : c->xg.epoch) e = 0;
}
}  // namespace

dvsg_status dvsg_shard_export(dvsg_ctx* c, void* handle_out) {
  return guarded([&] {
    set_device(c);
    if (!c->sh.active) fail(DVSG_EINVAL, "shard_export: call dvsg_shard_init first");
    cudaIpcMemHandle_t h;
    cuda_check(cudaIpcGetMemHandle(&h, c->sh.arena), "cudaIpcGetMemHandle");
    std::memcpy(handle_out, &h, sizeof h);
  });
}

dvsg_status dvsg_shard_connect(dvsg_ctx* c, const void* handles) {
  return guarded([&] {
    set_device(c);
    auto& sh = c->sh;
    if (!sh.active) fail(DVSG_EINVAL, "shard_connect: call dvsg_shard_init first");
    sh.peers.assign((size_t)sh.nranks, nullptr);
    for (int r = 0; r < sh.nranks; ++r) {
      if (r == sh.rank) {
        sh.peers[(size_t)r] = sh.arena;
        continue;
      }
      cudaIpcMemHandle_t h;
      std::memcpy(&h, static_cast<const char*>(handles) + (size_t)r * sizeof h, sizeof h);
      void* ptr = nullptr;
      cuda_check(cudaIpcOpenMemHandle(&ptr, h, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
      sh.peers[(size_t)r] = static_cast<unsigned char*>(ptr);
    }
    sh.connected = true;
  });
}

dvsg_status dvsg_shard_prepare(dvsg_ctx* c) {
  return guarded([&] {
    set_device(c);
    if (!c->sh.active) fail(DVSG_EINVAL, "shard_prepare: call dvsg_shard_init first");
    cuda_check(cudaMemsetAsync(c->sh.arena, 0, c->sh.xg_off + kXgHeader, c->stream), "arena reset");
    cuda_check(cudaStreamSynchronize(c->stream), "arena reset");
    for (auto& e : c->xg.epoch) e = 0;
  });
}

dvsg_status dvsg_search_sharded_device(dvsg_ctx* c, const float* d_queries, uint64_t nq, int dim,
                                       const dvsg_search_params* p, uint32_t* d_out_ids,
                                       float* d_out_dists, uint32_t* d_out_count, uint64_t* d_out_visited) {
  return guarded([&] {
    set_device(c);
    if (use_bulk_exchange(c)) search_xchg(c, false, c->sh.nranks, d_queries, nq, dim, p, d_out_ids, d_out_dists, d_out_count, d_out_visited);
    else search_sharded(c, false, c->sh.nranks, d_queries, nq, dim, p, d_out_ids, d_out_dists, d_out_count, d_out_visited);
  });
}

dvsg_status dvsg_assign_top_c(dvsg_ctx* c, const float* queries, uint64_t nq, int dim, int cc, uint32_t* out) {
  return guarded([&] {
    set_device(c);
    if (c->clusters < 1) fail(DVSG_EINVAL, "assign_top_c: empty centroids");
    if (cc < 1 || cc > c->clusters) fail(DVSG_EINVAL, "assign_top_c: c=%d out of range for %d clusters", cc, c->clusters);
    if (dim != c->dim) fail(DVSG_EINVAL, "assign_top_c: query dim %d != centroid dim %d", dim, c->dim);
    if (nq == 0) return;
    if (!finite_all(queries, nq * (uint64_t)dim)) fail(DVSG_EINVAL, "Dataset: non-finite query element");
    const float* d_q = stage(c->io_f, queries, nq * (uint64_t)dim, c->stream);
    c->assign.reserve(nq * (uint64_t)cc, c->stream);
    c->assign_scratch.reserve(dvsg::assign_scratch_words(nq, dim, c->clusters, cc), c->stream);
    cuda_check(dvsg::launch_assign(d_q, nq, dim, c->d_cents.p, c->d_cent_norms.p, c->clusters, cc, c->assign.p, c->assign_scratch.p, c->stream, &c->assign_path), "assign");
    c->launches += assign_launches(c->assign_path);
    cuda_check(cudaMemcpyAsync(out, c->assign.p, nq * (uint64_t)cc * 4, cudaMemcpyDeviceToHost, c->stream), "D2H");
    cuda_check(cudaStreamSynchronize(c->stream), "assign");
  });
}

dvsg_status dvsg_assign_top_c_device(dvsg_ctx* c, const float* d_queries, uint64_t nq, int dim, int cc,
                                     uint32_t* d_out) {
  return guarded([&] {
    set_device(c);
    if (c->clusters < 1) fail(DVSG_EINVAL, "assign_top_c: empty centroids");
    if (cc < 1 || cc > c->clusters) fail(DVSG_EINVAL, "assign_top_c: c=%d out of range for %d clusters", cc, c->clusters);
    if (dim != c->dim) fail(DVSG_EINVAL, "assign_top_c: query dim %d != centroid dim %d", dim, c->dim);
    if (nq == 0) return;
    c->assign_scratch.reserve(dvsg::assign_scratch_words(nq, dim, c->clusters, cc), c->stream);
    cuda_check(dvsg::launch_assign(d_queries, nq, dim, c->d_cents.p, c->d_cent_norms.p, c->clusters, cc, d_out, c->assign_scratch.p, c->stream, &c->assign_path), "assign");
    c->launches += assign_launches(c->assign_path);
  });
}

dvsg_status dvsg_combine_results_device(dvsg_ctx* c, uint64_t nq, int nparts, const uint32_t* d_ids,
                                        const float* d_dists, const uint32_t* d_counts, int stride, int k,
                                        uint32_t* d_out_ids, float* d_out_dists, uint32_t* d_out_count) {
  return guarded([&] {
    set_device(c);
    if (k < 1) fail(DVSG_EINVAL, "combine_results: k must be >= 1");
    if (nparts < 1 || nparts > 32) fail(DVSG_EINVAL, "combine_results: %d partials outside the device merge width 1..32", nparts);
    if (stride < k) fail(DVSG_EINVAL, "combine_results: stride %d below k %d", stride, k);
    if (nq == 0) return;
    c->err_flag.reserve(1, c->stream);
    cuda_check(cudaMemsetAsync(c->err_flag.p, 0, sizeof(int), c->stream), "err reset");
    cuda_check(dvsg::launch_combine(nq, nparts, d_ids, d_dists, d_counts, stride, k, d_out_ids, d_out_dists, d_out_count, c->err_flag.p, c->stream), "combine");
    c->launches += 1;
    check_err_flag(c, "combine_results: partial list not sorted by (dist, id)");
  });
}

dvsg_status dvsg_gather_vectors_device(dvsg_ctx* c, const uint32_t* d_ids, const uint32_t* d_counts,
                                       uint64_t n, int k, float* d_out) {
  return guarded([&] {
    set_device(c);
    if (c->parts.empty()) fail(DVSG_EINVAL, "gather_vectors: no resident partition");
    if (n == 0) return;
    build_locator(c);
    cuda_check(dvsg::launch_gather_vectors(d_ids, d_counts, n, k, c->d_locator.p, c->vec.p, c->dim, c->dpad, d_out, c->stream), "gather vectors");
    c->launches += 1;
  });
}

dvsg_status dvsg_combine_results(dvsg_ctx* c, uint64_t nq, int nparts, const uint32_t* ids,
                                 const float* dists, const uint32_t* counts, int stride, int k,
                                 uint32_t* out_ids, float* out_dists, uint32_t* out_count) {
  return guarded([&] {
    set_device(c);
    if (k < 1) fail(DVSG_EINVAL, "combine_results: k must be >= 1");
    if (nparts < 0 || nparts > 32) fail(DVSG_EINVAL, "combine_results: %d partials above the device merge width 32", nparts);
    if (stride < 0) fail(DVSG_EINVAL, "combine_results: negative stride");
    for (uint64_t i = 0; i < nq * (uint64_t)nparts; ++i)
      if ((int64_t)counts[i] > stride) fail(DVSG_EINVAL, "combine_results: partial count %u above stride %d", counts[i], stride);
    if (nq == 0) return;
    if (nparts == 0) {
      for (uint64_t q = 0; q < nq; ++q) out_count[q] = 0;
      return;
    }
    const uint64_t tot = nq * (uint64_t)nparts * (uint64_t)stride;
    DevBuf<uint32_t> di, dc, oi, oc;
    DevBuf<float> dd, od;
    stage(di, ids, tot, c->stream);
    stage(dd, dists, tot, c->stream);
    stage(dc, counts, nq * (uint64_t)nparts, c->stream);
    oi.reserve(nq * (uint64_t)k, c->stream);
    od.reserve(nq * (uint64_t)k, c->stream);
    oc.reserve(nq, c->stream);
    c->err_flag.reserve(1, c->stream);
    cuda_check(cudaMemsetAsync(c->err_flag.p, 0, sizeof(int), c->stream), "err reset");
    cuda_check(dvsg::launch_combine(nq, nparts, di.p, dd.p, dc.p, stride, k, oi.p, od.p, oc.p, c->err_flag.p, c->stream), "combine");
    c->launches += 1;
    check_err_flag(c, "combine_results: partial list not sorted by (dist, id)");
    cuda_check(cudaMemcpy(out_ids, oi.p, nq * (uint64_t)k * 4, cudaMemcpyDeviceToHost), "D2H");
    cuda_check(cudaMemcpy(out_dists, od.p, nq * (uint64_t)k * 4, cudaMemcpyDeviceToHost), "D2H");
    cuda_check(cudaMemcpy(out_count, oc.p, nq * 4, cudaMemcpyDeviceToHost), "D2H");
  });
}

dvsg_status dvsg_run_pipeline(dvsg_ctx* c, const float* queries, uint64_t nq, int dim,
                              const dvsg_search_params* p, int fanout, int ranks, int batch_index,
                              uint32_t* out_ids, float* out_dists, uint32_t* out_count,
                              float* out_vectors, uint64_t* visited_total) {
  return guarded([&] {
    set_device(c);
    validate_params(p);
    // simulator.cpp:250-273 validation order
    if (c->clusters < 1 || c->parts.empty()) fail(DVSG_EINVAL, "BuiltIndex: index is not built");
    if ((int)c->parts.size() != c->clusters) fail(DVSG_EINVAL, "BuiltIndex: %zu graphs for %d clusters", c->parts.size(), c->clusters);
    if (dim != c->dim) fail(DVSG_EINVAL, "run_pipeline: query dim %d != index dim %d", dim, c->dim);
    if (fanout < 1 || fanout > c->clusters) fail(DVSG_EINVAL, "run_pipeline: fanout %d out of range for %d clusters", fanout, c->clusters);
    if (ranks != c->ranks) fail(DVSG_EINVAL, "run_pipeline: placement built for %d ranks, topology has %d", c->ranks, ranks);
    if (nq < 2) fail(DVSG_EINVAL, "run_pipeline: two_microbatch mode needs >= 2 queries");
    if (batch_index < 0) fail(DVSG_EINVAL, "origin_rank_for_batch: negative batch index");
    const uint64_t k = (uint64_t)p->k;
    c->io_f.reserve(nq * (uint64_t)dim, c->stream);
    c->io_u.reserve(nq * k + nq, c->stream);
    DevBuf<float>& od = c->io_dists;
    DevBuf<float>& ov = c->io_vecs;
    od.reserve(nq * k, c->stream);
    if (out_vectors) ov.reserve(nq * k * (uint64_t)dim, c->stream);
    c->u_visited.reserve(nq * (uint64_t)fanout, c->stream);
    c->io_u64.reserve(1, c->stream);
    c->err_flag.reserve(1, c->stream);
    if (out_vectors) build_locator(c);
    sync_slots(c);
    cuda_check(cudaMemsetAsync(c->err_flag.p, 0, sizeof(int), c->stream), "err reset");
    // Microbatch pipeline -- the reference's two_microbatch schedule
    // (simulator.cpp:295-297, replay_schedule :111-168) made real: H2D of
    // batch i+1 and D2H of batch i-1 on the copy stream overlap batch i's
    // search on the compute stream.  Pinned host buffers are needed for the
    // copies to be asynchronous.
    static const uint64_t mb_queries = [] {
      const char* e = std::getenv("DVSG_MB_QUERIES");
      return e ? std::max<uint64_t>(1, std::strtoull(e, nullptr, 10)) : 25000ull;
    }();
    const uint64_t mb = std::max<uint64_t>(2, std::min<uint64_t>(16, nq / mb_queries));
    cudaEvent_t* evh = c->mb_ev;
    cudaEvent_t* evc = c->mb_ev + 16;
    const cudaStream_t cs = c->stream, xs = c->comm;
    // the copy stream must not start before buffers are reset on the compute stream
    cuda_check(cudaEventRecord(evc[15], cs), "event");
    cuda_check(cudaStreamWaitEvent(xs, evc[15], 0), "wait");
    // decreasing microbatch sizes (weights mb, mb-1, ..., 1): the last D2H --
    // the only copy nothing overlaps -- is the smallest
    static const bool taper = [] {
      const char* e = std::getenv("DVSG_MB_TAPER");
      return e ? std::atoi(e) != 0 : true;
    }();
    const uint64_t wsum = taper ? mb * (mb + 1) / 2 : mb;
    auto edge = [&](uint64_t i) -> uint64_t {  // prefix of the first i microbatches
      const uint64_t w = taper ? i * mb - i * (i - 1) / 2 : i;
      return nq * w / wsum;
    };
    // measured timeline (timing on): 6 events per microbatch
    const bool tl = c->timing;
    cudaEvent_t* tv = c->tl_ev + 1;
    c->tl_mb = tl ? (int)mb : 0;
    if (tl) cuda_check(cudaEventRecord(c->tl_ev[0], xs), "event");
    auto h2d = [&](uint64_t i) {
      const uint64_t q0 = edge(i), n_i = edge(i + 1) - q0;
      if (tl) cuda_check(cudaEventRecord(tv[6 * i + 0], xs), "event");
      if (n_i)
        cuda_check(cudaMemcpyAsync(c->io_f.p + q0 * (uint64_t)dim, queries + q0 * (uint64_t)dim,
                                   n_i * (uint64_t)dim * 4, cudaMemcpyHostToDevice, xs), "H2D");
      if (tl) cuda_check(cudaEventRecord(tv[6 * i + 1], xs), "event");
      cuda_check(cudaEventRecord(evh[i], xs), "event");
    };
    auto compute = [&](uint64_t i) {
      const uint64_t q0 = edge(i), n_i = edge(i + 1) - q0;
      if (n_i == 0) {
        if (tl) {
          cuda_check(cudaEventRecord(tv[6 * i + 2], cs), "event");
          cuda_check(cudaEventRecord(tv[6 * i + 3], cs), "event");
        }
        return;
      }
      float* dq = c->io_f.p + q0 * (uint64_t)dim;
      cuda_check(cudaStreamWaitEvent(cs, evh[i], 0), "wait");
      if (tl) cuda_check(cudaEventRecord(tv[6 * i + 2], cs), "event");
      cuda_check(dvsg::launch_check_finite(dq, n_i * (uint64_t)dim, c->err_flag.p, cs), "finite check");
      c->launches += 1;
      pipeline_device(c, dq, n_i, dim, p, fanout, c->io_u.p + q0 * k, od.p + q0 * k, c->io_u.p + nq * k + q0,
                      out_vectors ? ov.p + q0 * k * (uint64_t)dim : nullptr, c->u_visited.p + q0 * (uint64_t)fanout,
                      false);
      if (tl) cuda_check(cudaEventRecord(tv[6 * i + 3], cs), "event");
      cuda_check(cudaEventRecord(evc[i], cs), "event");
    };
    auto d2h = [&](uint64_t i) {
      const uint64_t q0 = edge(i), n_i = edge(i + 1) - q0;
      if (n_i == 0) {
        if (tl) {
          cuda_check(cudaEventRecord(tv[6 * i + 4], xs), "event");
          cuda_check(cudaEventRecord(tv[6 * i + 5], xs), "event");
        }
        return;
      }
      cuda_check(cudaStreamWaitEvent(xs, evc[i], 0), "wait");
      if (tl) cuda_check(cudaEventRecord(tv[6 * i + 4], xs), "event");
      cuda_check(cudaMemcpyAsync(out_ids + q0 * k, c->io_u.p + q0 * k, n_i * k * 4, cudaMemcpyDeviceToHost, xs), "D2H");
      cuda_check(cudaMemcpyAsync(out_dists + q0 * k, od.p + q0 * k, n_i * k * 4, cudaMemcpyDeviceToHost, xs), "D2H");
      cuda_check(cudaMemcpyAsync(out_count + q0, c->io_u.p + nq * k + q0, n_i * 4, cudaMemcpyDeviceToHost, xs), "D2H");
      if (out_vectors)
        cuda_check(cudaMemcpyAsync(out_vectors + q0 * k * (uint64_t)dim, ov.p + q0 * k * (uint64_t)dim,
                                   n_i * k * (uint64_t)dim * 4, cudaMemcpyDeviceToHost, xs), "D2H");
      if (tl) cuda_check(cudaEventRecord(tv[6 * i + 5], xs), "event");
    };
    // Pageable host buffers make cudaMemcpyAsync host-synchronous: a D2H
    // returns only after its batch's compute and copy, so issued right after
    // that compute it would keep the host from queueing the next batch and
    // leave the GPU idle between microbatches.  Then the order is H2D(0),
    // C(0), H2D(1), C(1), D2H(0), H2D(2), C(2), D2H(1), ...: while the host
    // stages one copy the GPU already holds the next compute.
    auto pinned = [](const void* ptr) {
      cudaPointerAttributes at{};
      if (cudaPointerGetAttributes(&at, ptr) != cudaSuccess) {
        cudaGetLastError();
        return false;
      }
      return at.type == cudaMemoryTypeHost || at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
    };
    const bool pageable = !pinned(queries) || !pinned(out_ids) || !pinned(out_dists) || !pinned(out_count) ||
                          (out_vectors && !pinned(out_vectors));
    c->pipeline_pageable = pageable;
    if (!pageable) {
      // every H2D first: a D2H queued on the copy stream waits for its batch's
      // compute, so an H2D queued behind it would serialize the whole pipeline
      for (uint64_t i = 0; i < mb; ++i) h2d(i);
      for (uint64_t i = 0; i < mb; ++i) {
        compute(i);
        d2h(i);
      }
    } else {
      h2d(0);
      for (uint64_t i = 0; i < mb; ++i) {
        compute(i);
        if (i + 1 < mb) h2d(i + 1);
        if (i >= 1) d2h(i - 1);
      }
      d2h(mb - 1);
    }
    cuda_check(dvsg::launch_reduce_u64(c->u_visited.p, nq * (uint64_t)fanout, reinterpret_cast<unsigned long long*>(c->io_u64.p), cs), "reduce");
    c->launches += 1;
    int flag = 0;
    cuda_check(cudaMemcpyAsync(&flag, c->err_flag.p, sizeof(int), cudaMemcpyDeviceToHost, cs), "D2H");
    if (visited_total) cuda_check(cudaMemcpyAsync(visited_total, c->io_u64.p, 8, cudaMemcpyDeviceToHost, cs), "D2H");
    cuda_check(cudaStreamSynchronize(cs), "run_pipeline");
    cuda_check(cudaStreamSynchronize(xs), "run_pipeline");
    if (flag & 4) fail(DVSG_EINVAL, "Dataset: non-finite query element");
    if (flag) fail(DVSG_EINTERNAL, "route: cluster id outside placement / not resident, or combine_results: partial list not sorted");
    read_timings(c, true);
  });
}

dvsg_status dvsg_run_pipeline_device(dvsg_ctx* c, const float* d_queries, uint64_t nq, int dim,
                                     const dvsg_search_params* p, int fanout, uint32_t* d_out_ids,
                                     float* d_out_dists, uint32_t* d_out_count, float* d_out_vectors,
                                     uint64_t* d_visited) {
  return guarded([&] {
    set_device(c);
    if (d_out_vectors) build_locator(c);
    pipeline_device(c, d_queries, nq, dim, p, fanout, d_out_ids, d_out_dists, d_out_count, d_out_vectors, d_visited);
  });
}

dvsg_status dvsg_build_graph(dvsg_ctx* c, const float* vectors, uint64_t n, int dim, int out_degree,
                             uint32_t* adjacency_out) {
  return guarded([&] {
    set_device(c);
    if (n == 0) fail(DVSG_EINVAL, "build_graph: empty partition");
    if (out_degree < 1) fail(DVSG_EINVAL, "build_graph: out_degree must be >= 1");
    if (out_degree > 32) fail(DVSG_EINVAL, "build_graph: out_degree %d above the device limit 32", out_degree);
    if (dim < 1) fail(DVSG_EINVAL, "Dataset: dim must be positive, got %d", dim);
    if (!finite_all(vectors, n * (uint64_t)dim)) fail(DVSG_EINVAL, "Dataset: non-finite element");
    const int dpad = (dim + 3) & ~3;
    DevBuf<float> dv;
    DevBuf<uint32_t> da;
    dv.reserve(n * (uint64_t)dpad, c->stream);
    da.reserve(n * (uint64_t)out_degree, c->stream);
    cuda_check(cudaMemset(dv.p, 0, n * (uint64_t)dpad * 4), "memset");
    cuda_check(cudaMemcpy2D(dv.p, (size_t)dpad * 4, vectors, (size_t)dim * 4, (size_t)dim * 4, n, cudaMemcpyHostToDevice), "H2D");
    legacy_fence();
    if (k6_fp32_exact(vectors, n, dim)) {
      cuda_check(dvsg::launch_knn_build(dv.p, n, dim, dpad, out_degree, da.p, c->stream), "knn build");
      c->launches += 1;
      c->knn_exact = 0;
    } else {  // float data: fp32 candidates + fp64 re-rank + certificate + fp64 fallback
      DevBuf<unsigned char> ks;
      ks.reserve(dvsg::knn_exact_scratch_bytes(n), c->stream);
      cuda_check(dvsg::launch_knn_exact(dv.p, n, dv.p, n, dim, dpad, out_degree, true, da.p, nullptr, ks.p,
                                        c->stream), "knn build (exact)");
      c->launches += 3;
      uint32_t fb = 0;
      cuda_check(cudaMemcpyAsync(&fb, ks.p, 4, cudaMemcpyDeviceToHost, c->stream), "fallbacks");
      cuda_check(cudaStreamSynchronize(c->stream), "knn build");
      c->knn_exact = 1;
      c->knn_fallbacks = fb;
    }
    cuda_check(cudaStreamSynchronize(c->stream), "knn build");
    cuda_check(cudaMemcpy(adjacency_out, da.p, n * (uint64_t)out_degree * 4, cudaMemcpyDeviceToHost), "D2H");
  });
}

dvsg_status dvsg_brute_force_topk(dvsg_ctx* c, const float* db, uint64_t n, int dim, const float* queries,
                                  uint64_t nq, int k, uint32_t* out_ids, float* out_dists) {
  return guarded([&] {
    set_device(c);
    if (n == 0) fail(DVSG_EINVAL, "brute_force_topk: empty database");
    if (k < 1 || (uint64_t)k > n) fail(DVSG_EINVAL, "brute_force_topk: k=%d out of range for database of size %llu", k, (unsigned long long)n);
    if (k > 32) fail(DVSG_EINVAL, "brute_force_topk: k=%d above the device limit 32", k);
    if (dim < 1) fail(DVSG_EINVAL, "Dataset: dim must be positive, got %d", dim);
    if (nq == 0) return;
    const int dpad = (dim + 3) & ~3;
    DevBuf<float> dd, dq;
    DevBuf<uint32_t> oi;
    DevBuf<float> od;
    dd.reserve(n * (uint64_t)dpad, c->stream);
    dq.reserve(nq * (uint64_t)dpad, c->stream);
    oi.reserve(nq * (uint64_t)k, c->stream);
    od.reserve(nq * (uint64_t)k, c->stream);
    cuda_check(cudaMemset(dd.p, 0, n * (uint64_t)dpad * 4), "memset");
    cuda_check(cudaMemset(dq.p, 0, nq * (uint64_t)dpad * 4), "memset");
    cuda_check(cudaMemcpy2D(dd.p, (size_t)dpad * 4, db, (size_t)dim * 4, (size_t)dim * 4, n, cudaMemcpyHostToDevice), "H2D");
    cuda_check(cudaMemcpy2D(dq.p, (size_t)dpad * 4, queries, (size_t)dim * 4, (size_t)dim * 4, nq, cudaMemcpyHostToDevice), "H2D");
    legacy_fence();
    if (k6_fp32_exact2(db, n, queries, nq, dim)) {
      cuda_check(dvsg::launch_brute_force(dq.p, nq, dd.p, n, dpad, k, oi.p, od.p, c->stream), "brute force");
      c->launches += 1;
      c->knn_exact = 0;
    } else {
      DevBuf<unsigned char> ks;
      ks.reserve(dvsg::knn_exact_scratch_bytes(nq), c->stream);
      cuda_check(dvsg::launch_knn_exact(dq.p, nq, dd.p, n, dim, dpad, k, false, oi.p, od.p, ks.p, c->stream),
                 "brute force (exact)");
      c->launches += 3;
      uint32_t fb = 0;
      cuda_check(cudaMemcpyAsync(&fb, ks.p, 4, cudaMemcpyDeviceToHost, c->stream), "fallbacks");
      cuda_check(cudaStreamSynchronize(c->stream), "brute force");
      c->knn_exact = 1;
      c->knn_fallbacks = fb;
    }
    cuda_check(cudaStreamSynchronize(c->stream), "brute force");
    cuda_check(cudaMemcpy(out_ids, oi.p, nq * (uint64_t)k * 4, cudaMemcpyDeviceToHost), "D2H");
    cuda_check(cudaMemcpy(out_dists, od.p, nq * (uint64_t)k * 4, cudaMemcpyDeviceToHost), "D2H");
  });
}

// ---- large-index construction on the device (ivf_build.cu) ---------------

dvsg_status dvsg_row_norms_device(dvsg_ctx* c, const float* d_x, uint64_t n, int dpad, float* d_out) {
  return guarded([&] {
    set_device(c);
    if (dpad < 4 || dpad % 4) fail(DVSG_EINVAL, "row_norms: dpad %d must be a positive multiple of 4", dpad);
    cuda_check(dvsg::launch_row_norms(d_x, n, dpad, d_out, c->stream), "row norms");
    c->launches += 1;
    cuda_check(cudaStreamSynchronize(c->stream), "row norms");
  });
}

dvsg_status dvsg_range_topk_device(dvsg_ctx* c, const float* d_rows, const float* d_row_norms,
                                   const float* d_cols, const float* d_col_norms, int dpad,
                                   const uint32_t* d_row_map, const dvsg_range_block* d_blocks, uint64_t nblocks,
                                   const uint32_t* d_list_off, const uint32_t* d_ranges, int m,
                                   int flags, uint32_t* d_out_ids, float* d_out_dists,
                                   uint64_t out_stride) {
  static_assert(sizeof(dvsg_range_block) == sizeof(dvsg::RangeBlock), "range block layout");
  return guarded([&] {
    set_device(c);
    if (m < 1 || m > 32) fail(DVSG_EINVAL, "range_topk: m=%d outside 1..32", m);
    if (dpad < 4 || dpad % 4) fail(DVSG_EINVAL, "range_topk: dpad %d must be a positive multiple of 4", dpad);
    if ((uint64_t)m > out_stride) fail(DVSG_EINVAL, "range_topk: out_stride %llu < m", (unsigned long long)out_stride);
    if ((flags & DVSG_RANGE_MERGE) && !d_out_dists) fail(DVSG_EINVAL, "range_topk: DVSG_RANGE_MERGE needs d_out_dists");
    if (!d_rows || !d_cols || !d_row_norms || !d_col_norms || !d_out_ids || (nblocks && (!d_blocks || !d_list_off || !d_ranges)))
      fail(DVSG_EINVAL, "range_topk: null input");
    cuda_check(dvsg::launch_range_topk(d_rows, d_row_norms, d_cols, d_col_norms, dpad, d_row_map,
                                       reinterpret_cast<const dvsg::RangeBlock*>(d_blocks), nblocks,
                                       d_list_off, reinterpret_cast<const uint2*>(d_ranges), m, flags,
                                       d_out_ids, d_out_dists, out_stride, c->stream), "range_topk");
    c->launches += 1;
    cuda_check(cudaStreamSynchronize(c->stream), "range_topk");
  });
}

dvsg_status dvsg_to_bf16_device(dvsg_ctx* c, const float* d_x, uint64_t n, int dpad, int kpad, uint16_t* d_out) {
  return guarded([&] {
    set_device(c);
    if (kpad < dpad || kpad % 16) fail(DVSG_EINVAL, "to_bf16: kpad %d must be a multiple of 16 >= dpad %d", kpad, dpad);
    cuda_check(dvsg::launch_to_bf16(d_x, n, dpad, kpad, d_out, c->stream), "to bf16");
    c->launches += 1;
    cuda_check(cudaStreamSynchronize(c->stream), "to bf16");
  });
}

dvsg_status dvsg_range_topk_bf16_device(dvsg_ctx* c, const uint16_t* d_rows, const float* d_row_norms,
                                        const uint16_t* d_cols, const float* d_col_norms, int kpad,
                                        const uint32_t* d_row_map, const dvsg_range_block* d_blocks, uint64_t nblocks,
                                        const uint32_t* d_list_off, const uint32_t* d_ranges, int m, int flags,
                                        uint32_t* d_out_ids, float* d_out_dists, uint64_t out_stride) {
  return guarded([&] {
    set_device(c);
    if (m < 1 || m > 32) fail(DVSG_EINVAL, "range_topk: m=%d outside 1..32", m);
    if (kpad < 16 || kpad > 256 || kpad % 16) fail(DVSG_EINVAL, "range_topk (tensor cores): kpad %d outside 16..256 step 16", kpad);
    if ((uint64_t)m > out_stride) fail(DVSG_EINVAL, "range_topk: out_stride %llu < m", (unsigned long long)out_stride);
    if ((flags & DVSG_RANGE_MERGE) && !d_out_dists) fail(DVSG_EINVAL, "range_topk: DVSG_RANGE_MERGE needs d_out_dists");
    if (!d_rows || !d_cols || !d_row_norms || !d_col_norms || !d_out_ids || (nblocks && (!d_blocks || !d_list_off || !d_ranges)))
      fail(DVSG_EINVAL, "range_topk: null input");
    cuda_check(dvsg::launch_range_topk_tc(d_rows, d_row_norms, d_cols, d_col_norms, kpad, d_row_map,
                                          reinterpret_cast<const dvsg::RangeBlock*>(d_blocks), nblocks, d_list_off,
                                          reinterpret_cast<const uint2*>(d_ranges), m, flags, d_out_ids, d_out_dists,
                                          out_stride, c->stream), "range_topk tc");
    c->launches += 1;
    cuda_check(cudaStreamSynchronize(c->stream), "range_topk tc");
  });
}

dvsg_status dvsg_segment_means_device(dvsg_ctx* c, const float* d_x, int dpad, const uint32_t* d_idx,
                                      const uint64_t* d_off, uint32_t nseg, float* d_cents) {
  return guarded([&] {
    set_device(c);
    if (dpad < 1) fail(DVSG_EINVAL, "segment_means: dpad %d", dpad);
    cuda_check(dvsg::launch_segment_means(d_x, dpad, d_idx, d_off, nseg, d_cents, c->stream), "segment means");
    c->launches += 1;
    cuda_check(cudaStreamSynchronize(c->stream), "segment means");
  });
}

namespace {
void entry_order_device(dvsg_ctx* c, const float* d_x, uint64_t n, int dim, int dpad, uint32_t* d_out) {
  if (n == 0 || dim < 1) fail(DVSG_EINVAL, "compute_entry_order: empty partition");
  if (dim > 1024) fail(DVSG_EINVAL, "compute_entry_order (device): dim %d above 1024", dim);
  const size_t bytes = dvsg::entry_order_scratch_bytes(n);
  DevBuf<unsigned char> scratch;
  scratch.reserve(bytes, c->stream);
  cuda_check(dvsg::launch_entry_order(d_x, n, dim, dpad, scratch.p, bytes, d_out, c->stream), "entry order");
  c->launches += 4;
  cuda_check(cudaStreamSynchronize(c->stream), "entry order");
}
}  // namespace

dvsg_status dvsg_compute_entry_order_device(dvsg_ctx* c, const float* d_x, uint64_t n, int dim, int dpad,
                                            uint32_t* d_out) {
  return guarded([&] {
    set_device(c);
    if (dpad < dim || dpad % 4) fail(DVSG_EINVAL, "compute_entry_order: dpad %d (dim %d)", dpad, dim);
    entry_order_device(c, d_x, n, dim, dpad, d_out);
  });
}

dvsg_status dvsg_partition_alloc_device(dvsg_ctx* c, uint32_t cluster, uint64_t n, int dim, int out_degree,
                                        float** d_vectors, uint32_t** d_adjacency, uint32_t** d_global_ids,
                                        uint32_t** d_entry_order) {
  return guarded([&] {
    set_device(c);
    if (c->pend.active) fail(DVSG_EINVAL, "partition_alloc: partition %u not committed yet", c->pend.cluster);
    if (c->sh.active) fail(DVSG_EINVAL, "partition_alloc: this context holds one rank's shard");
    if (n == 0) fail(DVSG_EINVAL, "BuiltIndex: empty partition");
    if (n >= (1ull << 31)) fail(DVSG_EINVAL, "load_partition: %llu rows exceed the 2^31 local-id limit", (unsigned long long)n);
    if (dim < 1) fail(DVSG_EINVAL, "Dataset: dim must be positive, got %d", dim);
    if (out_degree < 1) fail(DVSG_EINVAL, "build_graph: out_degree must be >= 1");
    if (c->dim && c->dim != dim) fail(DVSG_EINVAL, "BuiltIndex: graph dim mismatch (%d vs %d)", dim, c->dim);
    if (c->dg && c->dg != out_degree) fail(DVSG_EINVAL, "BuiltIndex: graph out-degree mismatch (%d vs %d)", out_degree, c->dg);
    if (slot_of(c, cluster) >= 0) fail(DVSG_EINVAL, "load_partition: cluster %u already resident", cluster);
    cuda_check(cudaStreamSynchronize(c->stream), "sync");
    const int dpad = (dim + 3) & ~3;
    const uint64_t r0 = c->rows, r1 = r0 + n;
    c->vec.reserve(r1 * (uint64_t)dpad, c->stream, true, r0 * (uint64_t)dpad);
    c->adj.reserve(r1 * (uint64_t)out_degree, c->stream, true, r0 * (uint64_t)out_degree);
    c->gids.reserve(r1, c->stream, true, r0);
    c->entry.reserve(r1, c->stream, true, r0);
    c->dim = dim;
    c->dpad = dpad;
    c->dg = out_degree;
    if (dpad != dim) cuda_check(cudaMemset(c->vec.p + r0 * dpad, 0, n * (uint64_t)dpad * 4), "pad");
    legacy_fence();
    c->pend = dvsg_ctx::Pending{true, cluster, n, r0};
    if (d_vectors) *d_vectors = c->vec.p + r0 * dpad;
    if (d_adjacency) *d_adjacency = c->adj.p + r0 * out_degree;
    if (d_global_ids) *d_global_ids = c->gids.p + r0;
    if (d_entry_order) *d_entry_order = c->entry.p + r0;
  });
}

dvsg_status dvsg_partition_commit_device(dvsg_ctx* c, int flags) {
  return guarded([&] {
    set_device(c);
    if (!c->pend.active) fail(DVSG_EINVAL, "partition_commit: no partition allocated");
    const auto pd = c->pend;
    c->pend.active = false;  // a failed commit drops the partition
    const float* v = c->vec.p + pd.r0 * c->dpad;
    uint32_t* gids = c->gids.p + pd.r0;
    if (flags & DVSG_COMMIT_IOTA_IDS) cuda_check(dvsg::launch_iota(gids, pd.n, c->stream), "iota");
    c->err_flag.reserve(1, c->stream);
    cuda_check(cudaMemsetAsync(c->err_flag.p, 0, sizeof(int), c->stream), "flag");
    cuda_check(dvsg::launch_check_partition(v, pd.n, c->dim, c->dpad, c->adj.p + pd.r0 * c->dg, c->dg, gids,
                                            c->err_flag.p, c->stream), "check partition");
    int flag = 0;
    cuda_check(cudaMemcpyAsync(&flag, c->err_flag.p, sizeof(int), cudaMemcpyDeviceToHost, c->stream), "flag");
    cuda_check(cudaStreamSynchronize(c->stream), "check partition");
    c->launches += 2;
    if (flag & 1) fail(DVSG_EFORMAT, "index file: neighbor id out of range in cluster %u", pd.cluster);
    if (flag & 4) fail(DVSG_EINVAL, "Dataset: non-finite element in partition %u", pd.cluster);
    if (flag & 32) fail(DVSG_EINVAL, "partition_commit: pad columns %d..%d must be zero", c->dim, c->dpad - 1);
    if (flags & DVSG_COMMIT_ENTRY_ORDER) entry_order_device(c, v, pd.n, c->dim, c->dpad, c->entry.p + pd.r0);
    c->parts.push_back(dvsg::PartDesc{pd.r0, (uint32_t)pd.n, pd.cluster});
    c->part_mono.push_back((flag & 64) == 0);
    c->all_integral = c->all_integral && (flag & 16) == 0;
    c->rows = pd.r0 + pd.n;
    c->vec_gen += 1;
    c->parts_dirty = c->slot_dirty = c->locator_dirty = c->anchors_dirty = true;
  });
}

dvsg_status dvsg_optimize_graph_device(dvsg_ctx* c, uint32_t* d_adjacency, uint64_t n, int out_degree,
                                       int keep) {
  return guarded([&] {
    set_device(c);
    if (out_degree < 2 || out_degree > 32) fail(DVSG_EINVAL, "optimize_graph: out_degree %d outside 2..32", out_degree);
    if (keep < 1 || keep > out_degree) fail(DVSG_EINVAL, "optimize_graph: keep %d outside 1..%d", keep, out_degree);
    if (n == 0 || n >= (1ull << 27)) fail(DVSG_EINVAL, "optimize_graph: n %llu outside 1..2^27", (unsigned long long)n);
    const size_t bytes = dvsg::graph_opt_scratch_bytes(n, out_degree, keep);
    DevBuf<unsigned char> scratch;
    scratch.reserve(bytes, c->stream);
    cuda_check(dvsg::launch_graph_optimize(d_adjacency, n, out_degree, keep, scratch.p, bytes, c->stream), "optimize graph");
    c->launches += 5;
    cuda_check(cudaStreamSynchronize(c->stream), "optimize graph");
  });
}

dvsg_status dvsg_partition_view_device(dvsg_ctx* c, uint32_t cluster, const float** d_vectors,
                                       const uint32_t** d_adjacency, const uint32_t** d_global_ids,
                                       const uint32_t** d_entry_order, uint64_t* n) {
  return guarded([&] {
    const int32_t s = slot_of(c, cluster);
    if (s < 0) fail(DVSG_EINVAL, "cluster %u not resident", cluster);
    const auto& pd = c->parts[(size_t)s];
    if (c->sh.active) fail(DVSG_EINVAL, "partition_view: this context holds one rank's shard");
    if (d_vectors) *d_vectors = c->vec.p + pd.row_off * c->dpad;
    if (d_adjacency) *d_adjacency = c->adj.p + pd.row_off * c->dg;
    if (d_global_ids) *d_global_ids = c->gids.p + pd.row_off;
    if (d_entry_order) *d_entry_order = c->entry.p + pd.row_off;
    if (n) *n = pd.n;
  });
}

dvsg_status dvsg_index_integral(dvsg_ctx* c, int* out) {
  return guarded([&] {
    if (!out) fail(DVSG_EINVAL, "index_integral: null out");
    *out = c->all_integral ? 1 : 0;
  });
}

// ---- kmeans_train / partition_database (kmeans.cpp:189-300) ---------------
namespace {

void validate_dataset(const float* x, uint64_t n, int dim) {
  if (dim <= 0) fail(DVSG_EINVAL, "Dataset: dim must be positive, got %d", dim);
  for (uint64_t i = 0; i < n * (uint64_t)dim; ++i)
    if (!std::isfinite(x[i])) fail(DVSG_EINVAL, "Dataset: non-finite element at flat index %llu", (unsigned long long)i);
}

std::vector<double> center_norms(const std::vector<float>& cents, int clusters, int dim) {
  std::vector<double> out((size_t)clusters);  // refresh_center_norms, kmeans.cpp:34-40
  for (int j = 0; j < clusters; ++j) {
    double acc = 0.0;
    for (int i = 0; i < dim; ++i) {
      const double v = (double)cents[(size_t)j * dim + i];
      acc += v * v;
    }
    out[(size_t)j] = acc;
  }
  return out;
}

// nearest_center of every row (kmeans.cpp:50-82) == K5 top-1, in query chunks
// that keep K5's (rows x clusters) key scratch under 512 MB
void assign_nearest(dvsg_ctx* c, const float* d_x, uint64_t n, int dim, const float* d_cents,
                    const double* d_norms, int clusters, uint32_t* d_labels, DevBuf<uint64_t>& scratch) {
  uint64_t chunk = std::max<uint64_t>(1024, (512ull << 20) / (8ull * (uint64_t)(clusters + 1)));
  if (dvsg::assign_scratch_words(chunk, dim, clusters, 1) < chunk * (uint64_t)(clusters + 1))
    chunk = std::max<uint64_t>(chunk, 1ull << 20);  // tensor-core path: O(rows x dim) scratch
  scratch.reserve(dvsg::assign_scratch_words(std::min<uint64_t>(chunk, n), dim, clusters, 1), c->stream);
  for (uint64_t b = 0; b < n; b += chunk) {
    const uint64_t m = std::min<uint64_t>(chunk, n - b);
    int path = 0;
    cuda_check(dvsg::launch_assign(d_x + b * (uint64_t)dim, m, dim, d_cents, d_norms, clusters, 1, d_labels + b,
                                   scratch.p, c->stream, &path), "assign");
    c->launches += assign_launches(path);
  }
}

}  // namespace

dvsg_status dvsg_kmeans_train(dvsg_ctx* c, const float* db, uint64_t n, int dim, int clusters, int max_iters,
                              uint64_t seed, float* centroids_out, int* iterations_out, double* wcss_out) {
  return guarded([&] {
    set_device(c);
    validate_dataset(db, n, dim);
    if (clusters < 1 || (uint64_t)clusters > n)
      fail(DVSG_EINVAL, "kmeans_train: clusters=%d out of range for database of size %llu", clusters, (unsigned long long)n);
    if (max_iters < 1) fail(DVSG_EINVAL, "kmeans_train: max_iters must be >= 1");
    if (!centroids_out) fail(DVSG_EINVAL, "kmeans_train: null output");
    cudaStream_t s = c->stream;
    const size_t C = (size_t)clusters, D = (size_t)dim;
    DevBuf<float> x, dc, od;
    DevBuf<double> d2, scan, dn;
    DevBuf<uint32_t> lab, keys, order, iota;
    DevBuf<uint64_t> ascratch;
    DevBuf<unsigned long long> pick;
    DevBuf<unsigned char> temp;
    x.reserve(n * D, s);
    cuda_check(cudaMemcpyAsync(x.p, db, n * D * 4, cudaMemcpyHostToDevice, s), "db H2D");
    dc.reserve(C * D, s);
    d2.reserve(n, s);
    scan.reserve(n, s);
    lab.reserve(n, s);
    od.reserve(n, s);
    dn.reserve(C, s);
    pick.reserve(1, s);
    const size_t tb = dvsg::kmeans_scan_bytes(n);
    temp.reserve(tb, s);
    std::mt19937_64 rng(seed);
    auto uniform01 = [&] { return (double)(rng() >> 11) * 0x1.0p-53; };
    auto uniform_index = [&](uint64_t m) {
      const uint64_t i = (uint64_t)(uniform01() * (double)m);
      return i < m ? i : m - 1;
    };
    std::vector<float> cents(C * D);
    auto set_center = [&](size_t j, uint64_t row) {
      std::memcpy(cents.data() + j * D, db + row * D, D * 4);
      cuda_check(cudaMemcpyAsync(dc.p + j * D, db + row * D, D * 4, cudaMemcpyHostToDevice, s), "center H2D");
    };
    // ---- init_kmeanspp (kmeans.cpp:150-187)
    set_center(0, uniform_index(n));
    cuda_check(dvsg::launch_kpp_d2(x.p, n, dim, dc.p, d2.p, 1, s), "kpp d2");
    for (size_t j = 1; j < C; ++j) {
      cuda_check(dvsg::launch_kpp_scan(d2.p, scan.p, n, temp.p, tb, s), "kpp scan");
      double total = 0.0;
      cuda_check(cudaMemcpyAsync(&total, scan.p + (n - 1), 8, cudaMemcpyDeviceToHost, s), "total");
      cuda_check(cudaStreamSynchronize(s), "sync");
      uint64_t p;
      if (total <= 0.0) {
        p = uniform_index(n);  // all residual mass gone (duplicates)
      } else {
        const double r = uniform01() * total;
        const unsigned long long init = n - 1;
        cuda_check(cudaMemcpyAsync(pick.p, &init, 8, cudaMemcpyHostToDevice, s), "pick init");
        cuda_check(dvsg::launch_first_gt(scan.p, n, r, pick.p, s), "first > r");
        unsigned long long pk = 0;
        cuda_check(cudaMemcpyAsync(&pk, pick.p, 8, cudaMemcpyDeviceToHost, s), "pick");
        cuda_check(cudaStreamSynchronize(s), "sync");
        p = pk;
      }
      set_center(j, p);
      cuda_check(dvsg::launch_kpp_d2(x.p, n, dim, dc.p + j * D, d2.p, 0, s), "kpp d2");
      c->launches += 3;
    }
    // ---- Lloyd (kmeans.cpp:216-226)
    std::vector<uint32_t> labels(n), prev;
    std::vector<float> dist(n);
    auto assign_all = [&] {
      const std::vector<double> norms = center_norms(cents, clusters, dim);
      cuda_check(cudaMemcpyAsync(dn.p, norms.data(), C * 8, cudaMemcpyHostToDevice, s), "norms");
      assign_nearest(c, x.p, n, dim, dc.p, dn.p, clusters, lab.p, ascratch);
      cuda_check(cudaMemcpyAsync(labels.data(), lab.p, n * 4, cudaMemcpyDeviceToHost, s), "labels");
      cuda_check(cudaStreamSynchronize(s), "sync");
    };
    auto own_dists = [&] {
      cuda_check(dvsg::launch_own_dist(x.p, n, dim, dc.p, lab.p, od.p, s), "own dist");
      cuda_check(cudaMemcpyAsync(dist.data(), od.p, n * 4, cudaMemcpyDeviceToHost, s), "dists");
      cuda_check(cudaStreamSynchronize(s), "sync");
      c->launches += 1;
    };
    // repair_empty_clusters (kmeans.cpp:84-117): every empty cluster takes the
    // row farthest from its own centroid among clusters that can spare one
    auto repair = [&] {
      std::vector<uint64_t> sizes(C, 0);
      for (uint32_t l : labels) ++sizes[l];
      if (std::find(sizes.begin(), sizes.end(), 0ull) == sizes.end()) return false;
      own_dists();  // unchanged by the moves below except for moved rows, which become ineligible
      bool changed = false;
      for (size_t e = 0; e < C; ++e) {
        if (sizes[e] > 0) continue;
        uint64_t worst = n;
        float wd = -1.0f;
        for (uint64_t i = 0; i < n; ++i) {
          if (sizes[labels[i]] < 2) continue;
          if (dist[i] > wd) {
            wd = dist[i];
            worst = i;
          }
        }
        if (worst == n) {  // nothing movable: the reference returns false, keeping earlier moves
          if (changed) cuda_check(cudaMemcpyAsync(lab.p, labels.data(), n * 4, cudaMemcpyHostToDevice, s), "labels H2D");
          return false;
        }
        set_center(e, worst);
        --sizes[labels[worst]];
        labels[worst] = (uint32_t)e;
        ++sizes[e];
        changed = true;
      }
      if (changed) cuda_check(cudaMemcpyAsync(lab.p, labels.data(), n * 4, cudaMemcpyHostToDevice, s), "labels H2D");
      return changed;
    };
    keys.reserve(n, s);
    order.reserve(n, s);
    iota.reserve(n, s);
    int iters = 0;
    for (int it = 0; it < max_iters; ++it) {
      assign_all();
      repair();
      if (labels == prev) break;  // fixed point: means would not move
      cuda_check(dvsg::launch_cluster_means(x.p, n, dim, lab.p, clusters, dc.p, keys.p, order.p, iota.p, temp.p, tb, s),
                 "update means");
      c->launches += 3;
      cuda_check(cudaMemcpyAsync(cents.data(), dc.p, C * D * 4, cudaMemcpyDeviceToHost, s), "cents D2H");
      if (wcss_out) {  // compute_wcss (kmeans.cpp:135-143): row-order fp64 sum
        own_dists();
        double acc = 0.0;
        for (uint64_t i = 0; i < n; ++i) acc += (double)dist[i];
        wcss_out[it] = acc;
      } else {
        cuda_check(cudaStreamSynchronize(s), "sync");
      }
      iters = it + 1;
      prev = labels;
    }
    // the returned centroids must induce a partition with no empty cluster (:229-240)
    for (int round = 0; round <= clusters; ++round) {
      assign_all();
      std::vector<char> seen(C, 0);
      for (uint32_t l : labels) seen[l] = 1;
      if (std::find(seen.begin(), seen.end(), 0) == seen.end()) {
        std::memcpy(centroids_out, cents.data(), C * D * 4);
        if (iterations_out) *iterations_out = iters;
        return;
      }
      if (!repair()) break;
    }
    fail(DVSG_EINVAL, "kmeans_train: cannot keep %d clusters non-empty; the dataset has too few distinct points", clusters);
  });
}

dvsg_status dvsg_partition_database(dvsg_ctx* c, const float* db, uint64_t n, int dim, const float* centroids,
                                    int clusters, uint32_t* labels_out) {
  return guarded([&] {
    set_device(c);
    validate_dataset(db, n, dim);
    if (clusters < 1 || !centroids) fail(DVSG_EINVAL, "partition_database: empty centroids");
    if (!labels_out) fail(DVSG_EINVAL, "partition_database: null output");
    cudaStream_t s = c->stream;
    std::vector<float> cents(centroids, centroids + (size_t)clusters * dim);
    const std::vector<double> norms = center_norms(cents, clusters, dim);
    DevBuf<float> x, dc;
    DevBuf<double> dn;
    DevBuf<uint32_t> lab;
    DevBuf<uint64_t> scratch;
    x.reserve(std::max<uint64_t>(n, 1) * (uint64_t)dim, s);
    dc.reserve((size_t)clusters * dim, s);
    dn.reserve((size_t)clusters, s);
    lab.reserve(std::max<uint64_t>(n, 1), s);
    if (n == 0) return;
    cuda_check(cudaMemcpyAsync(x.p, db, n * (uint64_t)dim * 4, cudaMemcpyHostToDevice, s), "db H2D");
    cuda_check(cudaMemcpyAsync(dc.p, centroids, (size_t)clusters * dim * 4, cudaMemcpyHostToDevice, s), "cents H2D");
    cuda_check(cudaMemcpyAsync(dn.p, norms.data(), (size_t)clusters * 8, cudaMemcpyHostToDevice, s), "norms H2D");
    assign_nearest(c, x.p, n, dim, dc.p, dn.p, clusters, lab.p, scratch);
    cuda_check(cudaMemcpyAsync(labels_out, lab.p, n * 4, cudaMemcpyDeviceToHost, s), "labels D2H");
    cuda_check(cudaStreamSynchronize(s), "sync");
  });
}

// ---- cluster-sharded run_pipeline with device-initiated exchange ----------
namespace {

size_t al256(size_t b) { return (b + 255) & ~(size_t)255; }
constexpr size_t kClHeader = 4096;  // flags [8] u32 @0, cursor [2][8] u32 @64

dvsg::ClArena cl_view(const dvsg_ctx* c, unsigned char* base) {
  const auto& cl = c->cl;
  dvsg::ClArena v{};
  v.flags = reinterpret_cast<unsigned*>(base);
  v.cursor = reinterpret_cast<unsigned*>(base + 64);
  v.inbox_q = reinterpret_cast<float*>(base + cl.off_q);
  v.inbox_meta = reinterpret_cast<uint2*>(base + cl.off_meta);
  v.r_ids = reinterpret_cast<uint32_t*>(base + cl.off_ids);
  v.r_dists = reinterpret_cast<float*>(base + cl.off_dists);
  v.r_count = reinterpret_cast<uint32_t*>(base + cl.off_count);
  v.r_visited = reinterpret_cast<uint64_t*>(base + cl.off_vis);
  v.r_vec = cl.with_vectors ? reinterpret_cast<float*>(base + cl.off_vec) : nullptr;
  return v;
}

void cl_connect(dvsg_ctx* c, const std::vector<unsigned char*>& bases) {
  auto& cl = c->cl;
  std::vector<dvsg::ClArena> views((size_t)cl.nranks);
  for (int r = 0; r < cl.nranks; ++r) views[(size_t)r] = cl_view(c, bases[(size_t)r]);
  c->cl_peers.reserve((size_t)cl.nranks, c->stream);
  cuda_check(cudaMemcpyAsync(c->cl_peers.p, views.data(), views.size() * sizeof(dvsg::ClArena), cudaMemcpyHostToDevice, c->stream), "peers");
  cuda_check(cudaStreamSynchronize(c->stream), "sync");
  cl.peers = bases;
  cl.connected = true;
}

void cl_check(dvsg_ctx* c) {
  if (!c->cl.active || !c->cl_err.p) return;
  int flag = 0, comb = 0;
  cuda_check(cudaMemcpyAsync(&flag, c->cl_err.p, sizeof(int), cudaMemcpyDeviceToHost, c->stream), "cl err");
  if (c->err_flag.p) cuda_check(cudaMemcpyAsync(&comb, c->err_flag.p, sizeof(int), cudaMemcpyDeviceToHost, c->stream), "err");
  cuda_check(cudaStreamSynchronize(c->stream), "sync");
  if (!flag && !comb) return;
  cuda_check(cudaMemsetAsync(c->cl_err.p, 0, sizeof(int), c->stream), "cl err reset");
  if (c->err_flag.p) cuda_check(cudaMemsetAsync(c->err_flag.p, 0, sizeof(int), c->stream), "err reset");
  if (flag & 1) fail(DVSG_EINTERNAL, "cluster exchange: a query was assigned a cluster id outside the routing table");
  if (flag & 2) fail(DVSG_EINVAL, "cluster exchange: an owner's inbox overflowed (raise max_queries/max_fanout)");
  if (flag & 4) fail(DVSG_EINTERNAL, "cluster exchange: a unit was routed to a rank that does not hold its cluster");
  if (flag & 8) fail(DVSG_EINTERNAL, "cluster exchange: a rank did not reach the barrier within 20 s");
  fail(DVSG_EINTERNAL, "combine_results: partial result list is not sorted");
}

}  // namespace

dvsg_status dvsg_cluster_comm_init(dvsg_ctx* c, int nranks, int rank, uint64_t max_queries, int max_fanout, int k,
                                   int with_vectors) {
  return guarded([&] {
    set_device(c);
    if (nranks < 1 || nranks > dvsg::kXgMaxRanks || rank < 0 || rank >= nranks)
      fail(DVSG_EINVAL, "cluster_comm_init: rank %d of %d", rank, nranks);
    if (c->dim < 1) fail(DVSG_EINVAL, "cluster_comm_init: load this rank's partitions and centroids first");
    if (max_queries < 1 || max_fanout < 1 || max_fanout > 32 || k < 1)
      fail(DVSG_EINVAL, "cluster_comm_init: bad capacity (max_queries %llu, max_fanout %d, k %d)",
           (unsigned long long)max_queries, max_fanout, k);
    auto& cl = c->cl;
    for (size_t r = 0; r < cl.peers.size(); ++r)
      if ((int)r != cl.rank && cl.peers[r] && !cl.own_peers) cudaIpcCloseMemHandle(cl.peers[r]);
    if (cl.arena) cudaFree(cl.arena);
    cl = dvsg_ctx::Cl{};
    cl.nranks = nranks;
    cl.rank = rank;
    cl.k = k;
    cl.max_fanout = max_fanout;
    cl.max_queries = max_queries;
    cl.dim = c->dim;
    cl.with_vectors = with_vectors != 0;
    cl.cap = max_queries * (uint64_t)max_fanout;  // worst case: every unit of an origin to one owner
    cl.ucap = cl.cap;
    size_t o = kClHeader;
    cl.off_q = o;
    o = al256(o + (size_t)nranks * cl.cap * (size_t)c->dim * 4);
    cl.off_meta = o;
    o = al256(o + (size_t)nranks * cl.cap * 8);
    cl.off_ids = o;
    o = al256(o + cl.ucap * (size_t)k * 4);
    cl.off_dists = o;
    o = al256(o + cl.ucap * (size_t)k * 4);
    cl.off_count = o;
    o = al256(o + cl.ucap * 4);
    cl.off_vis = o;
    o = al256(o + cl.ucap * 8);
    cl.off_vec = o;
    if (cl.with_vectors) o = al256(o + cl.ucap * (size_t)k * (size_t)c->dim * 4);
    cl.bytes = o;
    cuda_check(cudaMalloc(&cl.arena, cl.bytes), "cluster arena");
    cuda_check(cudaMemset(cl.arena, 0, kClHeader), "cluster arena header");
    const uint64_t units = (uint64_t)nranks * cl.cap;
    c->cl_uq.reserve(units, c->stream);
    c->cl_up.reserve(units, c->stream);
    c->cl_ids.reserve(units * (uint64_t)k, c->stream);
    c->cl_dists.reserve(units * (uint64_t)k, c->stream);
    c->cl_count.reserve(units, c->stream);
    c->cl_vis.reserve(units, c->stream);
    c->cl_nunits.reserve(1, c->stream);
    c->cl_err.reserve(1, c->stream);
    cuda_check(cudaMemset(c->cl_err.p, 0, sizeof(int)), "err");
    std::vector<uint32_t> place(c->placement.begin(), c->placement.end());
    if (place.empty()) fail(DVSG_EINVAL, "cluster_comm_init: no routing table (dvsg_set_centroids)");
    for (uint32_t r : place)
      if ((int)r >= nranks) fail(DVSG_EINVAL, "cluster_comm_init: placement names rank %u of %d", r, nranks);
    c->cl_place.reserve(place.size(), c->stream);
    cuda_check(cudaMemcpy(c->cl_place.p, place.data(), place.size() * 4, cudaMemcpyHostToDevice), "placement");
    legacy_fence();
    cl.active = true;
  });
}

dvsg_status dvsg_cluster_comm_export(dvsg_ctx* c, void* handle_out) {
  return guarded([&] {
    set_device(c);
    if (!c->cl.active) fail(DVSG_EINVAL, "cluster_comm_export: call dvsg_cluster_comm_init first");
    cudaIpcMemHandle_t h;
    cuda_check(cudaIpcGetMemHandle(&h, c->cl.arena), "ipc handle");
    std::memcpy(handle_out, &h, sizeof(h));
  });
}

dvsg_status dvsg_cluster_comm_connect(dvsg_ctx* c, const void* handles) {
  return guarded([&] {
    set_device(c);
    if (!c->cl.active) fail(DVSG_EINVAL, "cluster_comm_connect: call dvsg_cluster_comm_init first");
    std::vector<unsigned char*> bases((size_t)c->cl.nranks, nullptr);
    for (int r = 0; r < c->cl.nranks; ++r) {
      if (r == c->cl.rank) {
        bases[(size_t)r] = c->cl.arena;
        continue;
      }
      cudaIpcMemHandle_t h;
      std::memcpy(&h, static_cast<const unsigned char*>(handles) + (size_t)r * sizeof(h), sizeof(h));
      void* p = nullptr;
      cuda_check(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess), "ipc open");
      bases[(size_t)r] = static_cast<unsigned char*>(p);
    }
    c->cl.own_peers = false;
    cl_connect(c, bases);
  });
}

void* dvsg_cluster_comm_arena(dvsg_ctx* c) { return c && c->cl.active ? c->cl.arena : nullptr; }

dvsg_status dvsg_cluster_comm_connect_local(dvsg_ctx* c, void* const* arenas) {
  return guarded([&] {
    set_device(c);
    if (!c->cl.active) fail(DVSG_EINVAL, "cluster_comm_connect: call dvsg_cluster_comm_init first");
    std::vector<unsigned char*> bases((size_t)c->cl.nranks);
    for (int r = 0; r < c->cl.nranks; ++r) bases[(size_t)r] = static_cast<unsigned char*>(arenas[r]);
    c->cl.own_peers = true;
    cl_connect(c, bases);
  });
}

dvsg_status dvsg_run_pipeline_cluster_device(dvsg_ctx* c, const float* d_q, uint64_t nq, int dim,
                                             const dvsg_search_params* p, int fanout, uint32_t* d_ids,
                                             float* d_dists, uint32_t* d_count, float* d_vectors,
                                             uint64_t* d_visited_total) {
  return guarded([&] {
    set_device(c);
    auto& cl = c->cl;
    if (!cl.active || !cl.connected) fail(DVSG_EINVAL, "cluster exchange: call dvsg_cluster_comm_init / connect first");
    cl_check(c);  // errors of the previous step
    validate_params(p);
    if (dim != c->dim) fail(DVSG_EINVAL, "run_pipeline: query dim %d != index dim %d", dim, c->dim);
    if (fanout < 1 || fanout > c->clusters)
      fail(DVSG_EINVAL, "run_pipeline: fanout %d out of range for %d clusters", fanout, c->clusters);
    if (fanout > cl.max_fanout || nq > cl.max_queries || p->k != cl.k)
      fail(DVSG_EINVAL, "cluster exchange: batch (nq %llu, fanout %d, k %d) exceeds the arena (%llu, %d, %d)",
           (unsigned long long)nq, fanout, p->k, (unsigned long long)cl.max_queries, cl.max_fanout, cl.k);
    if (d_vectors && !cl.with_vectors) fail(DVSG_EINVAL, "cluster exchange: arena built without hit vectors");
    sync_slots(c);
    if (cl.with_vectors) build_locator(c);
    const dvsg::ClArena mine = cl_view(c, cl.arena);
    const uint64_t nu = nq * (uint64_t)fanout;
    cudaStream_t s = c->stream;
    c->err_flag.reserve(1, s);
    cuda_check(cudaMemsetAsync(c->err_flag.p, 0, sizeof(int), s), "err reset");
    // assign (K5) -> dispatch (K3, peer stores) -> barrier
    c->assign.reserve(std::max<uint64_t>(nu, 1), s);
    c->assign_scratch.reserve(dvsg::assign_scratch_words(nq, dim, c->clusters, fanout), s);
    if (nq) cuda_check(dvsg::launch_assign(d_q, nq, dim, c->d_cents.p, c->d_cent_norms.p, c->clusters, fanout,
                                           c->assign.p, c->assign_scratch.p, s, &c->assign_path), "assign");
    cuda_check(dvsg::launch_cl_dispatch(c->cl_peers.p, cl.nranks, cl.rank, cl.parity, d_q, nq, dim, fanout,
                                        c->assign.p, c->cl_place.p, (uint32_t)c->clusters, cl.cap, c->cl_err.p, s),
               "dispatch");
    cuda_check(dvsg::launch_cl_barrier(c->cl_peers.p, cl.nranks, cl.rank, ++cl.epoch, c->cl_err.p, s), "barrier");
    cuda_check(dvsg::launch_cl_reset(c->cl_peers.p, cl.rank, cl.parity, s), "reset");
    // owner: the units in this rank's inbox -> K1 -> replies (peer stores) -> barrier
    cuda_check(dvsg::launch_cl_units(c->cl_peers.p, cl.nranks, cl.rank, cl.parity, cl.cap, c->d_cluster_slot.p,
                                     c->slot_map_n, c->cl_uq.p, c->cl_up.p, c->cl_nunits.p, c->cl_err.p, s), "units");
    const uint64_t max_units = (uint64_t)cl.nranks * cl.cap;
    search_units(c, mine.inbox_q, max_units, dim, c->cl_uq.p, c->cl_up.p, max_units, p, c->cl_ids.p,
                 c->cl_dists.p, c->cl_count.p, c->cl_vis.p, c->cl_nunits.p);
    cuda_check(dvsg::launch_cl_reply(c->cl_peers.p, cl.rank, cl.cap, c->cl_uq.p, c->cl_nunits.p, max_units, p->k,
                                     c->cl_ids.p, c->cl_dists.p, c->cl_count.p, c->cl_vis.p,
                                     cl.with_vectors ? c->d_locator.p : nullptr, c->vec.p, dim, c->dpad,
                                     cl.with_vectors ? 1 : 0, s), "reply");
    cuda_check(dvsg::launch_cl_barrier(c->cl_peers.p, cl.nranks, cl.rank, ++cl.epoch, c->cl_err.p, s), "barrier");
    // origin: combine (K4) over the replies in unit order, hit vectors, visited_total
    if (nq) {
      cuda_check(dvsg::launch_combine(nq, fanout, mine.r_ids, mine.r_dists, mine.r_count, p->k, p->k, d_ids, d_dists,
                                      d_count, c->err_flag.p, s), "combine");
      if (d_vectors)
        cuda_check(dvsg::launch_cl_pick_vectors(d_ids, d_count, nq, p->k, fanout, mine.r_ids, mine.r_count,
                                                mine.r_vec, dim, d_vectors, s), "pick vectors");
      if (d_visited_total) {
        cuda_check(cudaMemsetAsync(d_visited_total, 0, 8, s), "visited reset");
        cuda_check(dvsg::launch_reduce_u64(mine.r_visited, nu, reinterpret_cast<unsigned long long*>(d_visited_total), s), "visited");
      }
    }
    c->launches += 9;
    cl.parity ^= 1;
  });
}

dvsg_status dvsg_cluster_comm_check(dvsg_ctx* c) {
  return guarded([&] {
    set_device(c);
    cl_check(c);
  });
}

dvsg_status dvsg_set_shard_exchange(dvsg_ctx* c, int mode) {
  return guarded([&] {
    if (mode < 0 || mode > 2) fail(DVSG_EINVAL, "set_shard_exchange: mode %d (0 bulk, 1 fused, 2 nccl)", mode);
    c->shard_exchange = mode;
  });
}

dvsg_status dvsg_nccl_unique_id(dvsg_ctx* c, void* out128) {
  return guarded([&] {
    (void)c;
    ncclUniqueId id;
    nccl_check(nccl_api().get_unique_id(&id), "ncclGetUniqueId");
    std::memcpy(out128, &id, sizeof id);
  });
}

dvsg_status dvsg_nccl_connect(dvsg_ctx* c, const void* id128) {
  return guarded([&] {
    set_device(c);
    if (!c->sh.active) fail(DVSG_EINVAL, "nccl_connect: call dvsg_shard_init first");
    if (c->nccl) {
      nccl_api().comm_destroy(c->nccl);
      c->nccl = nullptr;
    }
    ncclUniqueId id;
    std::memcpy(&id, id128, sizeof id);
    nccl_check(nccl_api().comm_init_rank(&c->nccl, c->sh.nranks, id, c->sh.rank), "ncclCommInitRank");
  });
}

dvsg_status dvsg_last_pipeline_timeline(dvsg_ctx* c, double* out, int max_microbatches, int* n_out) {
  return guarded([&] {
    set_device(c);
    *n_out = 0;
    if (!c->tl_mb) return;
    cuda_check(cudaEventSynchronize(c->tl_ev[6 * c->tl_mb]), "timeline");
    const int m = std::min(c->tl_mb, max_microbatches);
    for (int i = 0; i < m; ++i)
      for (int e = 0; e < 6; ++e) {
        float ms = 0;
        cuda_check(cudaEventElapsedTime(&ms, c->tl_ev[0], c->tl_ev[1 + 6 * i + e]), "elapsed");
        out[6 * i + e] = ms;
      }
    *n_out = m;
  });
}

dvsg_status dvsg_last_sharded_timeline(dvsg_ctx* c, double* out, int max_intervals, int* n_out) {
  return guarded([&] {
    set_device(c);
    *n_out = 0;
    const int n = std::min((int)c->xg_tl.size(), max_intervals);
    if (n == 0) return;
    cuda_check(cudaEventSynchronize(c->xg_tl_ev[2 * (c->xg_tl.size() - 1) + 1]), "timeline");
    for (int i = 0; i < n; ++i) {
      float a = 0, b = 0;
      cuda_check(cudaEventElapsedTime(&a, c->xg_tl_ev[0], c->xg_tl_ev[2 * i]), "elapsed");
      cuda_check(cudaEventElapsedTime(&b, c->xg_tl_ev[0], c->xg_tl_ev[2 * i + 1]), "elapsed");
      out[3 * i] = c->xg_tl[(size_t)i];
      out[3 * i + 1] = a;
      out[3 * i + 2] = b;
    }
    *n_out = n;
  });
}

dvsg_status dvsg_set_timing(dvsg_ctx* c, int enabled) {
  return guarded([&] { c->timing = enabled != 0; });
}

dvsg_status dvsg_last_timings(dvsg_ctx* c, float* search_ms, float* assign_ms, float* combine_ms, float* total_ms) {
  return guarded([&] {
    if (c->timing_pending) read_timings(c, c->timing_pending == 2);
    if (search_ms) *search_ms = c->t_search;
    if (assign_ms) *assign_ms = c->t_assign;
    if (combine_ms) *combine_ms = c->t_combine;
    if (total_ms) *total_ms = c->t_total;
  });
}

uint64_t dvsg_kernel_launches(dvsg_ctx* c) { return c ? c->launches.load() : 0; }

dvsg_status dvsg_set_vector_storage(dvsg_ctx* c, int mode) {
  return guarded([&] {
    set_device(c);
    if (mode == DVSG_STORAGE_F32) {
      c->want_u8 = false;
      return;
    }
    if (mode != DVSG_STORAGE_U8) fail(DVSG_EINVAL, "set_vector_storage: unknown mode %d", mode);
    if (c->rows == 0) fail(DVSG_EINVAL, "set_vector_storage: no resident rows");
    if (c->sh.active) fail(DVSG_EINVAL, "set_vector_storage: U8 serves the whole-graph search only");
    if (c->dpad > 256) fail(DVSG_EINVAL, "set_vector_storage: U8 needs dim <= 256");
    const uint64_t n = c->rows * (uint64_t)c->dpad;
    c->vec8.reserve(n, c->stream);
    c->err_flag.reserve(1, c->stream);
    cuda_check(cudaMemsetAsync(c->err_flag.p, 0, sizeof(int), c->stream), "err reset");
    cuda_check(dvsg::launch_to_u8(c->vec.p, n, c->vec8.p, c->err_flag.p, c->stream), "to u8");
    c->launches += 1;
    int bad = 0;
    cuda_check(cudaMemcpyAsync(&bad, c->err_flag.p, sizeof(int), cudaMemcpyDeviceToHost, c->stream), "flag");
    cuda_check(cudaStreamSynchronize(c->stream), "to u8");
    if (bad) fail(DVSG_EINVAL, "set_vector_storage: U8 needs every coordinate to be an integer in [0, 255]");
    c->want_u8 = true;
    c->u8_gen = c->vec_gen;
  });
}

dvsg_status dvsg_last_knn_info(dvsg_ctx* c, int* exact_mode, uint64_t* fallbacks) {
  return guarded([&] {
    if (exact_mode) *exact_mode = c->knn_exact;
    if (fallbacks) *fallbacks = c->knn_exact == 1 ? c->knn_fallbacks : 0;
  });
}

dvsg_status dvsg_last_assign_info(dvsg_ctx* c, int* path, uint64_t* fallbacks) {
  return guarded([&] {
    if (path) *path = c->assign_path;
    if (fallbacks) {
      *fallbacks = 0;
      if (c->assign_path == 2) {
        uint32_t n = 0;
        cuda_check(cudaStreamSynchronize(c->stream), "assign info");
        cuda_check(cudaMemcpy(&n, c->assign_scratch.p, sizeof(n), cudaMemcpyDeviceToHost), "assign info");
        *fallbacks = n;
      }
    }
  });
}

dvsg_status dvsg_debug_counters(dvsg_ctx* c, uint64_t* out16) {
  return guarded([&] {
    set_device(c);
    if (!c->counter.p) fail(DVSG_EINVAL, "no search launched yet");
    cuda_check(cudaMemcpyAsync(out16, c->counter.p, 16 * sizeof(uint64_t), cudaMemcpyDeviceToHost, c->stream), "counters");
    cuda_check(cudaStreamSynchronize(c->stream), "counters");
  });
}

dvsg_status dvsg_last_search_stats(dvsg_ctx* c, uint64_t* units, uint64_t* visited, uint64_t* expanded) {
  return guarded([&] {
    set_device(c);
    if (c->stats_pending) {
      cuda_check(cudaMemcpyAsync(c->last_stats, c->counter.p + 1, 3 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, c->stream), "stats");
      cuda_check(cudaStreamSynchronize(c->stream), "stats");
      c->stats_pending = false;
    }
    if (units) *units = c->last_stats[0];
    if (visited) *visited = c->last_stats[1];
    if (expanded) *expanded = c->last_stats[2];
  });
}

// ---- FNSY v1 -------------------------------------------------------------
dvsg_status dvsg_load_index_file(dvsg_ctx* c, const char* path, int rank) {
  return guarded([&] {
    set_device(c);
    FileReader r(path);
    char magic[4];
    if (!r.read(magic, 4) || std::memcmp(magic, "FNSY", 4) != 0) fail(DVSG_EFORMAT, "index file: bad magic (expected FNSY) (byte offset 0)");
    unsigned char vb[4];
    if (!r.read(vb, 4) || ((uint32_t)vb[0] | ((uint32_t)vb[1] << 8) | ((uint32_t)vb[2] << 16) | ((uint32_t)vb[3] << 24)) != 1u)
      fail(DVSG_EFORMAT, "index file: unsupported version (byte offset 4)");
    // scan section headers (index_file.cpp:164-195)
    Section secs[6] = {};
    bool have[6] = {};
    static const char* names[6] = {"", "centroids", "placement", "global ids", "adjacency", "vectors"};
    uint64_t off = 8;
    for (;;) {
      unsigned char h[12];
      const size_t got = std::fread(h, 1, 12, r.f);
      if (got == 0) break;
      if (got < 4) fail(DVSG_EFORMAT, "index file: truncated section header (byte offset %llu)", (unsigned long long)off);
      if (got < 12) fail(DVSG_EFORMAT, "index file: truncated section length (byte offset %llu)", (unsigned long long)(off + 4));
      uint32_t id = (uint32_t)h[0] | ((uint32_t)h[1] << 8) | ((uint32_t)h[2] << 16) | ((uint32_t)h[3] << 24);
      uint64_t len = 0;
      for (int i = 0; i < 8; ++i) len |= (uint64_t)h[4 + i] << (8 * i);
      if (id < 1 || id > 5) fail(DVSG_EFORMAT, "index file: unknown section id %u (byte offset %llu)", id, (unsigned long long)off);
      if (have[id]) fail(DVSG_EFORMAT, "index file: duplicate %s section (byte offset %llu)", names[id], (unsigned long long)off);
      if (fseeko(r.f, 0, SEEK_END) != 0) fail(DVSG_EFORMAT, "index file: seek failed");
      const uint64_t fsize = (uint64_t)ftello(r.f);
      if (off + 12 + len > fsize) fail(DVSG_EFORMAT, "index file: truncated section payload (byte offset %llu)", (unsigned long long)(off + 12));
      have[id] = true;
      secs[id] = Section{id, off + 12, len};
      off += 12 + len;
      r.seek(off);
    }
    for (uint32_t id = 1; id <= 5; ++id)
      if (!have[id]) fail(DVSG_EFORMAT, "index file: missing section id %u (byte offset %llu)", id, (unsigned long long)off);

    SecCursor cent(r, secs[1], names[1]);
    const uint32_t clusters = cent.u32();
    const uint32_t dim = cent.u32();
    if (clusters == 0 || dim == 0) fail(DVSG_EFORMAT, "index file: empty centroids section (byte offset %llu)", (unsigned long long)cent.offset());
    std::vector<float> centroids((size_t)clusters * dim);
    cent.bulk(centroids.data(), centroids.size() * 4);
    cent.expect_consumed();

    SecCursor plac(r, secs[2], names[2]);
    if (plac.u32() != clusters) fail(DVSG_EFORMAT, "index file: placement cluster count mismatch (byte offset %llu)", (unsigned long long)plac.offset());
    const uint32_t ranks = plac.u32();
    std::vector<uint32_t> placement(clusters);
    for (auto& x : placement) {
      x = plac.u32();
      if (x >= ranks) fail(DVSG_EFORMAT, "index file: placement rank out of range (byte offset %llu)", (unsigned long long)plac.offset());
    }
    plac.expect_consumed();

    SecCursor gid(r, secs[3], names[3]);
    if (gid.u32() != clusters) fail(DVSG_EFORMAT, "index file: global id cluster count mismatch (byte offset %llu)", (unsigned long long)gid.offset());
    std::vector<uint64_t> gid_off(clusters), sizes(clusters);
    for (uint32_t cl = 0; cl < clusters; ++cl) {
      sizes[cl] = gid.u32();
      gid_off[cl] = gid.offset();
      gid.skip(sizes[cl] * 4);
    }
    gid.expect_consumed();

    SecCursor adj(r, secs[4], names[4]);
    if (adj.u32() != clusters) fail(DVSG_EFORMAT, "index file: adjacency cluster count mismatch (byte offset %llu)", (unsigned long long)adj.offset());
    const uint32_t dg = adj.u32();
    if ((int32_t)dg < 1) fail(DVSG_EFORMAT, "index file: non-positive out-degree (byte offset %llu)", (unsigned long long)adj.offset());
    std::vector<uint64_t> adj_off(clusters);
    for (uint32_t cl = 0; cl < clusters; ++cl) {
      const uint32_t cnt = adj.u32();
      if (cnt != sizes[cl]) fail(DVSG_EFORMAT, "index file: adjacency node count mismatch in cluster %u (byte offset %llu)", cl, (unsigned long long)adj.offset());
      adj_off[cl] = adj.offset();
      adj.skip((uint64_t)cnt * dg * 4);
    }
    adj.expect_consumed();

    SecCursor vs(r, secs[5], names[5]);
    if (vs.u32() != clusters) fail(DVSG_EFORMAT, "index file: vector cluster count mismatch (byte offset %llu)", (unsigned long long)vs.offset());
    if (vs.u32() != dim) fail(DVSG_EFORMAT, "index file: vector dim mismatch (byte offset %llu)", (unsigned long long)vs.offset());
    std::vector<uint64_t> vec_off(clusters);
    for (uint32_t cl = 0; cl < clusters; ++cl) {
      const uint32_t cnt = vs.u32();
      if (cnt != sizes[cl]) fail(DVSG_EFORMAT, "index file: vector node count mismatch in cluster %u (byte offset %llu)", cl, (unsigned long long)vs.offset());
      vec_off[cl] = vs.offset();
      vs.skip((uint64_t)cnt * dim * 4);
    }
    vs.expect_consumed();
    for (uint32_t cl = 0; cl < clusters; ++cl)
      if (sizes[cl] == 0) fail(DVSG_EINVAL, "BuiltIndex: empty partition");

    // all structural checks passed: reset and upload the owned partitions
    c->parts.clear();
    c->part_mono.clear();
    c->all_integral = true;
    c->pend = dvsg_ctx::Pending{};
    c->rows = 0;
    c->vec_gen += 1;
    c->dim = c->dpad = c->dg = 0;
    c->parts_dirty = c->slot_dirty = c->locator_dirty = true;
    std::vector<float> v;
    std::vector<uint32_t> a, g;
    for (uint32_t cl = 0; cl < clusters; ++cl) {
      if (rank >= 0 && placement[cl] != (uint32_t)rank) continue;
      const uint64_t n = sizes[cl];
      v.resize(n * dim);
      a.resize(n * dg);
      g.resize(n);
      r.seek(gid_off[cl]);
      if (!r.read(g.data(), n * 4)) fail(DVSG_EFORMAT, "index file: truncated global ids section");
      r.seek(adj_off[cl]);
      if (!r.read(a.data(), n * dg * 4)) fail(DVSG_EFORMAT, "index file: truncated adjacency section");
      for (uint64_t i = 0; i < n * dg; ++i)
        if (a[i] >= n) fail(DVSG_EFORMAT, "index file: neighbor id out of range in cluster %u (byte offset %llu)", cl, (unsigned long long)(adj_off[cl] + 4 * i));
      r.seek(vec_off[cl]);
      if (!r.read(v.data(), n * dim * 4)) fail(DVSG_EFORMAT, "index file: truncated vectors section");
      const dvsg_status st = dvsg_load_partition(c, cl, n, (int)dim, (int)dg, v.data(), a.data(), g.data(), nullptr);
      if (st != DVSG_OK) fail(st, "%s", g_err.c_str());
    }
    const dvsg_status st = dvsg_set_centroids(c, centroids.data(), (int)clusters, (int)dim, placement.data(), (int)ranks);
    if (st != DVSG_OK) fail(st, "%s", g_err.c_str());
  });
}

dvsg_status dvsg_save_index_file(const char* path, int clusters, int dim, int out_degree,
                                 const float* centroids, const uint32_t* cluster_to_rank, int ranks,
                                 const uint64_t* offsets, const float* vectors,
                                 const uint32_t* adjacency, const uint32_t* global_ids) {
  return guarded([&] {
    if (clusters < 1 || dim < 1 || out_degree < 1 || ranks < 1) fail(DVSG_EINVAL, "BuiltIndex: index is not built");
    FILE* f = std::fopen(path, "wb");
    if (!f) fail(DVSG_EFORMAT, "cannot open %s for writing (byte offset 0)", path);
    std::unique_ptr<FILE, int (*)(FILE*)> guard(f, std::fclose);
    auto w = [&](const void* p, size_t n) {
      if (n && std::fwrite(p, 1, n, f) != n) fail(DVSG_EFORMAT, "write failure on %s (byte offset 0)", path);
    };
    auto section = [&](uint32_t id, const std::vector<unsigned char>& head, const std::vector<std::pair<const void*, uint64_t>>& bulk) {
      uint64_t len = head.size();
      for (auto& b : bulk) len += b.second;
      std::vector<unsigned char> h;
      put_u32(h, id);
      put_u32(h, (uint32_t)(len & 0xffffffffu));
      put_u32(h, (uint32_t)(len >> 32));
      w(h.data(), h.size());
      w(head.data(), head.size());
      for (auto& b : bulk) w(b.first, b.second);
    };
    w("FNSY", 4);
    std::vector<unsigned char> v;
    put_u32(v, 1);
    w(v.data(), 4);
    const uint32_t C = (uint32_t)clusters;
    std::vector<unsigned char> h;
    put_u32(h, C);
    put_u32(h, (uint32_t)dim);
    section(1, h, {{centroids, (uint64_t)C * dim * 4}});
    h.clear();
    put_u32(h, C);
    put_u32(h, (uint32_t)ranks);
    std::vector<uint32_t> plc(C);
    for (uint32_t i = 0; i < C; ++i) plc[i] = cluster_to_rank ? cluster_to_rank[i] : i % (uint32_t)ranks;
    section(2, h, {{plc.data(), (uint64_t)C * 4}});
    // per-cluster sections interleave a u32 count before each payload
    std::vector<std::vector<unsigned char>> counts(C);
    std::vector<std::pair<const void*, uint64_t>> bulk;
    for (uint32_t cl = 0; cl < C; ++cl) {
      put_u32(counts[cl], (uint32_t)(offsets[cl + 1] - offsets[cl]));
    }
    h.clear();
    put_u32(h, C);
    bulk.clear();
    for (uint32_t cl = 0; cl < C; ++cl) {
      bulk.push_back({counts[cl].data(), 4});
      bulk.push_back({global_ids + offsets[cl], (offsets[cl + 1] - offsets[cl]) * 4});
    }
    section(3, h, bulk);
    h.clear();
    put_u32(h, C);
    put_u32(h, (uint32_t)out_degree);
    bulk.clear();
    for (uint32_t cl = 0; cl < C; ++cl) {
      bulk.push_back({counts[cl].data(), 4});
      bulk.push_back({adjacency + offsets[cl] * (uint64_t)out_degree, (offsets[cl + 1] - offsets[cl]) * (uint64_t)out_degree * 4});
    }
    section(4, h, bulk);
    h.clear();
    put_u32(h, C);
    put_u32(h, (uint32_t)dim);
    bulk.clear();
    for (uint32_t cl = 0; cl < C; ++cl) {
      bulk.push_back({counts[cl].data(), 4});
      bulk.push_back({vectors + offsets[cl] * (uint64_t)dim, (offsets[cl + 1] - offsets[cl]) * (uint64_t)dim * 4});
    }
    section(5, h, bulk);
    if (std::fflush(f) != 0) fail(DVSG_EFORMAT, "write failure on %s (byte offset 0)", path);
  });
}

}  // extern "C"
