// route_kernels.cu -- K5 assign, route, K4 combine, hit-vector gather.
//
//   K5 assign   : assign_top_c, /root/reference/proj/src/kmeans.cpp:243-280.
//                 The reference's own sequential fp64 dot / norm (kmeans.cpp
//                 :44-48 expanded_dist), so the f32 distances are bit-exact:
//                 C < 8: one warp per query, each lane owns whole centroids;
//                 C >= 8: register-tiled 64 x 64 fp64 tiles (same per-output
//                 accumulation order) + a per-lane top-c selection (SURVEY
//                 8f-3; 12x faster at C = 4096).
//   route       : router.cpp:52-79 -- one unit per (query, assigned cluster).
//   K4 combine  : combine_results, simulator.cpp:219-243.  One warp per query
//                 runs a <=32-way merge of the sorted partial lists on
//                 (dist, id) keys, dedups by id, truncates at k, and flags an
//                 unsorted partial (internal_error in the reference).
//   gather      : simulator.cpp:329-333 -- attach the hit vectors.
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

#include "dvsg_internal.h"

namespace dvsg {
namespace {

__device__ __forceinline__ uint32_t f2ord(float f) {
  if (f == 0.0f) f = 0.0f;
  const uint32_t u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

__device__ __forceinline__ float ord2f(uint32_t o) {
  const uint32_t u = (o & 0x80000000u) ? (o & 0x7FFFFFFFu) : ~o;
  return __uint_as_float(u);
}

__device__ __forceinline__ uint64_t warp_min_u64(uint64_t v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const uint64_t w = __shfl_xor_sync(0xFFFFFFFFu, v, o);
    v = w < v ? w : v;
  }
  return v;
}

// squared_norm, distance.cpp:44-50 (sequential fp64)
__device__ __forceinline__ double exact_sqnorm(const float* __restrict__ qp, int dim) {
  double qn = 0.0;
  for (int i = 0; i < dim; ++i) qn = __dadd_rn(qn, __dmul_rn((double)qp[i], (double)qp[i]));
  return qn;
}

// expanded_dist (kmeans.cpp:44-48) rounded to f32 and keyed (ord(dist) << 32 | cluster)
__device__ __forceinline__ uint64_t expanded_key(double qn, double cn, double dot, uint32_t j) {
  const double d = __dsub_rn(__dadd_rn(qn, cn), __dmul_rn(2.0, dot));
  const float f = (float)(d < 0.0 ? 0.0 : d);
  return ((uint64_t)f2ord(f) << 32) | j;
}

__device__ __forceinline__ uint64_t exact_key(const float* __restrict__ qp, const float* __restrict__ cp, int dim,
                                              double qn, double cn, uint32_t j) {
  double dot = 0.0;  // dot, distance.cpp:35-42 (sequential)
  for (int i = 0; i < dim; ++i) dot = __dadd_rn(dot, __dmul_rn((double)qp[i], (double)cp[i]));
  return expanded_key(qn, cn, dot, j);
}

// one query, one warp: keys into row[0..clusters), then c rounds of warp-min
// over keys strictly above the last selected one
__device__ __forceinline__ void assign_one(const float* __restrict__ qp, int dim, const float* __restrict__ cents,
                                           const double* __restrict__ cent_norms, int clusters, int c,
                                           uint64_t* __restrict__ row, uint32_t* __restrict__ out, int lane) {
  const double qn = exact_sqnorm(qp, dim);
  for (int j = lane; j < clusters; j += 32)
    row[j] = exact_key(qp, cents + (uint64_t)j * (uint64_t)dim, dim, qn, cent_norms[j], (uint32_t)j);
  __syncwarp();
  uint64_t last = 0;
  for (int r = 0; r < c; ++r) {
    uint64_t best = ~0ull;
    for (int j = lane; j < clusters; j += 32) {
      const uint64_t key = row[j];
      if ((r == 0 || key > last) && key < best) best = key;
    }
    best = warp_min_u64(best);
    if (lane == 0) out[r] = (uint32_t)best;
    last = best;
  }
  __syncwarp();
}

// scratch: nq x clusters keys (ord(dist) << 32 | cluster)
__global__ void assign_kernel(const float* __restrict__ queries, uint64_t nq, int dim,
                              const float* __restrict__ cents,
                              const double* __restrict__ cent_norms, int clusters, int c,
                              uint64_t* __restrict__ scratch, uint32_t* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const uint64_t q = (uint64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  if (q >= nq) return;
  assign_one(queries + q * (uint64_t)dim, dim, cents, cent_norms, clusters, c, scratch + q * (uint64_t)clusters,
             out + q * (uint64_t)c, lane);
}

// ---- K5 at large C: register-tiled fp64 "GEMM" with the reference's order --
// 64 queries x 64 centroids per CTA, 4 x 4 outputs per thread, k-chunks of
// 16 staged in smem as fp64.  Every output still accumulates its dot product
// over i = 0..dim-1 in order with separate round-to-nearest multiply and add
// (distance.cpp:35-42 as compiled for x86-64: no contraction), so the keys
// are bit-identical to assign_kernel's; only the data movement changes
// (coalesced tiles instead of 32 strided centroid rows per warp).
constexpr int kAT = 64, kAK = 16;

__global__ void qnorm_kernel(const float* __restrict__ queries, uint64_t nq, int dim,
                             double* __restrict__ qn) {
  const uint64_t q = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= nq) return;
  const float* qp = queries + q * (uint64_t)dim;
  double s = 0.0;  // squared_norm, distance.cpp:44-50 (sequential)
  for (int i = 0; i < dim; ++i) s = __dadd_rn(s, __dmul_rn((double)qp[i], (double)qp[i]));
  qn[q] = s;
}

__global__ void __launch_bounds__(256) assign_tile_kernel(const float* __restrict__ queries, uint64_t nq,
                                                          int dim, const float* __restrict__ cents,
                                                          const double* __restrict__ cent_norms,
                                                          int clusters, const double* __restrict__ qn,
                                                          uint64_t* __restrict__ scratch) {
  __shared__ double qs[kAK][kAT];
  __shared__ double cs[kAK][kAT];
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  const uint64_t q0 = (uint64_t)blockIdx.y * kAT;
  const int c0 = blockIdx.x * kAT;
  double acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;
  for (int k0 = 0; k0 < dim; k0 += kAK) {
    // 64 rows x 16 dims of each operand: thread loads 4 elements of each
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int e = tid + r * 256;  // 0..1023
      const int row = e >> 4, kk = e & 15;
      const int k = k0 + kk;
      const uint64_t q = q0 + row;
      qs[kk][row] = (q < nq && k < dim) ? (double)queries[q * (uint64_t)dim + k] : 0.0;
      const int cc = c0 + row;
      cs[kk][row] = (cc < clusters && k < dim) ? (double)cents[(uint64_t)cc * (uint64_t)dim + k] : 0.0;
    }
    __syncthreads();
    const int kn = dim - k0 < kAK ? dim - k0 : kAK;
    for (int kk = 0; kk < kn; ++kk) {
      double qv[4], cv[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) qv[i] = qs[kk][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) cv[j] = cs[kk][tx * 4 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = __dadd_rn(acc[i][j], __dmul_rn(qv[i], cv[j]));
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const uint64_t q = q0 + ty * 4 + i;
    if (q >= nq) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int cc = c0 + tx * 4 + j;
      if (cc >= clusters) continue;
      const double d = __dsub_rn(__dadd_rn(qn[q], cent_norms[cc]), __dmul_rn(2.0, acc[i][j]));
      const float f = (float)(d < 0.0 ? 0.0 : d);
      scratch[q * (uint64_t)clusters + cc] = ((uint64_t)f2ord(f) << 32) | (uint32_t)cc;
    }
  }
}

// top-c keys of each query row (c <= 32): per-lane sorted top-c in registers
// over a strided pass, then c rounds of warp-min over the lane heads.
template <int MC>
__global__ void select_topc_kernel(const uint64_t* __restrict__ scratch, uint64_t nq, int clusters,
                                   int c, uint32_t* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const uint64_t q = (uint64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  if (q >= nq) return;
  const uint64_t* row = scratch + q * (uint64_t)clusters;
  uint64_t top[MC];
#pragma unroll
  for (int r = 0; r < MC; ++r) top[r] = ~0ull;
  for (int j = lane; j < clusters; j += 32) {
    uint64_t key = row[j];
    if (key >= top[MC - 1]) continue;  // keeps the lane's MC >= c smallest
#pragma unroll
    for (int r = 0; r < MC; ++r) {  // insertion: carry the larger key down
      if (key < top[r]) {
        const uint64_t t = top[r];
        top[r] = key;
        key = t;
      }
    }
  }
  for (int r = 0; r < c; ++r) {
    const uint64_t best = warp_min_u64(top[0]);
    if (lane == 0) out[q * (uint64_t)c + r] = (uint32_t)best;
    if (top[0] == best) {  // keys are unique (cluster id in the low bits): one owner pops
#pragma unroll
      for (int s = 0; s < MC - 1; ++s) top[s] = top[s + 1];
      top[MC - 1] = ~0ull;
    }
  }
}

__global__ void route_kernel(const uint32_t* __restrict__ assign, uint64_t nq, int fanout,
                             const int32_t* __restrict__ cluster_to_slot, uint32_t nmap,
                             uint32_t* __restrict__ unit_query, uint32_t* __restrict__ unit_part,
                             int* err) {
  const uint64_t u = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (u >= nq * (uint64_t)fanout) return;
  const uint32_t cl = assign[u];
  const int32_t slot = cl < nmap ? cluster_to_slot[cl] : -1;  // unknown or non-resident cluster
  if (slot < 0) {
    atomicOr(err, 1);
    unit_part[u] = 0;
  } else {
    unit_part[u] = (uint32_t)slot;
  }
  unit_query[u] = (uint32_t)(u / (uint64_t)fanout);
}

__global__ void combine_kernel(uint64_t nq, int nparts, const uint32_t* __restrict__ ids,
                               const float* __restrict__ dists,
                               const uint32_t* __restrict__ counts, int stride, int k,
                               uint32_t* __restrict__ out_ids, float* __restrict__ out_dists,
                               uint32_t* __restrict__ out_count, int* err) {
  const int lane = threadIdx.x & 31;
  const uint64_t q = (uint64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  if (q >= nq) return;
  const uint64_t base = q * (uint64_t)nparts;
  // lane j < nparts owns partial list j
  uint32_t cnt = 0, head = 0;
  const uint32_t* li = nullptr;
  const float* ld = nullptr;
  if (lane < nparts) {
    cnt = counts[base + lane];
    li = ids + (base + lane) * (uint64_t)stride;
    ld = dists + (base + lane) * (uint64_t)stride;
    for (uint32_t i = 1; i < cnt; ++i) {
      const uint64_t a = ((uint64_t)f2ord(ld[i - 1]) << 32) | li[i - 1];
      const uint64_t b = ((uint64_t)f2ord(ld[i]) << 32) | li[i];
      if (b < a) atomicOr(err, 1);  // "partial list not sorted by (dist, id)"
    }
  }
  uint32_t* oi = out_ids + q * (uint64_t)k;
  float* od = out_dists + q * (uint64_t)k;
  int outn = 0;
  for (;;) {
    const uint64_t mine = head < cnt ? (((uint64_t)f2ord(ld[head]) << 32) | li[head]) : ~0ull;
    const uint64_t best = warp_min_u64(mine);
    if (best == ~0ull || outn >= k) break;
    // unique winner (keys unique across lanes unless equal (dist,id) pairs)
    const unsigned who = __ballot_sync(0xFFFFFFFFu, mine == best);
    const int src = __ffs(who) - 1;
    if (lane == src) ++head;
    const uint32_t id = (uint32_t)best;
    bool dup = false;
    for (int i = lane; i < outn; i += 32) dup |= (oi[i] == id);
    dup = __any_sync(0xFFFFFFFFu, dup);
    if (!dup) {
      if (lane == 0) {
        oi[outn] = id;
        od[outn] = ord2f((uint32_t)(best >> 32));
      }
      ++outn;
    }
    __syncwarp();
  }
  if (lane == 0) out_count[q] = (uint32_t)outn;
}

__global__ void gather_vectors_kernel(const uint32_t* __restrict__ ids,
                                      const uint32_t* __restrict__ counts, uint64_t nq, int k,
                                      const uint64_t* __restrict__ locator,
                                      const float* __restrict__ vectors, int dim, int dpad,
                                      float* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const uint64_t slot = (uint64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  if (slot >= nq * (uint64_t)k) return;
  const uint64_t q = slot / (uint64_t)k;
  const uint32_t h = (uint32_t)(slot - q * (uint64_t)k);
  if (h >= counts[q]) return;
  const uint64_t row = locator[ids[slot]];
  const float* src = vectors + row * (uint64_t)dpad;
  float* dst = out + slot * (uint64_t)dim;
  for (int i = lane; i < dim; i += 32) dst[i] = src[i];
}

// Dataset validate (dataset.cpp:18-33) on the device: flag bit 2 if any
// query element is non-finite, so the host need not scan the batch.
__global__ void check_finite_kernel(const float* __restrict__ x, uint64_t n, int* flag) {
  bool bad = false;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    bad |= !isfinite(x[i]);
  if (__any_sync(0xFFFFFFFFu, bad) && (threadIdx.x & 31) == 0) atomicOr(flag, 4);
}

// one warp per unit: nearest anchor (fp32, order-only) -> bucket; histogram
__global__ void anchor_bucket_kernel(const float* __restrict__ queries, int dim,
                                     const uint32_t* __restrict__ unit_query, uint64_t nunits,
                                     const float* __restrict__ anchors, int na, int dpad,
                                     uint32_t* __restrict__ bucket, uint32_t* __restrict__ hist) {
  const int lane = threadIdx.x & 31;
  const uint64_t u = (uint64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  if (u >= nunits) return;
  const float* q = queries + (uint64_t)unit_query[u] * (uint64_t)dim;
  float qv[8];
#pragma unroll
  for (int v = 0; v < 8; ++v) {
    const int i = lane + 32 * v;
    qv[v] = i < dim ? q[i] : 0.f;
  }
  float best = 3.4e38f;
  int besti = 0;
  for (int a = 0; a < na; ++a) {
    const float* av = anchors + (uint64_t)a * dpad;
    float acc = 0.f;
#pragma unroll
    for (int v = 0; v < 8; ++v) {
      const int i = lane + 32 * v;
      if (i < dim) {
        const float d = qv[v] - av[i];
        acc = fmaf(d, d, acc);
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xFFFFFFFFu, acc, o);
    if (acc < best) {
      best = acc;
      besti = a;
    }
  }
  if (lane == 0) {
    bucket[u] = (uint32_t)besti;
    atomicAdd(hist + besti, 1u);
  }
}

__global__ void exclusive_scan_small(uint32_t* __restrict__ hist, int n) {
  // single block; n <= 1024
  __shared__ uint32_t s[1024];
  const int t = threadIdx.x;
  s[t] = t < n ? hist[t] : 0u;
  __syncthreads();
  for (int off = 1; off < 1024; off <<= 1) {
    const uint32_t v = t >= off ? s[t - off] : 0u;
    __syncthreads();
    s[t] += v;
    __syncthreads();
  }
  if (t < n) hist[t] = t == 0 ? 0u : s[t - 1];
}

__global__ void bucket_scatter_kernel(const uint32_t* __restrict__ bucket, uint64_t nunits,
                                      uint32_t* __restrict__ offs, uint32_t* __restrict__ order) {
  const uint64_t u = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (u >= nunits) return;
  order[atomicAdd(offs + bucket[u], 1u)] = (uint32_t)u;
}

__global__ void reduce_u64_kernel(const uint64_t* __restrict__ in, uint64_t n,
                                  unsigned long long* out) {
  unsigned long long acc = 0;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    acc += in[i];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xFFFFFFFFu, acc, o);
  if ((threadIdx.x & 31) == 0 && acc) atomicAdd(out, acc);
}


// ---- K5 on the tensor cores ------------------------------------------------
// The reference's top-c by (f32(expanded_dist), id) is reproduced exactly:
//   1. centre queries and centroids on the centroid mean (fp32), pad to kpad;
//   2. K7 over TF32 (ivf_tc.cu, tcgen05 kind::tf32): the kTcM = 32 smallest
//      approximate squared distances per query;
//   3. re-rank those 32 with the reference's own fp64 arithmetic (exact_key),
//      warp bitonic sort, take c;
//   4. certificate: every non-candidate j had approx_j >= a_32 (the 32nd
//      approximate distance), and |approx - reference fp64 value| <= eps_q
//      (bound below), so if a_32 - eps_q >= nextafter(f_c) every
//      non-candidate's f32 key is strictly above the c-th selected one and the
//      selection is the reference's, ties included;
//   5. queries whose certificate fails go to a list that the exact warp kernel
//      (assign_one) finishes -- the result never depends on the approximation.
// eps_q: TF32 truncates each operand to 10 mantissa bits (|rel| < 2^-10), so
// |dot' - x'.c'| <= (2^-9 + (d+1) 2^-22) |x'||c'| (products exact in fp32,
// any-order fp32 accumulation with truncation); the fp32 norms and the
// epilogue add (d+6) 2^-22 (|x'|^2 + |c'|^2); centring in fp32 moves the true
// distance by <= 2^-21 (|x'| + |c'|)^2; the reference's fp64 expansion is
// within (d+3) 2^-51 (|x|^2 + |c|^2) of the true value.  eps_q doubles the sum.
constexpr int kTcM = 32;
constexpr int kTcMaxDim = 128;
constexpr int kTcMaxC = 24;
constexpr int kTcRows = 128;   // K7 rows per block
constexpr int kTcFbWarps = 512;

int tc_min_clusters() {
  static const int v = [] {
    const char* e = std::getenv("DVSG_ASSIGN_TC_MIN");
    return e ? std::atoi(e) : 256;
  }();
  return v;
}

bool use_tc(uint64_t nq, int dim, int clusters, int c) {
  const int mn = tc_min_clusters();
  return mn > 0 && clusters >= mn && clusters >= kTcM && dim <= kTcMaxDim && c <= kTcMaxC && nq > 0;
}

// scratch layout (256-byte aligned regions, in u64 words)
struct TcCarve {
  uint64_t fail_count, stats, mu, qp, qn2, cp, cn2, blocks, meta, cand_ids, cand_d, fail_list, fb_rows, total;
};

TcCarve tc_carve(uint64_t nq, int dim, int clusters) {
  const int kpad = (dim + 7) & ~7;
  const uint64_t nb = (nq + kTcRows - 1) / kTcRows;
  const uint64_t fbw = nq < (uint64_t)kTcFbWarps ? nq : (uint64_t)kTcFbWarps;
  TcCarve t{};
  uint64_t o = 0;
  auto take = [&](uint64_t bytes) {
    const uint64_t at = o;
    o += ((bytes + 255) / 256) * 32;
    return at;
  };
  t.fail_count = take(8);
  t.stats = take(4 * sizeof(double));
  t.mu = take((uint64_t)kpad * 4);
  t.qp = take(nq * (uint64_t)kpad * 4);
  t.qn2 = take(nq * 4);
  t.cp = take((uint64_t)clusters * kpad * 4);
  t.cn2 = take((uint64_t)clusters * 4);
  t.blocks = take(nb * sizeof(RangeBlock));
  t.meta = take(4 * sizeof(uint32_t) + sizeof(uint2));
  t.cand_ids = take(nq * kTcM * 4);
  t.cand_d = take(nq * kTcM * 4);
  t.fail_list = take(nq * 4);
  t.fb_rows = take(fbw * (uint64_t)clusters * 8);
  t.total = o;
  return t;
}

// centroid mean per column (fp64, in order), padded with zeros to kpad
__global__ void tc_mean_kernel(const float* __restrict__ cents, int clusters, int dim, int kpad,
                               float* __restrict__ mu) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= kpad) return;
  double s = 0.0;
  if (k < dim)
    for (int j = 0; j < clusters; ++j) s += (double)cents[(uint64_t)j * dim + k];
  mu[k] = k < dim ? (float)(s / clusters) : 0.f;
}

// warp per row: out = fl(x - mu) padded to kpad, n2 = |out|^2 in fp32
__global__ void tc_center_kernel(const float* __restrict__ x, uint64_t n, int dim, int kpad,
                                 const float* __restrict__ mu, float* __restrict__ out, float* __restrict__ n2) {
  const int lane = threadIdx.x & 31;
  const uint64_t r = (uint64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  if (r >= n) return;
  float acc = 0.f;
  for (int k = lane; k < kpad; k += 32) {
    const float v = k < dim ? __fsub_rn(x[r * dim + k], mu[k]) : 0.f;
    out[r * kpad + k] = v;
    acc = fmaf(v, v, acc);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xFFFFFFFFu, acc, o);
  if (lane == 0) n2[r] = acc;
}

// stats[0] = max centred |c'|^2, stats[1] = max reference |c|^2; the block
// list (one 128-row block per query tile, all over column list 0 = [0, C));
// zero the failure counter
__global__ void tc_setup_kernel(const float* __restrict__ cn2, const double* __restrict__ cent_norms, int clusters,
                                uint64_t nq, double* __restrict__ stats, RangeBlock* __restrict__ blocks,
                                uint32_t* __restrict__ meta, uint32_t* __restrict__ fail_count) {
  const uint64_t nb = (nq + kTcRows - 1) / kTcRows;
  for (uint64_t b = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; b < nb; b += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t r0 = b * kTcRows;
    blocks[b] = RangeBlock{(uint32_t)r0, (uint32_t)(nq - r0 < kTcRows ? nq - r0 : kTcRows), 0u, (uint32_t)r0};
  }
  if (blockIdx.x != 0) return;
  __shared__ double m0[32], m1[32];
  double a = 0.0, b = 0.0;
  for (int j = threadIdx.x; j < clusters; j += blockDim.x) {
    a = fmax(a, (double)cn2[j]);
    b = fmax(b, cent_norms[j]);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    a = fmax(a, __shfl_xor_sync(0xFFFFFFFFu, a, o));
    b = fmax(b, __shfl_xor_sync(0xFFFFFFFFu, b, o));
  }
  if ((threadIdx.x & 31) == 0) {
    m0[threadIdx.x >> 5] = a;
    m1[threadIdx.x >> 5] = b;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) {
      a = fmax(a, m0[w]);
      b = fmax(b, m1[w]);
    }
    stats[0] = a;
    stats[1] = b;
    meta[0] = 0;  // list_off = {0, 1}
    meta[1] = 1;
    reinterpret_cast<uint2*>(meta + 2)[0] = make_uint2(0u, (uint32_t)clusters);  // ranges[0]
    *fail_count = 0;
  }
}

__device__ __forceinline__ uint64_t warp_sort_u64(uint64_t v, int lane) {
#pragma unroll
  for (int k = 2; k <= 32; k <<= 1)
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1) {
      const uint64_t o = __shfl_xor_sync(0xFFFFFFFFu, v, j);
      const bool keep_min = ((lane & j) == 0) == ((lane & k) == 0);
      v = keep_min ? (o < v ? o : v) : (o > v ? o : v);
    }
  return v;
}

// warp per query: exact re-rank of the candidates + certificate.  Lane j
// scores candidate j; the 32 candidate rows are staged 32 dims at a time in
// shared memory by coalesced row loads (stride 33: conflict-free column
// reads), the query chunk is broadcast by shuffles, and every lane keeps the
// reference's sequential order (i = 0..dim-1) for the norm and the dot.
constexpr int kRerankWarps = 8;
__global__ void __launch_bounds__(32 * kRerankWarps)
tc_rerank_kernel(const float* __restrict__ queries, uint64_t nq, int dim, const float* __restrict__ cents,
                 const double* __restrict__ cent_norms, const float* __restrict__ qn2c,
                 const double* __restrict__ stats, const uint32_t* __restrict__ cand_ids,
                 const float* __restrict__ cand_d, int c, uint32_t* __restrict__ out,
                 uint32_t* __restrict__ fail_list, uint32_t* __restrict__ fail_count) {
  __shared__ float stage[kRerankWarps][32][33];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const uint64_t q = (uint64_t)blockIdx.x * kRerankWarps + wib;
  if (q >= nq) return;  // warp-uniform; the kernel has no block barrier
  float (*sw)[33] = stage[wib];
  const float* qp = queries + q * (uint64_t)dim;
  const uint32_t id = cand_ids[q * kTcM + lane];
  const uint32_t safe = id == 0xFFFFFFFFu ? 0u : id;
  double qn = 0.0, dot = 0.0;
  for (int i0 = 0; i0 < dim; i0 += 32) {
    const int w = dim - i0 < 32 ? dim - i0 : 32;
    const float qv = lane < w ? qp[i0 + lane] : 0.f;
#pragma unroll 8
    for (int j = 0; j < 32; ++j) {
      const uint32_t cj = __shfl_sync(0xFFFFFFFFu, safe, j);
      if (lane < w) sw[j][lane] = cents[(uint64_t)cj * dim + i0 + lane];
    }
    __syncwarp();
    for (int i = 0; i < w; ++i) {
      const double qi = (double)__shfl_sync(0xFFFFFFFFu, qv, i);
      qn = __dadd_rn(qn, __dmul_rn(qi, qi));  // squared_norm, distance.cpp:44-50
      dot = __dadd_rn(dot, __dmul_rn(qi, (double)sw[lane][i]));  // dot, distance.cpp:35-42
    }
    __syncwarp();
  }
  const uint64_t key = id == 0xFFFFFFFFu ? ~0ull : expanded_key(qn, cent_norms[id], dot, id);
  const uint64_t sorted = warp_sort_u64(key, lane);
  const uint64_t kc = __shfl_sync(0xFFFFFFFFu, sorted, c - 1);
  const uint32_t last_id = __shfl_sync(0xFFFFFFFFu, id, kTcM - 1);
  bool cert = last_id == 0xFFFFFFFFu;  // fewer than kTcM columns: every column is a candidate
  if (!cert && kc != ~0ull) {
    const double xn = sqrt((double)qn2c[q]), cm = sqrt(stats[0]), d = (double)dim;
    double eps = (0x1p-9 + (d + 1) * 0x1p-22) * 2.0 * xn * cm + (d + 6) * 0x1p-22 * (xn * xn + cm * cm) +
                 0x1p-21 * (xn + cm) * (xn + cm) + (d + 3) * 0x1p-51 * (qn + stats[1]);
    eps *= 2.0;
    const float fc = ord2f((uint32_t)(kc >> 32));
    const double lower = (double)cand_d[q * kTcM + kTcM - 1] - eps;
    // a non-finite bound (fp32 overflow of the approximate pass) never certifies
    cert = isfinite(lower) && lower >= (double)nextafterf(fc, __int_as_float(0x7F800000));
  }
  if (cert) {
    if (lane < c) out[q * (uint64_t)c + lane] = (uint32_t)sorted;
  } else if (lane == 0) {
    fail_list[atomicAdd(fail_count, 1u)] = (uint32_t)q;
  }
}

// the exact warp kernel over the rejected queries (device-side count)
__global__ void assign_list_kernel(const float* __restrict__ queries, int dim, const float* __restrict__ cents,
                                   const double* __restrict__ cent_norms, int clusters, int c,
                                   const uint32_t* __restrict__ list, const uint32_t* __restrict__ count,
                                   uint64_t* __restrict__ rows, uint32_t* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const uint32_t w = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  const uint32_t nw = gridDim.x * (blockDim.x / 32);
  const uint32_t n = *count;
  for (uint32_t i = w; i < n; i += nw) {
    const uint64_t q = list[i];
    assign_one(queries + q * (uint64_t)dim, dim, cents, cent_norms, clusters, c, rows + (uint64_t)w * clusters,
               out + q * (uint64_t)c, lane);
  }
}

cudaError_t launch_assign_tc(const float* queries, uint64_t nq, int dim, const float* cents,
                             const double* cent_norms, int clusters, int c, uint32_t* out, uint64_t* scratch,
                             cudaStream_t stream) {
  const int kpad = (dim + 7) & ~7;
  const TcCarve t = tc_carve(nq, dim, clusters);
  uint32_t* fail_count = reinterpret_cast<uint32_t*>(scratch + t.fail_count);
  double* stats = reinterpret_cast<double*>(scratch + t.stats);
  float* mu = reinterpret_cast<float*>(scratch + t.mu);
  float* qp = reinterpret_cast<float*>(scratch + t.qp);
  float* qn2 = reinterpret_cast<float*>(scratch + t.qn2);
  float* cp = reinterpret_cast<float*>(scratch + t.cp);
  float* cn2 = reinterpret_cast<float*>(scratch + t.cn2);
  RangeBlock* blocks = reinterpret_cast<RangeBlock*>(scratch + t.blocks);
  uint32_t* meta = reinterpret_cast<uint32_t*>(scratch + t.meta);
  uint32_t* cand_ids = reinterpret_cast<uint32_t*>(scratch + t.cand_ids);
  float* cand_d = reinterpret_cast<float*>(scratch + t.cand_d);
  uint32_t* fail_list = reinterpret_cast<uint32_t*>(scratch + t.fail_list);
  const uint64_t nb = (nq + kTcRows - 1) / kTcRows;
  const uint64_t fbw = nq < (uint64_t)kTcFbWarps ? nq : (uint64_t)kTcFbWarps;

  tc_mean_kernel<<<(kpad + 127) / 128, 128, 0, stream>>>(cents, clusters, dim, kpad, mu);
  tc_center_kernel<<<(unsigned)((clusters + 7) / 8), 256, 0, stream>>>(cents, clusters, dim, kpad, mu, cp, cn2);
  tc_center_kernel<<<(unsigned)((nq + 7) / 8), 256, 0, stream>>>(queries, nq, dim, kpad, mu, qp, qn2);
  const unsigned sg = (unsigned)((nb + 255) / 256);
  tc_setup_kernel<<<sg < 1184 ? sg : 1184, 256, 0, stream>>>(cn2, cent_norms, clusters, nq, stats, blocks, meta,
                                                              fail_count);
  cudaError_t e = launch_range_topk_tf32(qp, qn2, cp, cn2, kpad, nullptr, blocks, nb, meta,
                                         reinterpret_cast<const uint2*>(meta + 2), kTcM, 0, cand_ids, cand_d, kTcM,
                                         stream);
  if (e != cudaSuccess) return e;
  tc_rerank_kernel<<<(unsigned)((nq + kRerankWarps - 1) / kRerankWarps), 32 * kRerankWarps, 0, stream>>>(queries, nq, dim, cents, cent_norms, qn2, stats,
                                                                  cand_ids, cand_d, c, out, fail_list, fail_count);
  assign_list_kernel<<<(unsigned)((fbw + 7) / 8), 256, 0, stream>>>(queries, dim, cents, cent_norms, clusters, c,
                                                                    fail_list, fail_count, scratch + t.fb_rows, out);
  return cudaGetLastError();
}

}  // namespace

size_t assign_scratch_words(uint64_t nq, int dim, int clusters, int c) {
  if (use_tc(nq, dim, clusters, c)) return tc_carve(nq, dim, clusters).total;
  return (nq > 0 ? nq : 1) * ((uint64_t)clusters + 1);
}

cudaError_t launch_assign(const float* queries, uint64_t nq, int dim, const float* cents,
                          const double* cent_norms, int clusters, int c, uint32_t* out,
                          uint64_t* scratch, cudaStream_t stream, int* path) {
  if (nq == 0) return cudaSuccess;
  if (use_tc(nq, dim, clusters, c)) {
    if (path) *path = 2;
    return launch_assign_tc(queries, nq, dim, cents, cent_norms, clusters, c, out, scratch, stream);
  }
  static const int tiled_min = [] {
    const char* e = std::getenv("DVSG_ASSIGN_TILED_MIN");
    return e ? std::atoi(e) : 8;  // measured: tiled 9x faster already at C=64
  }();
  if (tiled_min > 0 && clusters >= tiled_min && c <= 32) {
    if (path) *path = 1;
    // scratch holds nq x clusters keys + nq query norms (host reserves both)
    double* qn = reinterpret_cast<double*>(scratch + nq * (uint64_t)clusters);
    qnorm_kernel<<<(unsigned)((nq + 255) / 256), 256, 0, stream>>>(queries, nq, dim, qn);
    const dim3 grid((unsigned)((clusters + kAT - 1) / kAT), (unsigned)((nq + kAT - 1) / kAT));
    assign_tile_kernel<<<grid, 256, 0, stream>>>(queries, nq, dim, cents, cent_norms, clusters, qn, scratch);
    const unsigned g = (unsigned)((nq + 7) / 8);
    if (c <= 4) select_topc_kernel<4><<<g, 256, 0, stream>>>(scratch, nq, clusters, c, out);
    else if (c <= 8) select_topc_kernel<8><<<g, 256, 0, stream>>>(scratch, nq, clusters, c, out);
    else if (c <= 16) select_topc_kernel<16><<<g, 256, 0, stream>>>(scratch, nq, clusters, c, out);
    else select_topc_kernel<32><<<g, 256, 0, stream>>>(scratch, nq, clusters, c, out);
    return cudaGetLastError();
  }
  if (path) *path = 0;
  const int wpb = 4;
  assign_kernel<<<(unsigned)((nq + wpb - 1) / wpb), 32 * wpb, 0, stream>>>(
      queries, nq, dim, cents, cent_norms, clusters, c, scratch, out);
  return cudaGetLastError();
}

cudaError_t launch_route(const uint32_t* assign, uint64_t nq, int fanout,
                         const int32_t* cluster_to_slot, uint32_t nmap, uint32_t* unit_query,
                         uint32_t* unit_part, int* err_flag, cudaStream_t stream) {
  const uint64_t n = nq * (uint64_t)fanout;
  if (n == 0) return cudaSuccess;
  route_kernel<<<(unsigned)((n + 255) / 256), 256, 0, stream>>>(assign, nq, fanout,
                                                                 cluster_to_slot, nmap, unit_query,
                                                                 unit_part, err_flag);
  return cudaGetLastError();
}

cudaError_t launch_combine(uint64_t nq, int nparts, const uint32_t* ids, const float* dists,
                           const uint32_t* counts, int stride, int k, uint32_t* out_ids,
                           float* out_dists, uint32_t* out_count, int* err_flag,
                           cudaStream_t stream) {
  if (nq == 0) return cudaSuccess;
  if (nparts < 1 || nparts > 32) return cudaErrorInvalidValue;
  const int wpb = 8;
  combine_kernel<<<(unsigned)((nq + wpb - 1) / wpb), 32 * wpb, 0, stream>>>(
      nq, nparts, ids, dists, counts, stride, k, out_ids, out_dists, out_count, err_flag);
  return cudaGetLastError();
}

cudaError_t launch_gather_vectors(const uint32_t* ids, const uint32_t* counts, uint64_t nq,
                                  int k, const uint64_t* locator, const float* vectors,
                                  int dim, int dpad, float* out, cudaStream_t stream) {
  const uint64_t n = nq * (uint64_t)k;
  if (n == 0) return cudaSuccess;
  const int wpb = 8;
  gather_vectors_kernel<<<(unsigned)((n + wpb - 1) / wpb), 32 * wpb, 0, stream>>>(
      ids, counts, nq, k, locator, vectors, dim, dpad, out);
  return cudaGetLastError();
}

cudaError_t launch_check_finite(const float* x, uint64_t n, int* flag, cudaStream_t stream) {
  if (n == 0) return cudaSuccess;
  uint64_t blocks = (n + 255) / 256;
  if (blocks > 1184) blocks = 1184;
  check_finite_kernel<<<(unsigned)blocks, 256, 0, stream>>>(x, n, flag);
  return cudaGetLastError();
}

cudaError_t launch_locality_order(const float* queries, int dim, const uint32_t* unit_query,
                                  uint64_t nunits, const float* anchors, int na, int dpad,
                                  uint32_t* scratch, uint32_t* order, cudaStream_t stream) {
  if (nunits == 0) return cudaSuccess;
  if (na < 1 || na > 1024 || dim > 256) return cudaErrorInvalidValue;
  uint32_t* bucket = scratch;
  uint32_t* hist = scratch + nunits;
  cudaError_t e = cudaMemsetAsync(hist, 0, sizeof(uint32_t) * (size_t)na, stream);
  if (e != cudaSuccess) return e;
  const int wpb = 8;
  anchor_bucket_kernel<<<(unsigned)((nunits + wpb - 1) / wpb), 32 * wpb, 0, stream>>>(
      queries, dim, unit_query, nunits, anchors, na, dpad, bucket, hist);
  exclusive_scan_small<<<1, 1024, 0, stream>>>(hist, na);
  bucket_scatter_kernel<<<(unsigned)((nunits + 255) / 256), 256, 0, stream>>>(bucket, nunits, hist,
                                                                             order);
  return cudaGetLastError();
}

cudaError_t launch_reduce_u64(const uint64_t* in, uint64_t n, unsigned long long* out,
                              cudaStream_t stream) {
  cudaError_t e = cudaMemsetAsync(out, 0, sizeof(unsigned long long), stream);
  if (e != cudaSuccess || n == 0) return e;
  uint64_t blocks = (n + 255) / 256;
  if (blocks > 1184) blocks = 1184;
  reduce_u64_kernel<<<(unsigned)blocks, 256, 0, stream>>>(in, n, out);
  return cudaGetLastError();
}

}  // namespace dvsg
