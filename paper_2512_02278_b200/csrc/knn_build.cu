// knn_build.cu -- K6: exact kNN graph rows on the GPU (build_graph,
// /root/reference/proj/src/graph_index.cpp:46-97).
//
// Row v = the out_degree nearest other nodes by (dist, id); partitions with
// n - 1 <= out_degree repeat the sorted list cyclically; a lone node pads
// with itself.  The distance is fp32 sum of (x - y)^2: exact (hence
// bit-identical to the reference's fp64-then-round) for integer-valued data
// whose squared norms stay below 2^24 (SIFT-like bytes at d <= 256), within
// fp32 rounding otherwise.
//
// Tiling: a CTA owns 64 rows and streams all n points in 64-column tiles;
// 256 threads each accumulate a 4x4 register block over d in 64-float
// chunks staged transposed in shared memory (conflict-free float4 reads).
// Survivors of the per-row cutoff (current 32nd key) go to a per-row smem
// buffer; one warp per row then inserts them into its register-resident
// sorted top list (lane i holds the i-th smallest key).
//
// Exact mode (any float data; build_graph / brute_force_topk bit-identical to
// the reference's fp64 squared_l2, distance.cpp:19-27): the tile pass keeps
// the 32 best fp32 candidates per row plus the smallest fp32 key of every
// column it did NOT keep (evicted, rejected by the list or by the cutoff);
// exact_rerank_kernel re-scores the 32 with the reference's sequential fp64
// sum, sorts them, and certifies the row when that lower bound, less the fp32
// error bound (d+4) 2^-24 relative, is at or above the next float after the
// deg-th exact distance -- then no column outside the 32 can reach the top
// deg, ties included.  Rows that fail go to a device list that
// exact_rows_kernel scans in fp64 against every column.
#include <algorithm>
#include <cstdint>
#include <cuda_runtime.h>

#include "dvsg_internal.h"

namespace dvsg {
namespace {

constexpr int TR = 64;     // rows per CTA
constexpr int TC = 64;     // columns per tile
constexpr int DC = 64;     // dims per smem chunk
constexpr int MAXDEG = 32; // out_degree handled by one warp-resident list

__device__ __forceinline__ uint32_t f2ord(float f) {
  if (f == 0.0f) f = 0.0f;
  const uint32_t u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

// rows x cols exact top-`deg` by (dist, id).  Graph build: rows == cols ==
// the partition, self excluded, tiny partitions cyclic (graph_index.cpp:46-97).
// Brute force (topk.cpp:12-30): rows = queries, cols = database.
template <bool EXACT>
__global__ void __launch_bounds__(256) knn_kernel(const float* __restrict__ rowv, uint64_t nrows,
                                                  const float* __restrict__ vec, uint64_t n,
                                                  int dpad, int deg, bool build,
                                                  uint32_t* __restrict__ adj,
                                                  float* __restrict__ out_dists,
                                                  uint64_t* __restrict__ lower) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  // transposed row / column chunks, then per-row survivors of this tile
  float (*xs)[TR] = reinterpret_cast<float (*)[TR]>(smem_raw);
  float (*ys)[TC] = reinterpret_cast<float (*)[TC]>(smem_raw + sizeof(float) * DC * TR);
  uint64_t (*cbuf)[TC] =
      reinterpret_cast<uint64_t (*)[TC]>(smem_raw + sizeof(float) * DC * (TR + TC));
  __shared__ int ccount[TR];
  __shared__ uint64_t cutoff[TR];
  __shared__ uint64_t rejf[EXACT ? TR : 1];  // exact: smallest key refused by the cutoff

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int tx = tid & 15, ty = tid >> 4;  // 16 x 16 threads, 4x4 outputs each
  const uint64_t r0 = (uint64_t)blockIdx.x * TR;

  // warp w owns rows w*8 .. w*8+7; lane i holds the i-th smallest key
  uint64_t top[8];
  uint64_t rejb[8];  // exact: smallest key the list evicted or refused (warp-uniform)
#pragma unroll
  for (int i = 0; i < 8; ++i) top[i] = rejb[i] = ~0ull;
  if (tid < TR) {
    cutoff[tid] = ~0ull;
    ccount[tid] = 0;
    if (EXACT) rejf[tid] = ~0ull;
  }
  const int keep = EXACT ? 32 : deg;  // list entries the cutoff protects

  for (uint64_t c0 = 0; c0 < n; c0 += TC) {
    float acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;

    for (int d0 = 0; d0 < dpad; d0 += DC) {
      __syncthreads();
      // stage: thread t loads row t%64, float4 chunk t/64 (+4 per pass)
      for (int pass = 0; pass < DC / 16; ++pass) {
        const int r = tid & 63, ch = (tid >> 6) + pass * 4;
        const int dd = d0 + ch * 4;
        float4 vx = make_float4(0.f, 0.f, 0.f, 0.f), vy = vx;
        if (dd < dpad) {
          if (r0 + r < nrows) vx = *reinterpret_cast<const float4*>(rowv + (r0 + r) * dpad + dd);
          if (c0 + r < n) vy = *reinterpret_cast<const float4*>(vec + (c0 + r) * dpad + dd);
        }
        xs[ch * 4 + 0][r] = vx.x; xs[ch * 4 + 1][r] = vx.y;
        xs[ch * 4 + 2][r] = vx.z; xs[ch * 4 + 3][r] = vx.w;
        ys[ch * 4 + 0][r] = vy.x; ys[ch * 4 + 1][r] = vy.y;
        ys[ch * 4 + 2][r] = vy.z; ys[ch * 4 + 3][r] = vy.w;
      }
      __syncthreads();
#pragma unroll 8
      for (int d = 0; d < DC; ++d) {
        const float4 a = *reinterpret_cast<const float4*>(&xs[d][ty * 4]);
        const float4 b = *reinterpret_cast<const float4*>(&ys[d][tx * 4]);
        const float av[4] = {a.x, a.y, a.z, a.w}, bv[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const float t = av[i] - bv[j];
            acc[i][j] = fmaf(t, t, acc[i][j]);
          }
      }
    }
    // cutoff filter -> per-row survivor buffers
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int rl = ty * 4 + i;
      const uint64_t row = r0 + rl;
      const uint64_t cut = cutoff[rl];
      uint64_t rmin = ~0ull;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint64_t col = c0 + tx * 4 + j;
        if (row < nrows && col < n && (!build || col != row)) {
          const uint64_t key = ((uint64_t)f2ord(acc[i][j]) << 32) | (uint32_t)col;
          if (key < cut) cbuf[rl][atomicAdd(&ccount[rl], 1)] = key;
          else if (EXACT) rmin = key < rmin ? key : rmin;
        }
      }
      if (EXACT) {  // min over the 16 threads of this row (a half warp), one writer
#pragma unroll
        for (int o = 8; o > 0; o >>= 1) {
          const uint64_t w = __shfl_xor_sync(0xFFFFFFFFu, rmin, o);
          rmin = w < rmin ? w : rmin;
        }
        if (tx == 0 && rmin < rejf[rl]) rejf[rl] = rmin;
      }
    }
    __syncthreads();
    // warp-resident sorted insertion
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int rl = warp * 8 + i;
      const int cnt = ccount[rl];
      for (int c = 0; c < cnt; ++c) {
        const uint64_t key = cbuf[rl][c];
        const unsigned gt = __ballot_sync(0xFFFFFFFFu, top[i] > key);
        if (gt == 0) {  // not among the 32 smallest
          if (EXACT && key < rejb[i]) rejb[i] = key;
          continue;
        }
        if (EXACT) {
          const uint64_t ev = __shfl_sync(0xFFFFFFFFu, top[i], 31);  // leaves the list
          if (ev < rejb[i]) rejb[i] = ev;
        }
        const int pos = __ffs(gt) - 1;
        const uint64_t up = __shfl_up_sync(0xFFFFFFFFu, top[i], 1);
        if (lane > pos) top[i] = up;
        if (lane == pos) top[i] = key;
      }
      const uint64_t last = __shfl_sync(0xFFFFFFFFu, top[i], keep - 1);
      if (lane == 0) {
        cutoff[rl] = last;
        ccount[rl] = 0;
      }
    }
    __syncthreads();
  }
  // emit rows (cyclic repeat for tiny partitions, graph_index.cpp:86-92)
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const uint64_t row = r0 + warp * 8 + i;
    if (row >= nrows) continue;
    if (EXACT) {  // the 32 candidates (0xFFFFFFFF: none) + the lower bound of the rest
      adj[row * 32ull + lane] = top[i] == ~0ull ? 0xFFFFFFFFu : (uint32_t)top[i];
      if (lane == 0) {
        const uint64_t f = rejf[warp * 8 + i];
        lower[row] = f < rejb[i] ? f : rejb[i];
      }
      continue;
    }
    if (!build) {  // brute force: the deg smallest (dist, id), k <= n checked on the host
      if (lane < deg) {
        adj[row * (uint64_t)deg + lane] = (uint32_t)top[i];
        const uint32_t o = (uint32_t)(top[i] >> 32);
        out_dists[row * (uint64_t)deg + lane] = __uint_as_float((o & 0x80000000u) ? (o & 0x7FFFFFFFu) : ~o);
      }
      continue;
    }
    const uint64_t valid = n - 1 < (uint64_t)deg ? n - 1 : (uint64_t)deg;
    for (int j = 0; j < deg; ++j) {
      const int src = valid > 0 ? (int)((uint64_t)j % valid) : 0;
      const uint32_t id = (uint32_t)__shfl_sync(0xFFFFFFFFu, top[i], src);
      // n == 1: the lone node pads with itself (local id 0)
      if (lane == 0) adj[row * (uint64_t)deg + j] = valid > 0 ? id : 0u;
    }
  }
}

__device__ __forceinline__ float ord2f(uint32_t o) {
  return __uint_as_float((o & 0x80000000u) ? (o & 0x7FFFFFFFu) : ~o);
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

// squared_l2 (distance.cpp:19-27): sequential fp64 sum of ((double)a - (double)b)^2
__device__ __forceinline__ double exact_sql2(const float* __restrict__ a, const float* __restrict__ b, int dim) {
  double acc = 0.0;
  for (int i = 0; i < dim; ++i) {
    const double t = __dsub_rn((double)a[i], (double)b[i]);
    acc = __dadd_rn(acc, __dmul_rn(t, t));
  }
  return acc;
}

// write row `row` from the sorted exact keys held by the warp (lane j = j-th)
__device__ __forceinline__ void emit_exact(uint64_t sorted, int nvalid, uint64_t row, int deg, bool build,
                                           uint32_t* __restrict__ out_ids, float* __restrict__ out_dists,
                                           int lane) {
  if (build) {
    // graph_index.cpp:70-92: deg nearest; tiny partitions repeat cyclically; a lone node pads with itself
    for (int j = 0; j < deg; ++j) {
      const int src = nvalid > 0 ? j % nvalid : 0;
      const uint64_t kj = __shfl_sync(0xFFFFFFFFu, sorted, src);
      if (lane == 0) out_ids[row * (uint64_t)deg + j] = nvalid > 0 ? (uint32_t)kj : 0u;
    }
  } else if (lane < deg) {
    out_ids[row * (uint64_t)deg + lane] = (uint32_t)sorted;
    out_dists[row * (uint64_t)deg + lane] = ord2f((uint32_t)(sorted >> 32));
  }
}

// Exact mode, warp per row: re-score the 32 fp32 candidates in fp64 (rows
// staged 32 dims at a time, stride 33: coalesced loads, conflict-free reads),
// sort, certify against the lower bound of the columns not kept.
constexpr int kRrWarps = 8;
__global__ void __launch_bounds__(32 * kRrWarps)
exact_rerank_kernel(const float* __restrict__ rowv, uint64_t nrows, const float* __restrict__ vec, uint64_t n,
                    int dim, int dpad, const uint32_t* __restrict__ cand, const uint64_t* __restrict__ lower,
                    int deg, bool build, uint32_t* __restrict__ out_ids, float* __restrict__ out_dists,
                    uint32_t* __restrict__ fail_list, uint32_t* __restrict__ fail_count) {
  __shared__ float stage[kRrWarps][32][33];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const uint64_t row = (uint64_t)blockIdx.x * kRrWarps + wib;
  if (row >= nrows) return;  // warp-uniform, no block barrier below
  float (*sw)[33] = stage[wib];
  const float* rp = rowv + row * (uint64_t)dpad;
  const uint32_t id = cand[row * 32ull + lane];
  const uint32_t safe = id == 0xFFFFFFFFu ? 0u : id;
  double acc = 0.0;
  for (int i0 = 0; i0 < dim; i0 += 32) {
    const int w = dim - i0 < 32 ? dim - i0 : 32;
    const float rv = lane < w ? rp[i0 + lane] : 0.f;
#pragma unroll 8
    for (int j = 0; j < 32; ++j) {
      const uint32_t cj = __shfl_sync(0xFFFFFFFFu, safe, j);
      if (lane < w) sw[j][lane] = vec[(uint64_t)cj * dpad + i0 + lane];
    }
    __syncwarp();
    for (int i = 0; i < w; ++i) {
      const double t = __dsub_rn((double)__shfl_sync(0xFFFFFFFFu, rv, i), (double)sw[lane][i]);
      acc = __dadd_rn(acc, __dmul_rn(t, t));
    }
    __syncwarp();
  }
  const uint64_t key = id == 0xFFFFFFFFu ? ~0ull : ((uint64_t)f2ord((float)acc) << 32) | id;
  const uint64_t sorted = warp_sort_u64(key, lane);
  const int nvalid = __popc(__ballot_sync(0xFFFFFFFFu, id != 0xFFFFFFFFu));
  const uint64_t others = build ? n - 1 : n;  // columns a row can take
  bool cert = others <= (uint64_t)nvalid;      // every column was a candidate
  if (!cert) {
    const uint64_t lb = lower[row];
    const uint64_t kd = __shfl_sync(0xFFFFFFFFu, sorted, deg - 1);
    if (lb != ~0ull && kd != ~0ull) {
      const double bound = (double)ord2f((uint32_t)(lb >> 32)) * (1.0 - (dim + 4) * 0x1p-24);
      const float fd = ord2f((uint32_t)(kd >> 32));
      cert = isfinite(bound) && bound >= (double)nextafterf(fd, __int_as_float(0x7F800000));
    }
  }
  if (cert) emit_exact(sorted, nvalid, row, deg, build, out_ids, out_dists, lane);
  else if (lane == 0) fail_list[atomicAdd(fail_count, 1u)] = (uint32_t)row;
}

// Exact fallback: a warp per rejected row scans every column in fp64 (per-lane
// sorted top-32, then deg rounds of warp-min).  Device-side count.
__global__ void __launch_bounds__(256) exact_rows_kernel(const float* __restrict__ rowv, const float* __restrict__ vec,
                                                         uint64_t n, int dim, int dpad, int deg, bool build,
                                                         const uint32_t* __restrict__ list,
                                                         const uint32_t* __restrict__ count,
                                                         uint32_t* __restrict__ out_ids, float* __restrict__ out_dists) {
  const int lane = threadIdx.x & 31;
  const uint32_t w = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  const uint32_t nw = gridDim.x * (blockDim.x / 32);
  const uint32_t cnt = *count;
  for (uint32_t it = w; it < cnt; it += nw) {
    const uint64_t row = list[it];
    const float* rp = rowv + row * (uint64_t)dpad;
    uint64_t top[MAXDEG];
#pragma unroll
    for (int r = 0; r < MAXDEG; ++r) top[r] = ~0ull;
    const double shrink = 1.0 - (dim + 4) * 0x1p-24;  // fp32 difference-form error bound (relative)
    for (uint64_t j = lane; j < n; j += 32) {
      if (build && j == row) continue;
      const float* cp = vec + j * (uint64_t)dpad;
      if (top[MAXDEG - 1] != ~0ull) {  // fp32 prefilter: skip columns that cannot enter this lane's list
        float a32 = 0.f;  // same arithmetic as the tiles (padding dims are 0 - 0)
        const float4* r4 = reinterpret_cast<const float4*>(rp);
        const float4* c4 = reinterpret_cast<const float4*>(cp);
        for (int i = 0; i < dpad / 4; ++i) {
          const float4 x = r4[i], y = __ldg(c4 + i);
          float t = x.x - y.x;
          a32 = fmaf(t, t, a32);
          t = x.y - y.y;
          a32 = fmaf(t, t, a32);
          t = x.z - y.z;
          a32 = fmaf(t, t, a32);
          t = x.w - y.w;
          a32 = fmaf(t, t, a32);
        }
        // exact > the lane's 32nd (strictly, so no tie can matter) -> skip
        if ((double)a32 * shrink >= (double)nextafterf(ord2f((uint32_t)(top[MAXDEG - 1] >> 32)),
                                                       __int_as_float(0x7F800000)))
          continue;
      }
      uint64_t key = ((uint64_t)f2ord((float)exact_sql2(rp, cp, dim)) << 32) | (uint32_t)j;
      if (key >= top[MAXDEG - 1]) continue;
#pragma unroll
      for (int r = 0; r < MAXDEG; ++r) {
        if (key < top[r]) {
          const uint64_t t = top[r];
          top[r] = key;
          key = t;
        }
      }
    }
    uint64_t mine = ~0ull;  // lane r ends with the r-th smallest
    for (int r = 0; r < MAXDEG; ++r) {
      uint64_t best = top[0];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const uint64_t x = __shfl_xor_sync(0xFFFFFFFFu, best, o);
        best = x < best ? x : best;
      }
      if (lane == r) mine = best;
      if (top[0] == best && best != ~0ull) {
#pragma unroll
        for (int s = 0; s < MAXDEG - 1; ++s) top[s] = top[s + 1];
        top[MAXDEG - 1] = ~0ull;
      }
    }
    const int nvalid = __popc(__ballot_sync(0xFFFFFFFFu, mine != ~0ull));
    emit_exact(mine, nvalid, row, deg, build, out_ids, out_dists, lane);
  }
}

}  // namespace

size_t knn_exact_scratch_bytes(uint64_t nrows) { return nrows * (32ull * 4 + 8 + 4) + 256; }

cudaError_t launch_knn_exact(const float* rowv, uint64_t nrows, const float* vec, uint64_t n, int dim, int dpad,
                             int deg, bool build, uint32_t* out_ids, float* out_dists, void* scratch,
                             cudaStream_t stream) {
  if (deg < 1 || deg > MAXDEG) return cudaErrorInvalidValue;
  if (nrows == 0) return cudaSuccess;
  unsigned char* p = static_cast<unsigned char*>(scratch);
  uint32_t* fail_count = reinterpret_cast<uint32_t*>(p);
  uint64_t* lower = reinterpret_cast<uint64_t*>(p + 256);
  uint32_t* cand = reinterpret_cast<uint32_t*>(lower + nrows);
  uint32_t* fail_list = cand + nrows * 32ull;
  cudaError_t e = cudaMemsetAsync(fail_count, 0, 4, stream);
  if (e != cudaSuccess) return e;
  const size_t smem = sizeof(float) * DC * (TR + TC) + sizeof(uint64_t) * TR * TC;
  e = cudaFuncSetAttribute(knn_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  knn_kernel<true><<<(unsigned)((nrows + TR - 1) / TR), 256, smem, stream>>>(rowv, nrows, vec, n, dpad, deg, build,
                                                                            cand, nullptr, lower);
  exact_rerank_kernel<<<(unsigned)((nrows + kRrWarps - 1) / kRrWarps), 32 * kRrWarps, 0, stream>>>(
      rowv, nrows, vec, n, dim, dpad, cand, lower, deg, build, out_ids, out_dists, fail_list, fail_count);
  exact_rows_kernel<<<(unsigned)std::min<uint64_t>((nrows + 7) / 8, 1184), 256, 0, stream>>>(
      rowv, vec, n, dim, dpad, deg, build, fail_list, fail_count, out_ids, out_dists);
  return cudaGetLastError();
}

cudaError_t launch_knn_build(const float* vectors, uint64_t n, int dim, int dpad,
                             int out_degree, uint32_t* adjacency, cudaStream_t stream) {
  (void)dim;
  if (out_degree < 1 || out_degree > MAXDEG) return cudaErrorInvalidValue;
  const uint64_t blocks = (n + TR - 1) / TR;
  const size_t smem = sizeof(float) * DC * (TR + TC) + sizeof(uint64_t) * TR * TC;
  cudaError_t e =
      cudaFuncSetAttribute(knn_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  knn_kernel<false><<<(unsigned)blocks, 256, smem, stream>>>(vectors, n, vectors, n, dpad, out_degree, true,
                                                             adjacency, nullptr, nullptr);
  return cudaGetLastError();
}

cudaError_t launch_brute_force(const float* queries, uint64_t nq, const float* db, uint64_t n,
                               int dpad, int k, uint32_t* out_ids, float* out_dists,
                               cudaStream_t stream) {
  if (k < 1 || k > MAXDEG || (uint64_t)k > n) return cudaErrorInvalidValue;
  const uint64_t blocks = (nq + TR - 1) / TR;
  const size_t smem = sizeof(float) * DC * (TR + TC) + sizeof(uint64_t) * TR * TC;
  cudaError_t e =
      cudaFuncSetAttribute(knn_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  knn_kernel<false><<<(unsigned)blocks, 256, smem, stream>>>(queries, nq, db, n, dpad, k, false, out_ids,
                                                             out_dists, nullptr);
  return cudaGetLastError();
}

}  // namespace dvsg
