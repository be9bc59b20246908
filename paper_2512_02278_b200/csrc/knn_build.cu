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
__global__ void __launch_bounds__(256) knn_kernel(const float* __restrict__ rowv, uint64_t nrows,
                                                  const float* __restrict__ vec, uint64_t n,
                                                  int dpad, int deg, bool build,
                                                  uint32_t* __restrict__ adj,
                                                  float* __restrict__ out_dists) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  // transposed row / column chunks, then per-row survivors of this tile
  float (*xs)[TR] = reinterpret_cast<float (*)[TR]>(smem_raw);
  float (*ys)[TC] = reinterpret_cast<float (*)[TC]>(smem_raw + sizeof(float) * DC * TR);
  uint64_t (*cbuf)[TC] =
      reinterpret_cast<uint64_t (*)[TC]>(smem_raw + sizeof(float) * DC * (TR + TC));
  __shared__ int ccount[TR];
  __shared__ uint64_t cutoff[TR];

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int tx = tid & 15, ty = tid >> 4;  // 16 x 16 threads, 4x4 outputs each
  const uint64_t r0 = (uint64_t)blockIdx.x * TR;

  // warp w owns rows w*8 .. w*8+7; lane i holds the i-th smallest key
  uint64_t top[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) top[i] = ~0ull;
  if (tid < TR) {
    cutoff[tid] = ~0ull;
    ccount[tid] = 0;
  }

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
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint64_t col = c0 + tx * 4 + j;
        if (row < nrows && col < n && (!build || col != row)) {
          const uint64_t key = ((uint64_t)f2ord(acc[i][j]) << 32) | (uint32_t)col;
          if (key < cut) cbuf[rl][atomicAdd(&ccount[rl], 1)] = key;
        }
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
        if (gt == 0) continue;  // not among the 32 smallest
        const int pos = __ffs(gt) - 1;
        const uint64_t up = __shfl_up_sync(0xFFFFFFFFu, top[i], 1);
        if (lane > pos) top[i] = up;
        if (lane == pos) top[i] = key;
      }
      const uint64_t last = __shfl_sync(0xFFFFFFFFu, top[i], deg - 1);
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

}  // namespace

cudaError_t launch_knn_build(const float* vectors, uint64_t n, int dim, int dpad,
                             int out_degree, uint32_t* adjacency, cudaStream_t stream) {
  (void)dim;
  if (out_degree < 1 || out_degree > MAXDEG) return cudaErrorInvalidValue;
  const uint64_t blocks = (n + TR - 1) / TR;
  const size_t smem = sizeof(float) * DC * (TR + TC) + sizeof(uint64_t) * TR * TC;
  cudaError_t e =
      cudaFuncSetAttribute(knn_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  knn_kernel<<<(unsigned)blocks, 256, smem, stream>>>(vectors, n, vectors, n, dpad, out_degree, true,
                                                      adjacency, nullptr);
  return cudaGetLastError();
}

cudaError_t launch_brute_force(const float* queries, uint64_t nq, const float* db, uint64_t n,
                               int dpad, int k, uint32_t* out_ids, float* out_dists,
                               cudaStream_t stream) {
  if (k < 1 || k > MAXDEG || (uint64_t)k > n) return cudaErrorInvalidValue;
  const uint64_t blocks = (nq + TR - 1) / TR;
  const size_t smem = sizeof(float) * DC * (TR + TC) + sizeof(uint64_t) * TR * TC;
  cudaError_t e =
      cudaFuncSetAttribute(knn_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  knn_kernel<<<(unsigned)blocks, 256, smem, stream>>>(queries, nq, db, n, dpad, k, false, out_ids,
                                                      out_dists);
  return cudaGetLastError();
}

}  // namespace dvsg
