// ivf_build.cu -- device-side index construction at 10M-100M rows.
//
// K7 `range_topk_kernel`: per-row exact top-m (m <= 32) by (squared L2,
// column id) of blocks of <= 128 rows against a list of column ranges.  One
// kernel serves every n^2-shaped setup step of a large index:
//
//   * cluster-restricted kNN graph rows (the stand-in for build_graph,
//     /root/reference/proj/src/graph_index.cpp:46-97, at sizes where the
//     reference's O(n^2) exact build is 10^16 distance pairs): rows = the
//     members of one cluster, columns = the members of its P nearest
//     clusters, m = out_degree, self excluded, short lists repeated
//     cyclically like graph_index.cpp:86-92;
//   * nearest-centroid assignment for the clustering (m = 1) and the
//     cluster-neighbour lists (rows = centroids, columns = centroids);
//   * brute-force ground truth (topk.cpp:12-30) split over column ranges.
//
// Distances use the dot form |x|^2 + |y|^2 - 2 x.y in fp32 with per-row
// norms precomputed.  On integer-valued data (the SIFT-/Deep-like bench
// generator: bytes) every term is an integer below 2^24, so the distance is
// exact and equal to the reference's fp64-then-round squared_l2; on float
// data it is an fp32 approximation (fine for a build: both arms search the
// same graph).  Keys are ord(dist) << 32 | col, so ties break by id exactly
// like scored_less (dataset.hpp:33-46) and the result does not depend on
// the order in which survivors arrive.
//
// Tiling: 256 threads, 128 x 128 output tile, each thread an 8 x 8 register
// block (rows ty*4+i and 64+ty*4+i, columns tx*4+j and 64+tx*4+j, so the
// float4 reads of the transposed smem chunks are conflict-free), dims staged
// 32 at a time.  Epilogue per tile in two column halves: candidates below the
// row's current m-th key go to a per-row smem buffer (<= 64 per half, so it
// never overflows), then warp w merges rows 16w..16w+15 into register lists
// (lane i holds the i-th smallest key) and republishes the threshold.
//
// Also here: the exact device compute_entry_order (graph_index.cpp:21-44:
// fp64 column sums in row order, f32 mean, fp64 sequential squared_l2 per
// row, sort by (f32 dist, id)), deterministic segment means for the
// clustering, and the device-side validators of a partition (adjacency in
// range, finite, integer-valued).
#include <cstdint>
#include <cub/cub.cuh>
#include <cuda_runtime.h>

#include "dvsg_internal.h"

namespace dvsg {
namespace {

constexpr int TR = 128;   // rows per block
constexpr int TC = 128;   // columns per tile
constexpr int DC = 32;    // dims per staged chunk
constexpr int CAP = 64;   // survivor slots per row and half tile

__device__ __forceinline__ uint32_t f2ord(float f) {
  if (f == 0.0f) f = 0.0f;
  const uint32_t u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float ord2f(uint32_t o) {
  return __uint_as_float((o & 0x80000000u) ? (o & 0x7FFFFFFFu) : ~o);
}

__global__ void __launch_bounds__(256, 2)
range_topk_kernel(const float* __restrict__ rows, const float* __restrict__ rnorm,
                  const float* __restrict__ cols, const float* __restrict__ cnorm, int dpad,
                  const uint32_t* __restrict__ row_map, const RangeBlock* __restrict__ blocks,
                  const uint32_t* __restrict__ list_off, const uint2* __restrict__ ranges, int m, int flags,
                  uint32_t* __restrict__ out_ids, float* __restrict__ out_dists,
                  uint64_t out_stride) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  float (*xs)[TR] = reinterpret_cast<float (*)[TR]>(smem_raw);
  float (*ys)[TC] = reinterpret_cast<float (*)[TC]>(smem_raw + sizeof(float) * DC * TR);
  uint64_t (*cbuf)[CAP] =
      reinterpret_cast<uint64_t (*)[CAP]>(smem_raw + sizeof(float) * DC * (TR + TC));
  __shared__ int ccount[TR];
  __shared__ uint64_t thr[TR];
  __shared__ float rn[TR];
  __shared__ float cn[TC];
  __shared__ uint32_t prow[TR];  // physical row of each block row (row_map)

  const RangeBlock blk = blocks[blockIdx.x];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int tx = tid & 15, ty = tid >> 4;
  const int nrows = (int)blk.nrows;
  const uint64_t row0 = blk.row0;

  uint64_t top[16];
#pragma unroll
  for (int r = 0; r < 16; ++r) top[r] = ~0ull;
  if (tid < TR) {
    thr[tid] = ~0ull;
    ccount[tid] = 0;
    const uint32_t pr = tid < nrows ? (row_map ? row_map[row0 + tid] : (uint32_t)(row0 + tid)) : 0u;
    prow[tid] = pr;
    rn[tid] = tid < nrows ? rnorm[pr] : 0.f;
  }
  __syncthreads();
  if (flags & 4) {
    // continue from the lists already in the output (a previous pass over
    // other column ranges): the union's top-m, as if scanned in one launch
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      const int rl = warp * 16 + r;
      if (rl >= nrows) continue;
      const uint64_t o = ((flags & 8) ? (uint64_t)prow[rl] : (uint64_t)blk.out_row0 + (uint64_t)rl) * out_stride;
      uint64_t key = ~0ull;
      if (lane < m) {
        const uint32_t id = out_ids[o + lane];
        if (id != 0xFFFFFFFFu) key = ((uint64_t)f2ord(out_dists[o + lane]) << 32) | id;
      }
      top[r] = key;
      const uint64_t mth = __shfl_sync(0xFFFFFFFFu, key, m - 1);
      if (lane == 0) thr[rl] = mth;
    }
  }

  const uint32_t l0 = list_off[blk.list], l1 = list_off[blk.list + 1];
  for (uint32_t l = l0; l < l1; ++l) {
    const uint2 rg = ranges[l];
    for (uint32_t c0 = rg.x; c0 < rg.y; c0 += TC) {
      float acc[8][8];
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = 0.f;

      for (int d0 = 0; d0 < dpad; d0 += DC) {
        __syncthreads();
#pragma unroll
        for (int p = 0; p < 4; ++p) {
          const int idx = tid + p * 256;
          const int r = idx & (TR - 1), ch = idx >> 7;  // ch: float4 chunk 0..7
          const int dd = d0 + ch * 4;
          float4 vx = make_float4(0.f, 0.f, 0.f, 0.f), vy = vx;
          if (dd < dpad) {
            if (r < nrows) vx = __ldg(reinterpret_cast<const float4*>(rows + (uint64_t)prow[r] * dpad + dd));
            if (c0 + r < rg.y) vy = __ldg(reinterpret_cast<const float4*>(cols + (uint64_t)(c0 + r) * dpad + dd));
          }
          xs[ch * 4 + 0][r] = vx.x; xs[ch * 4 + 1][r] = vx.y;
          xs[ch * 4 + 2][r] = vx.z; xs[ch * 4 + 3][r] = vx.w;
          ys[ch * 4 + 0][r] = vy.x; ys[ch * 4 + 1][r] = vy.y;
          ys[ch * 4 + 2][r] = vy.z; ys[ch * 4 + 3][r] = vy.w;
        }
        if (d0 == 0 && tid < TC) cn[tid] = c0 + tid < rg.y ? cnorm[c0 + tid] : 0.f;
        __syncthreads();
#pragma unroll 8
        for (int d = 0; d < DC; ++d) {
          const float4 a0 = *reinterpret_cast<const float4*>(&xs[d][ty * 4]);
          const float4 a1 = *reinterpret_cast<const float4*>(&xs[d][64 + ty * 4]);
          const float4 b0 = *reinterpret_cast<const float4*>(&ys[d][tx * 4]);
          const float4 b1 = *reinterpret_cast<const float4*>(&ys[d][64 + tx * 4]);
          const float av[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
          const float bv[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
          for (int i = 0; i < 8; ++i)
#pragma unroll
            for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
        }
      }

      // epilogue: two column halves so a row never has more than CAP survivors
#pragma unroll
      for (int h = 0; h < 2; ++h) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int rl = i < 4 ? ty * 4 + i : 64 + ty * 4 + (i - 4);
          if (rl >= nrows) continue;
          const uint64_t t = thr[rl];
          const float nr = rn[rl];
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int cl = h * 64 + tx * 4 + j;
            const uint32_t col = c0 + (uint32_t)cl;
            if (col >= rg.y) continue;
            if ((flags & 1) && col == prow[rl]) continue;
            const float dist = fmaxf(fmaf(-2.f, acc[i][h * 4 + j], nr + cn[cl]), 0.f);
            const uint64_t key = ((uint64_t)f2ord(dist) << 32) | col;
            if (key < t) cbuf[rl][atomicAdd(&ccount[rl], 1)] = key;
          }
        }
        __syncthreads();
#pragma unroll
        for (int r = 0; r < 16; ++r) {
          const int rl = warp * 16 + r;
          const int cnt = ccount[rl];
          for (int c = 0; c < cnt; ++c) {
            const uint64_t key = cbuf[rl][c];
            const unsigned gt = __ballot_sync(0xFFFFFFFFu, top[r] > key);
            if (gt == 0) continue;
            const int pos = __ffs(gt) - 1;
            const uint64_t up = __shfl_up_sync(0xFFFFFFFFu, top[r], 1);
            if (lane > pos) top[r] = up;
            if (lane == pos) top[r] = key;
          }
          const uint64_t mth = __shfl_sync(0xFFFFFFFFu, top[r], m - 1);
          if (lane == 0) {
            if (cnt) thr[rl] = mth;
            ccount[rl] = 0;
          }
        }
        __syncthreads();
      }
    }
  }

  // emit
#pragma unroll
  for (int r = 0; r < 16; ++r) {
    const int rl = warp * 16 + r;
    if (rl >= nrows) continue;
    const uint64_t orow = (flags & 8) ? (uint64_t)prow[rl] : (uint64_t)blk.out_row0 + (uint64_t)rl;
    const unsigned valid_mask = __ballot_sync(0xFFFFFFFFu, top[r] != ~0ull);
    const int valid = __popc(valid_mask);
    if (flags & 2) {
      // build_graph semantics (graph_index.cpp:86-92): fewer than m
      // candidates repeat cyclically; none at all pads with the row itself
      const int nv = valid < m ? valid : m;
      for (int j = 0; j < m; ++j) {
        const uint64_t kj = __shfl_sync(0xFFFFFFFFu, top[r], nv > 0 ? j % nv : 0);
        if (lane == 0) {
          out_ids[orow * out_stride + j] = nv > 0 ? (uint32_t)kj : prow[rl];
          if (out_dists) out_dists[orow * out_stride + j] = nv > 0 ? ord2f((uint32_t)(kj >> 32)) : 0.f;
        }
      }
    } else if (lane < m) {
      const bool ok = top[r] != ~0ull;
      out_ids[orow * out_stride + lane] = ok ? (uint32_t)top[r] : 0xFFFFFFFFu;
      if (out_dists) out_dists[orow * out_stride + lane] = ok ? ord2f((uint32_t)(top[r] >> 32)) : __int_as_float(0x7F800000);
    }
  }
}

// fp32 squared norms (exact on integer data below 2^24)
__global__ void row_norms_kernel(const float* __restrict__ x, uint64_t n, int dpad,
                                 float* __restrict__ out) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const float4* r = reinterpret_cast<const float4*>(x + i * (uint64_t)dpad);
  float acc = 0.f;
  for (int c = 0; c < dpad / 4; ++c) {
    const float4 v = __ldg(r + c);
    acc = fmaf(v.x, v.x, acc);
    acc = fmaf(v.y, v.y, acc);
    acc = fmaf(v.z, v.z, acc);
    acc = fmaf(v.w, v.w, acc);
  }
  out[i] = acc;
}

// ---- compute_entry_order (graph_index.cpp:21-44), exact --------------------
// Column sums: fp64, each column summed in row order (the reference's order,
// so the rounding is identical on any data).  One CTA streams the rows through
// shared memory in whole-row tiles with a register prefetch of the next tile.
constexpr int MEAN_THREADS = 512;
constexpr int MEAN_TILE = MEAN_THREADS * 16;  // floats per tile (32 KB)

__global__ void __launch_bounds__(MEAN_THREADS, 1)
column_mean_kernel(const float* __restrict__ x, uint64_t n, int dim, int dpad,
                   float* __restrict__ mean_out) {
  __shared__ __align__(16) float tile[MEAN_TILE];
  const int tid = threadIdx.x;
  const uint64_t trows = (uint64_t)(MEAN_TILE / dpad);
  const uint64_t ntiles = (n + trows - 1) / trows;
  double acc0 = 0.0, acc1 = 0.0;  // columns tid and tid + 512
  float4 pre[4];
  auto load = [&](uint64_t t) {
    const uint64_t r0 = t * trows;
    const uint64_t rows_here = (r0 + trows <= n ? trows : n - r0);
    const uint64_t nf4 = rows_here * (uint64_t)dpad / 4;
    const float4* src = reinterpret_cast<const float4*>(x + r0 * (uint64_t)dpad);
#pragma unroll
    for (int p = 0; p < 4; ++p) {
      const uint64_t idx = (uint64_t)tid + (uint64_t)p * MEAN_THREADS;
      pre[p] = idx < nf4 ? __ldg(src + idx) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
  };
  if (ntiles) load(0);
  for (uint64_t t = 0; t < ntiles; ++t) {
    __syncthreads();
#pragma unroll
    for (int p = 0; p < 4; ++p) reinterpret_cast<float4*>(tile)[tid + p * MEAN_THREADS] = pre[p];
    __syncthreads();
    if (t + 1 < ntiles) load(t + 1);
    const uint64_t r0 = t * trows;
    const int rows_here = (int)(r0 + trows <= n ? trows : n - r0);
    if (tid < dim) {
      for (int r = 0; r < rows_here; ++r) acc0 += (double)tile[r * dpad + tid];
    }
    if (tid + MEAN_THREADS < dim) {
      for (int r = 0; r < rows_here; ++r) acc1 += (double)tile[r * dpad + tid + MEAN_THREADS];
    }
  }
  if (tid < dim) mean_out[tid] = (float)(acc0 / (double)n);
  if (tid + MEAN_THREADS < dim) mean_out[tid + MEAN_THREADS] = (float)(acc1 / (double)n);
}

// key[i] = bits(f32(sum_j ((double)x_ij - (double)mean_j)^2)) << 32 | i
// (dist >= 0, so the raw bits order like the value; ties by id)
__global__ void entry_keys_kernel(const float* __restrict__ x, uint64_t n, int dim, int dpad,
                                  const float* __restrict__ mean, uint64_t* __restrict__ keys) {
  extern __shared__ double mshared[];
  for (int j = threadIdx.x; j < dim; j += blockDim.x) mshared[j] = (double)mean[j];
  __syncthreads();
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const float* r = x + i * (uint64_t)dpad;
  double acc = 0.0;
  int j = 0;
  for (; j + 4 <= dim; j += 4) {
    const float4 v = __ldg(reinterpret_cast<const float4*>(r + j));
    double d = __dsub_rn((double)v.x, mshared[j]);
    acc = __dadd_rn(acc, __dmul_rn(d, d));
    d = __dsub_rn((double)v.y, mshared[j + 1]);
    acc = __dadd_rn(acc, __dmul_rn(d, d));
    d = __dsub_rn((double)v.z, mshared[j + 2]);
    acc = __dadd_rn(acc, __dmul_rn(d, d));
    d = __dsub_rn((double)v.w, mshared[j + 3]);
    acc = __dadd_rn(acc, __dmul_rn(d, d));
  }
  for (; j < dim; ++j) {
    const double d = __dsub_rn((double)r[j], mshared[j]);
    acc = __dadd_rn(acc, __dmul_rn(d, d));
  }
  keys[i] = ((uint64_t)__float_as_uint((float)acc) << 32) | (uint32_t)i;
}

__global__ void low_words_kernel(const uint64_t* __restrict__ keys, uint64_t n,
                                 uint32_t* __restrict__ out) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = (uint32_t)keys[i];
}

// ---- validators ------------------------------------------------------------
// bit 0: neighbour id >= n; bit 2: non-finite element; bit 4: not integer-valued
// (or |x| >= 2^24); bit 5: pad column not zero; bit 6: global ids not strictly increasing
__global__ void check_partition_kernel(const float* __restrict__ x, uint64_t n, int dim, int dpad,
                                       const uint32_t* __restrict__ adj, int dg,
                                       const uint32_t* __restrict__ gids, int* __restrict__ flag) {
  int f = 0;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n * (uint64_t)dpad; i += stride) {
    const float v = x[i];
    const int col = (int)(i % (uint64_t)dpad);
    if (col >= dim) {
      if (v != 0.f) f |= 32;
      continue;
    }
    if (!isfinite(v)) f |= 4;
    else if (!(v == rintf(v) && fabsf(v) < 16777216.f)) f |= 16;
  }
  if (adj)
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n * (uint64_t)dg; i += stride)
      if (adj[i] >= n) f |= 1;
  if (gids)
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x + 1; i < n; i += stride)
      if (gids[i] <= gids[i - 1]) f |= 64;
  f |= __reduce_or_sync(0xFFFFFFFFu, f);
  if (f && (threadIdx.x & 31) == 0) atomicOr(flag, f);
}

__global__ void iota_kernel(uint32_t* __restrict__ out, uint64_t n) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = (uint32_t)i;
}

// ---- deterministic segment means (clustering) ------------------------------
// cents[c] = f32(fp64 sum of rows idx[off[c]..off[c+1]) in order / count);
// empty segments keep their centroid.  One CTA per segment, threads over dims.
__global__ void segment_mean_kernel(const float* __restrict__ x, int dpad, const uint32_t* __restrict__ idx,
                                    const uint64_t* __restrict__ off, float* __restrict__ cents) {
  const uint32_t c = blockIdx.x;
  const uint64_t b = off[c], e = off[c + 1];
  if (b == e) return;
  for (int j = threadIdx.x; j < dpad; j += blockDim.x) {
    double acc = 0.0;
    uint64_t i = b;
    for (; i + 4 <= e; i += 4) {
      const uint64_t r0 = idx ? idx[i] : i, r1 = idx ? idx[i + 1] : i + 1;
      const uint64_t r2 = idx ? idx[i + 2] : i + 2, r3 = idx ? idx[i + 3] : i + 3;
      const float v0 = x[r0 * dpad + j], v1 = x[r1 * dpad + j], v2 = x[r2 * dpad + j], v3 = x[r3 * dpad + j];
      acc += (double)v0;
      acc += (double)v1;
      acc += (double)v2;
      acc += (double)v3;
    }
    for (; i < e; ++i) acc += (double)x[(idx ? idx[i] : i) * (uint64_t)dpad + j];
    cents[(uint64_t)c * dpad + j] = (float)(acc / (double)(e - b));
  }
}

}  // namespace

size_t range_topk_smem_bytes() {
  return sizeof(float) * DC * (TR + TC) + sizeof(uint64_t) * TR * CAP;
}

cudaError_t launch_range_topk(const float* rows, const float* rnorm, const float* cols,
                              const float* cnorm, int dpad, const uint32_t* row_map, const RangeBlock* blocks,
                              uint64_t nblocks, const uint32_t* list_off, const uint2* ranges,
                              int m, int flags, uint32_t* out_ids, float* out_dists,
                              uint64_t out_stride, cudaStream_t stream) {
  if (m < 1 || m > 32 || dpad % 4) return cudaErrorInvalidValue;
  if (nblocks == 0) return cudaSuccess;
  const size_t smem = range_topk_smem_bytes();
  cudaError_t e = cudaFuncSetAttribute(range_topk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  for (uint64_t b0 = 0; b0 < nblocks; b0 += 0x7FFFFFFFull) {
    const uint64_t nb = nblocks - b0 < 0x7FFFFFFFull ? nblocks - b0 : 0x7FFFFFFFull;
    range_topk_kernel<<<(unsigned)nb, 256, smem, stream>>>(rows, rnorm, cols, cnorm, dpad, row_map, blocks + b0,
                                                           list_off, ranges, m, flags, out_ids,
                                                           out_dists, out_stride);
  }
  return cudaGetLastError();
}

cudaError_t launch_row_norms(const float* x, uint64_t n, int dpad, float* out, cudaStream_t stream) {
  if (n == 0) return cudaSuccess;
  row_norms_kernel<<<(unsigned)((n + 255) / 256), 256, 0, stream>>>(x, n, dpad, out);
  return cudaGetLastError();
}

size_t entry_order_scratch_bytes(uint64_t n) {
  size_t temp = 0;
  cub::DeviceRadixSort::SortKeys(nullptr, temp, (const uint64_t*)nullptr, (uint64_t*)nullptr, (int64_t)n);
  return 2 * n * sizeof(uint64_t) + 256 + ((temp + 255) & ~(size_t)255) + 4096;
}

cudaError_t launch_entry_order(const float* x, uint64_t n, int dim, int dpad, void* scratch,
                               size_t scratch_bytes, uint32_t* out, cudaStream_t stream) {
  if (n == 0) return cudaSuccess;
  unsigned char* s = static_cast<unsigned char*>(scratch);
  uint64_t* keys = reinterpret_cast<uint64_t*>(s);
  uint64_t* sorted = keys + n;
  float* mean = reinterpret_cast<float*>(s + 2 * n * sizeof(uint64_t));
  unsigned char* temp = s + 2 * n * sizeof(uint64_t) + 4096;
  size_t temp_bytes = scratch_bytes - 2 * n * sizeof(uint64_t) - 4096;
  column_mean_kernel<<<1, MEAN_THREADS, 0, stream>>>(x, n, dim, dpad, mean);
  entry_keys_kernel<<<(unsigned)((n + 255) / 256), 256, sizeof(double) * dpad, stream>>>(x, n, dim, dpad, mean, keys);
  cudaError_t e = cub::DeviceRadixSort::SortKeys(temp, temp_bytes, keys, sorted, (int64_t)n, 0, 64, stream);
  if (e != cudaSuccess) return e;
  low_words_kernel<<<(unsigned)((n + 255) / 256), 256, 0, stream>>>(sorted, n, out);
  return cudaGetLastError();
}

cudaError_t launch_check_partition(const float* x, uint64_t n, int dim, int dpad, const uint32_t* adj,
                                   int dg, const uint32_t* gids, int* flag, cudaStream_t stream) {
  check_partition_kernel<<<4 * 148, 256, 0, stream>>>(x, n, dim, dpad, adj, dg, gids, flag);
  return cudaGetLastError();
}

cudaError_t launch_iota(uint32_t* out, uint64_t n, cudaStream_t stream) {
  if (n == 0) return cudaSuccess;
  iota_kernel<<<(unsigned)((n + 255) / 256), 256, 0, stream>>>(out, n);
  return cudaGetLastError();
}

cudaError_t launch_segment_means(const float* x, int dpad, const uint32_t* idx, const uint64_t* off,
                                 uint32_t nseg, float* cents, cudaStream_t stream) {
  if (nseg == 0) return cudaSuccess;
  segment_mean_kernel<<<nseg, dpad < 128 ? 128 : 256, 0, stream>>>(x, dpad, idx, off, cents);
  return cudaGetLastError();
}

}  // namespace dvsg
