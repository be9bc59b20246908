// kmeans.cu -- device parts of kmeans_train (/root/reference/proj/src/kmeans.cpp:189-241).
//
// The host (host.cpp, dvsg_kmeans_train) runs the reference's control flow --
// the mt19937_64 stream of init_kmeanspp (:150-187), the Lloyd loop with its
// fixed-point test (:216-226), repair_empty_clusters (:84-117) and the final
// non-empty check (:229-240) -- and the device does the O(n*C*d) work:
//
//   * kmeans++ distances: d2[i] = min(d2[i], (double)squared_l2(x_i, c)) with
//     squared_l2 summed in fp64 in dimension order (distance.cpp:19-27);
//   * the weighted pick: inclusive fp64 scan of d2 (cub) and the first index
//     whose prefix exceeds r (:167-175);
//   * assign_all / nearest_center (:50-82): the library's K5 assign kernel
//     (route_kernels.cu), which is the reference's expanded_dist bit for bit;
//   * update_means (:119-133): rows sorted stably by label (cub), then one
//     CTA per cluster summing its rows in row order in fp64 and scaling by
//     1.0 / count -- the reference's order and rounding;
//   * each row's squared_l2 to its own centroid (repair_empty_clusters and
//     compute_wcss, :135-143), summed on the host in row order.
//
// Exactness: everything but the kmeans++ scan is in the reference's order.
// The scan's prefix sums are exact when every d2 is an integer (integer-
// valued data, sums < 2^53), so kmeans_train is bit-identical to the
// reference there (tests/test_gpu_kmeans.py); on float data it matches
// unless a prefix lands within rounding of r.
#include <cstdint>
#include <cub/cub.cuh>
#include <cuda_runtime.h>

#include "dvsg_internal.h"

namespace dvsg {
namespace {

__device__ __forceinline__ float sq_l2_seq(const float* __restrict__ a, const float* __restrict__ b, int dim) {
  double acc = 0.0;
  for (int j = 0; j < dim; ++j) {
    const double d = __dsub_rn((double)a[j], (double)b[j]);
    acc = __dadd_rn(acc, __dmul_rn(d, d));
  }
  return (float)acc;
}

__global__ void kpp_d2_kernel(const float* __restrict__ x, uint64_t n, int dim, const float* __restrict__ c,
                              double* __restrict__ d2, int first) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double d = (double)sq_l2_seq(x + i * (uint64_t)dim, c, dim);
  if (first || d < d2[i]) d2[i] = d;
}

__global__ void first_gt_kernel(const double* __restrict__ scan, uint64_t n, double r,
                                unsigned long long* __restrict__ out) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n && scan[i] > r) atomicMin(out, (unsigned long long)i);
}

__global__ void own_dist_kernel(const float* __restrict__ x, uint64_t n, int dim, const float* __restrict__ cents,
                                const uint32_t* __restrict__ labels, float* __restrict__ out) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  out[i] = sq_l2_seq(x + i * (uint64_t)dim, cents + (uint64_t)labels[i] * dim, dim);
}

__global__ void iota_u32_kernel(uint32_t* __restrict__ out, uint64_t n) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = (uint32_t)i;
}

// cents[c] = f32(fp64 in-order sum of rows order[off[c]..off[c+1]) * (1.0 / count))
__global__ void cluster_means_kernel(const float* __restrict__ x, int dim, const uint32_t* __restrict__ order,
                                     const uint32_t* __restrict__ sorted_labels, uint64_t n,
                                     float* __restrict__ cents, int clusters) {
  const int c = blockIdx.x;
  // segment of cluster c in the sorted labels (binary search; labels < clusters)
  uint64_t lo = 0, hi = n;
  while (lo < hi) {
    const uint64_t mid = (lo + hi) >> 1;
    if (sorted_labels[mid] < (uint32_t)c) lo = mid + 1; else hi = mid;
  }
  const uint64_t b = lo;
  hi = n;
  while (lo < hi) {
    const uint64_t mid = (lo + hi) >> 1;
    if (sorted_labels[mid] <= (uint32_t)c) lo = mid + 1; else hi = mid;
  }
  const uint64_t e = lo;
  if (b == e) return;  // empty: repaired separately (kmeans.cpp:127)
  const double inv = 1.0 / (double)(e - b);
  for (int j = threadIdx.x; j < dim; j += blockDim.x) {
    double acc = 0.0;
    for (uint64_t i = b; i < e; ++i) acc += (double)x[(uint64_t)order[i] * dim + j];
    cents[(uint64_t)c * dim + j] = (float)(acc * inv);
  }
}

}  // namespace

cudaError_t launch_kpp_d2(const float* x, uint64_t n, int dim, const float* center, double* d2, int first,
                          cudaStream_t s) {
  kpp_d2_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(x, n, dim, center, d2, first);
  return cudaGetLastError();
}

size_t kmeans_scan_bytes(uint64_t n) {
  size_t a = 0, b = 0;
  cub::DeviceScan::InclusiveSum(nullptr, a, (const double*)nullptr, (double*)nullptr, (int64_t)n);
  cub::DeviceRadixSort::SortPairs(nullptr, b, (const uint32_t*)nullptr, (uint32_t*)nullptr,
                                  (const uint32_t*)nullptr, (uint32_t*)nullptr, (int64_t)n);
  return (a > b ? a : b) + 256;
}

cudaError_t launch_kpp_scan(const double* d2, double* scan, uint64_t n, void* temp, size_t temp_bytes,
                            cudaStream_t s) {
  return cub::DeviceScan::InclusiveSum(temp, temp_bytes, d2, scan, (int64_t)n, s);
}

cudaError_t launch_first_gt(const double* scan, uint64_t n, double r, unsigned long long* out, cudaStream_t s) {
  first_gt_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(scan, n, r, out);
  return cudaGetLastError();
}

cudaError_t launch_own_dist(const float* x, uint64_t n, int dim, const float* cents, const uint32_t* labels,
                            float* out, cudaStream_t s) {
  own_dist_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(x, n, dim, cents, labels, out);
  return cudaGetLastError();
}

cudaError_t launch_cluster_means(const float* x, uint64_t n, int dim, const uint32_t* labels, int clusters,
                                 float* cents, uint32_t* keys_tmp, uint32_t* order, uint32_t* iota,
                                 void* temp, size_t temp_bytes, cudaStream_t s) {
  iota_u32_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(iota, n);
  // stable radix sort by label: within a cluster rows stay in row order
  cudaError_t e = cub::DeviceRadixSort::SortPairs(temp, temp_bytes, labels, keys_tmp, iota, order, (int64_t)n, 0,
                                                  32, s);
  if (e != cudaSuccess) return e;
  cluster_means_kernel<<<clusters, dim < 128 ? 128 : 256, 0, s>>>(x, dim, order, keys_tmp, n, cents, clusters);
  return cudaGetLastError();
}

}  // namespace dvsg
