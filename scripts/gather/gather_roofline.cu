// Random-row gather ceiling of HBM (the "HBM-gather roofline" north_star
// quotes K1 against): warps read rows of `row_bytes` at random row indices of
// a large array, U rows in flight per warp, and reduce them to one float per
// warp (so the only DRAM traffic is the gathered rows).  Measurement tool,
// not product code: built by scripts/gather_roofline.py.
#include <cstdint>
#include <cuda_runtime.h>

template <int U, int C>
__global__ void __launch_bounds__(256) gather_kernel(const float* __restrict__ base, uint64_t nrows, int dpad,
                                                     const uint32_t* __restrict__ idx, uint64_t nidx,
                                                     float* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const uint64_t warp = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  const int f4 = dpad / 4;  // float4 per row
  float acc = 0.f;
  for (uint64_t i0 = warp * U; i0 < nidx; i0 += nwarps * U) {
    float4 v[U][C];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t i = i0 + u < nidx ? i0 + u : i0;
      const float4* row = reinterpret_cast<const float4*>(base + (uint64_t)idx[i] * dpad);
#pragma unroll
      for (int c = 0; c < C; ++c) {
        const int k = lane + 32 * c;
        if (k < f4) {
          asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
                       : "=f"(v[u][c].x), "=f"(v[u][c].y), "=f"(v[u][c].z), "=f"(v[u][c].w)
                       : "l"(row + k));
        } else {
          v[u][c] = make_float4(0.f, 0.f, 0.f, 0.f);
        }
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int c = 0; c < C; ++c) acc += v[u][c].x + v[u][c].y + v[u][c].z + v[u][c].w;
  }
  if (lane == 0) out[warp] = acc;
}

extern "C" int gather_run(const float* base, uint64_t nrows, int dpad, const uint32_t* idx, uint64_t nidx,
                          float* out, int u, int blocks, float* ms) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  const int c = (dpad / 4 + 31) / 32;
#define GR(UU, CC) gather_kernel<UU, CC><<<blocks, 256>>>(base, nrows, dpad, idx, nidx, out)
  if (c <= 1) {
    switch (u) { case 1: GR(1, 1); break; case 2: GR(2, 1); break; case 4: GR(4, 1); break; case 8: GR(8, 1); break; default: return 1; }
  } else if (c <= 4) {
    switch (u) { case 1: GR(1, 4); break; case 2: GR(2, 4); break; case 4: GR(4, 4); break; default: return 1; }
  } else if (c <= 6) {
    switch (u) { case 1: GR(1, 6); break; case 2: GR(2, 6); break; case 4: GR(4, 6); break; default: return 1; }
  } else {
    return 1;
  }
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  return (int)cudaGetLastError();
}
