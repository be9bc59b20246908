// cluster_xchg.cu -- device-initiated dispatch / combine of the cluster-
// sharded run_pipeline (SURVEY 8e design A: the reference's own semantics,
// cluster i on rank placement[i], router.cpp:28-79, simulator.cpp:245-337).
//
// One step on every rank, all on the rank's stream, no host round trip:
//
//   K3 dispatch (cl_dispatch): one thread per routed unit u = q*fanout + j
//      (route, router.cpp:52-79, self-traffic kept); the lanes of a warp that
//      go to the same owner reserve their inbox slots with one peer atomic on
//      the owner's cursor[parity][me], then the warp copies each unit's query
//      row into the owner's inbox with coalesced NVLink peer stores, plus a
//      {cluster, origin unit} header;
//   -- peer-flag barrier --
//   owner: cl_units turns the per-origin cursors into a unit list for K1
//      (unit count left on the device: K1 reads it, nothing goes to the host),
//      K1 searches every received unit in its resident partition, and
//      cl_reply pushes each unit's k ids / dists / count / visited (and the k
//      hit vectors, simulator.cpp:329-333, gathered from the owner's rows)
//      into the origin's reply region at the unit's own index;
//   -- peer-flag barrier --
//   origin: K4 combine_results (simulator.cpp:219-243) over its nq x fanout
//      replies, cl_pick_vectors attaches each final hit's vector.
//
// Cursors are double-buffered by step parity: a rank clears the other
// parity's cursors between the two barriers, when no rank can be writing
// them (every dispatch of this step happened before barrier 1; the next
// step's dispatches start after barrier 2).
#include <cstdint>
#include <cuda_runtime.h>

#include "dvsg_internal.h"

namespace dvsg {
namespace {

__device__ __forceinline__ unsigned ld_acquire_sys(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(unsigned* p, unsigned v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// K3: warp w handles units [32w, 32w+32)
__global__ void cl_dispatch_kernel(const ClArena* __restrict__ peers, int nranks, int me, int parity,
                                   const float* __restrict__ q, uint64_t nq, int dim, int fanout,
                                   const uint32_t* __restrict__ assign, const uint32_t* __restrict__ placement,
                                   uint32_t nclusters, uint64_t cap, int* err) {
  const int lane = threadIdx.x & 31;
  const uint64_t u0 = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) & ~31ull;
  const uint64_t nu = nq * (uint64_t)fanout;
  if (u0 >= nu) return;
  const uint64_t u = u0 + lane;
  const bool act = u < nu;
  uint32_t cl = 0, owner = 0;
  if (act) {
    cl = assign[u];
    if (cl >= nclusters) {
      atomicOr(err, 1);
      cl = 0;
    }
    owner = placement[cl];
  }
  // one peer atomic per (warp, owner): slots for the lanes going there
  uint64_t slot = 0;
  for (int o = 0; o < nranks; ++o) {
    const unsigned m = __ballot_sync(0xFFFFFFFFu, act && owner == (uint32_t)o);
    if (!m) continue;
    unsigned base = 0;
    if (lane == __ffs(m) - 1) base = atomicAdd(peers[o].cursor + parity * kXgMaxRanks + me, (unsigned)__popc(m));
    base = __shfl_sync(0xFFFFFFFFu, base, __ffs(m) - 1);
    if (act && owner == (uint32_t)o) slot = base + __popc(m & ((1u << lane) - 1u));
  }
  if (act && slot >= cap) atomicOr(err, 2);  // capacity: set at dvsg_cluster_comm_init
  // the warp copies its units' rows, one row at a time, float4 peer stores
  const unsigned valid = __ballot_sync(0xFFFFFFFFu, act && slot < cap);
  for (int l = 0; l < 32; ++l) {
    if (!((valid >> l) & 1u)) continue;
    const uint64_t ul = __shfl_sync(0xFFFFFFFFu, u, l);
    const uint32_t ol = __shfl_sync(0xFFFFFFFFu, owner, l);
    const uint64_t sl = __shfl_sync(0xFFFFFFFFu, slot, l);
    const uint32_t cll = __shfl_sync(0xFFFFFFFFu, cl, l);
    const float* src = q + (ul / (uint64_t)fanout) * (uint64_t)dim;
    float* dst = peers[ol].inbox_q + ((uint64_t)me * cap + sl) * (uint64_t)dim;
    if ((dim & 3) == 0) {
      for (int i = lane; i < dim / 4; i += 32)
        reinterpret_cast<float4*>(dst)[i] = __ldg(reinterpret_cast<const float4*>(src) + i);
    } else {
      for (int i = lane; i < dim; i += 32) dst[i] = __ldg(src + i);
    }
    if (lane == 0) peers[ol].inbox_meta[(uint64_t)me * cap + sl] = make_uint2(cll, (uint32_t)ul);
  }
}

// owner: unit list over the inbox sections of every origin
__global__ void cl_units_kernel(const ClArena* __restrict__ peers, int nranks, int me, int parity, uint64_t cap,
                                const int32_t* __restrict__ cluster_to_slot, uint32_t nmap,
                                uint32_t* __restrict__ unit_query, uint32_t* __restrict__ unit_part,
                                unsigned long long* nunits, int* err) {
  __shared__ uint64_t off[kXgMaxRanks + 1];
  const ClArena& mine = peers[me];
  if (threadIdx.x == 0) {
    off[0] = 0;
    for (int o = 0; o < kXgMaxRanks; ++o) {
      uint64_t c = o < nranks ? (uint64_t)mine.cursor[parity * kXgMaxRanks + o] : 0;
      if (c > cap) c = cap;
      off[o + 1] = off[o] + c;
    }
    if (blockIdx.x == 0) *nunits = off[kXgMaxRanks];
  }
  __syncthreads();
  const uint64_t total = off[kXgMaxRanks];
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (uint64_t)gridDim.x * blockDim.x) {
    int o = 0;
    for (int s = 1; s < kXgMaxRanks; ++s) o += i >= off[s] ? 1 : 0;
    const uint64_t idx = (uint64_t)o * cap + (i - off[o]);
    const uint32_t cl = mine.inbox_meta[idx].x;
    const int32_t slot = cl < nmap ? cluster_to_slot[cl] : -1;
    if (slot < 0) atomicOr(err, 4);  // routed to a rank that does not hold the cluster
    unit_query[i] = (uint32_t)idx;
    unit_part[i] = slot < 0 ? 0u : (uint32_t)slot;
  }
}

// owner -> origin: one warp per searched unit
__global__ void cl_reply_kernel(const ClArena* __restrict__ peers, int me, uint64_t cap,
                                const uint32_t* __restrict__ unit_query, const unsigned long long* nunits,
                                int k, const uint32_t* __restrict__ ids, const float* __restrict__ dists,
                                const uint32_t* __restrict__ counts, const uint64_t* __restrict__ visited,
                                const uint64_t* __restrict__ locator, const float* __restrict__ vectors, int dim,
                                int dpad, int with_vectors) {
  const int lane = threadIdx.x & 31;
  const uint64_t w = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (w >= *nunits) return;
  const uint32_t idx = unit_query[w];
  const int origin = (int)(idx / cap);
  const uint32_t ou = peers[me].inbox_meta[idx].y;
  const ClArena& dst = peers[origin];
  const uint32_t cnt = counts[w];
  for (int i = lane; i < k; i += 32) {
    dst.r_ids[(uint64_t)ou * k + i] = ids[w * (uint64_t)k + i];
    dst.r_dists[(uint64_t)ou * k + i] = dists[w * (uint64_t)k + i];
  }
  if (lane == 0) {
    dst.r_count[ou] = cnt;
    dst.r_visited[ou] = visited[w];
  }
  if (with_vectors) {
    for (uint32_t h = 0; h < cnt; ++h) {
      const float* src = vectors + locator[ids[w * (uint64_t)k + h]] * (uint64_t)dpad;
      float* o = dst.r_vec + ((uint64_t)ou * k + h) * (uint64_t)dim;
      for (int i = lane; i < dim; i += 32) o[i] = src[i];
    }
  }
}

__global__ void cl_reset_kernel(const ClArena* __restrict__ peers, int me, int parity) {
  if (threadIdx.x < kXgMaxRanks) peers[me].cursor[(parity ^ 1) * kXgMaxRanks + threadIdx.x] = 0;
}

// each final hit's vector from the partial that produced it (clusters are
// disjoint, so a global id appears in at most one partial of a query)
__global__ void cl_pick_vectors_kernel(const uint32_t* __restrict__ ids, const uint32_t* __restrict__ counts,
                                       uint64_t nq, int k, int fanout, const uint32_t* __restrict__ r_ids,
                                       const uint32_t* __restrict__ r_count, const float* __restrict__ r_vec,
                                       int dim, float* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const uint64_t slot = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (slot >= nq * (uint64_t)k) return;
  const uint64_t q = slot / (uint64_t)k;
  const uint32_t h = (uint32_t)(slot - q * (uint64_t)k);
  if (h >= counts[q]) return;
  const uint32_t id = ids[slot];
  uint64_t src = ~0ull;
  for (int j = 0; j < fanout && src == ~0ull; ++j) {  // warp-uniform loop
    const uint64_t u = q * (uint64_t)fanout + j;
    const uint32_t c = r_count[u];
    for (uint32_t base = 0; base < c; base += 32) {
      const uint32_t i = base + lane;
      const unsigned m = __ballot_sync(0xFFFFFFFFu, i < c && r_ids[u * k + i] == id);
      if (m) {
        src = u * k + base + (__ffs(m) - 1);
        break;
      }
    }
  }
  if (src == ~0ull) return;
  for (int i = lane; i < dim; i += 32) out[slot * (uint64_t)dim + i] = r_vec[src * (uint64_t)dim + i];
}

__global__ void cl_barrier_kernel(const ClArena* __restrict__ peers, int nranks, int me, unsigned epoch, int* err) {
  if (threadIdx.x != 0 || *reinterpret_cast<volatile int*>(err)) return;
  __threadfence_system();
  for (int r = 0; r < nranks; ++r) st_release_sys(peers[r].flags + me, epoch);
  const unsigned* mine = peers[me].flags;
  const uint64_t t0 = globaltimer();
  for (int r = 0; r < nranks; ++r) {
    while ((int)(ld_acquire_sys(mine + r) - epoch) < 0) {
      if (globaltimer() - t0 > 20000000000ull) {
        atomicOr(err, 8);
        return;
      }
      __nanosleep(256);
    }
  }
  __threadfence_system();
}

}  // namespace

cudaError_t launch_cl_dispatch(const ClArena* peers, int nranks, int me, int parity, const float* q, uint64_t nq,
                               int dim, int fanout, const uint32_t* assign, const uint32_t* placement,
                               uint32_t nclusters, uint64_t cap, int* err, cudaStream_t s) {
  const uint64_t nu = nq * (uint64_t)fanout;
  if (nu == 0) return cudaSuccess;
  cl_dispatch_kernel<<<(unsigned)((nu + 255) / 256), 256, 0, s>>>(peers, nranks, me, parity, q, nq, dim, fanout,
                                                                  assign, placement, nclusters, cap, err);
  return cudaGetLastError();
}

cudaError_t launch_cl_units(const ClArena* peers, int nranks, int me, int parity, uint64_t cap,
                            const int32_t* cluster_to_slot, uint32_t nmap, uint32_t* unit_query,
                            uint32_t* unit_part, unsigned long long* nunits, int* err, cudaStream_t s) {
  cl_units_kernel<<<4 * 148, 256, 0, s>>>(peers, nranks, me, parity, cap, cluster_to_slot, nmap, unit_query,
                                          unit_part, nunits, err);
  return cudaGetLastError();
}

cudaError_t launch_cl_reply(const ClArena* peers, int me, uint64_t cap, const uint32_t* unit_query,
                            const unsigned long long* nunits, uint64_t max_units, int k, const uint32_t* ids,
                            const float* dists, const uint32_t* counts, const uint64_t* visited,
                            const uint64_t* locator, const float* vectors, int dim, int dpad, int with_vectors,
                            cudaStream_t s) {
  if (max_units == 0) return cudaSuccess;
  cl_reply_kernel<<<(unsigned)((max_units * 32 + 255) / 256), 256, 0, s>>>(
      peers, me, cap, unit_query, nunits, k, ids, dists, counts, visited, locator, vectors, dim, dpad,
      with_vectors);
  return cudaGetLastError();
}

cudaError_t launch_cl_reset(const ClArena* peers, int me, int parity, cudaStream_t s) {
  cl_reset_kernel<<<1, 32, 0, s>>>(peers, me, parity);
  return cudaGetLastError();
}

cudaError_t launch_cl_pick_vectors(const uint32_t* ids, const uint32_t* counts, uint64_t nq, int k, int fanout,
                                   const uint32_t* r_ids, const uint32_t* r_count, const float* r_vec, int dim,
                                   float* out, cudaStream_t s) {
  const uint64_t n = nq * (uint64_t)k;
  if (n == 0) return cudaSuccess;
  cl_pick_vectors_kernel<<<(unsigned)((n * 32 + 255) / 256), 256, 0, s>>>(ids, counts, nq, k, fanout, r_ids,
                                                                         r_count, r_vec, dim, out);
  return cudaGetLastError();
}

cudaError_t launch_cl_barrier(const ClArena* peers, int nranks, int me, unsigned epoch, int* err, cudaStream_t s) {
  cl_barrier_kernel<<<1, 32, 0, s>>>(peers, nranks, me, epoch, err);
  return cudaGetLastError();
}

}  // namespace dvsg
