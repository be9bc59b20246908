// search_kernel.cu -- K1: persistent batched greedy beam search for sm_100a.
//
// Semantics: beam_search_stats, /root/reference/proj/src/graph_index.cpp:105-187
// (exact visited set, pool cap = max(4k, 2*I*w), frontier = first w
// unexpanded pool entries, pool order (dist, local id), final order
// (dist, global id), visited = number of vectors scored).
//
// Design (one CTA of 256 threads per (query, partition) unit, persistent
// over a global work counter):
//   * pool      : sorted u64 keys in smem, key = ord(dist)<<32 | local<<1 | expanded
//                 (the expanded flag rides in bit 0, which never decides an
//                 order because local ids are unique) -- double buffered.
//   * visited   : exact open-addressing u32 hash, smem when it fits, else a
//                 per-CTA region in global memory (L2-resident); never forgets,
//                 like the reference's unordered_set (graph_index.cpp:133,165).
//   * per chunk of <= 2048 raw candidate ids (entry nodes, or the adjacency
//     rows of the frontier):
//       dedup      -> warp-aggregated append of new ids (visited += new)
//       score      -> one warp per vector, float4 gathers, U vectors in flight
//                     per warp, fp64 (parity) or fp32 (fast) lane partials and
//                     a butterfly tree
//       filter     -> exact: drop keys above the current cap-th pool key
//                     (they could not survive shrink())
//       sort/merge -> bitonic sort of survivors, co-rank merge into the pool,
//                     truncated at cap (== the reference's sort + resize)
//   Chunking is exact because top-cap(A u B u C) = top-cap(top-cap(A u B) u C)
//   for unique keys, and frontier selection only happens between iterations.
#include <algorithm>
#include <cstdint>
#include <cuda_runtime.h>

#include "dvsg_internal.h"
#include "k1_device.cuh"

namespace dvsg {
namespace {

// VPL: float4 slots per lane (dpad <= 128 * VPL).  U: vectors in flight per warp.
// FULL: dpad == 128 * VPL (every lane holds real dimensions; no bound check).

#ifndef DVSG_MINB
#define DVSG_MINB 5  // resident CTAs per SM the register budget is cut for (measured sweep)
#endif
// Wide rows (VPL >= 4, dim > 384): a 2-3 KB row per vector and pools that
// cap residency at 2 CTAs/SM by shared memory anyway (w = 256: 107 KB), so
// the register budget goes to more rows in flight per warp instead of more
// CTAs: U = 4 (VPL 4-6) / 2 (VPL 8) at 2 CTAs/SM (<= 128 registers, no
// spills).  Measured at 10M x 768 IP, w = 256 (configs[3]): 8.5k -> 15.4k QPS
// f32c, alg 2.59 -> 4.68 TB/s; 2M x 512/768/1024 at w = 64 and 256 +5-110%.
#ifndef DVSG_MINB_WIDE
#define DVSG_MINB_WIDE 2
#endif
#ifndef DVSG_UVEC
#define DVSG_UVEC 8  // vectors in flight per warp at VPL == 1 (measured sweep)
#endif
#ifndef DVSG_UVEC_WIDE
#define DVSG_UVEC_WIDE -1  // vectors in flight per warp at VPL >= 4 (-1: 4, or 2 at VPL 8; 0: DVSG_UVEC / VPL)
#endif
// U8: vectors read from the byte copy (a.vectors8): a quarter of the gather
// bytes, identical arithmetic (every byte converts exactly to float).
// Byte rows are a quarter of the bytes but the same latency per row, so they
// only pay with more rows in flight: a raw 32-bit word per lane and row.
#ifndef DVSG_UVEC8
#define DVSG_UVEC8 16
#endif
#ifndef DVSG_MINB8
#define DVSG_MINB8 4
#endif
template <int VPL, typename ACC, int METRIC, bool FULL, bool U8>
__global__ void __launch_bounds__(kThreads, U8 ? DVSG_MINB8 : VPL >= 4 ? DVSG_MINB_WIDE : DVSG_MINB)
    search_kernel(const SearchArgs a) {
  constexpr int UW = DVSG_UVEC_WIDE < 0 ? (VPL >= 8 ? 2 : 4) : DVSG_UVEC_WIDE;
  constexpr int U = U8 ? (DVSG_UVEC8 / VPL > 0 ? DVSG_UVEC8 / VPL : 1)
                       : (VPL >= 4 && UW > 0) ? UW : (VPL >= DVSG_UVEC ? 1 : (DVSG_UVEC / VPL));
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ BlockState st;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  uint64_t* pool = reinterpret_cast<uint64_t*>(smem);
  uint64_t* pool_alt = pool + a.cap;
  uint64_t* surv = pool_alt + a.cap;
  uint32_t* cand = reinterpret_cast<uint32_t*>(surv + a.chp);
  uint32_t* frontier = cand + kChunk;
  uint32_t* const region = a.hash_global ? a.hash_global + (size_t)blockIdx.x * (size_t)(a.hsize + a.hsmall)
                                         : frontier + ((a.beam + 3) & ~3);
  const uint32_t dg_magic = (uint32_t)((0x100000000ull + (uint64_t)a.dg - 1) / (uint64_t)a.dg);
  const unsigned full = 0xFFFFFFFFu;
  const unsigned lt_mask = (1u << lane) - 1u;

  const uint64_t nunits = a.nunits_dev ? (uint64_t)*a.nunits_dev : a.nunits;
  for (;;) {
    if (tid == 0) {
      const unsigned long long ticket = atomicAdd(a.work_counter, 1ull);
      st.unit = (a.unit_order && ticket < nunits) ? a.unit_order[ticket] : ticket;
    }
    __syncthreads();
    const uint64_t unit = st.unit;
    if (unit >= nunits) return;

    const uint32_t qi = a.unit_query[unit];
    const PartDesc part = a.parts[a.unit_part[unit]];
    const uint64_t row0 = part.row_off;
    const uint32_t n = part.n;
    const float* vbase = a.vectors + row0 * (uint64_t)a.dpad;
    const float* lbase = vbase + lane * 4;          // this lane's first dims of row 0
    const uint8_t* vbase8 = U8 ? a.vectors8 + row0 * (uint64_t)a.dpad : nullptr;
    const uint8_t* lbase8 = vbase8 + lane * 4;
    const uint32_t* abase = a.adjacency + row0 * (uint64_t)a.dg;
    const uint32_t rstride = (uint32_t)a.dpad;      // u32 x u32 -> u64: one IMAD.WIDE per row

    // query slice in registers: lane holds dims [lane*4 + 128 v, +4)
    float4 q[VPL];
    {
      const float* qp = a.queries + (uint64_t)qi * (uint64_t)a.dim;
#pragma unroll
      for (int v = 0; v < VPL; ++v) {
        const int b = lane * 4 + 128 * v;
        q[v].x = b + 0 < a.dim ? qp[b + 0] : 0.0f;
        q[v].y = b + 1 < a.dim ? qp[b + 1] : 0.0f;
        q[v].z = b + 2 < a.dim ? qp[b + 2] : 0.0f;
        q[v].w = b + 3 < a.dim ? qp[b + 3] : 0.0f;
      }
    }

    // visited table: the small one first when enabled (its lines stay in L2
    // at large beams), the full one only when it could pass 3/4 load
    uint32_t* table = region;
    uint32_t hmask = (uint32_t)(a.hsmall ? a.hsmall : a.hsize) - 1u;
    bool small = a.hsmall > 0;
    for (int i = tid; i <= (int)hmask; i += kThreads) table[i] = kEmpty;
    __syncthreads();

    int P = 0;
    uint64_t thresh = ~0ull;
    uint64_t visited = 0;
    uint64_t expanded = 0;

    const int entries = a.entry_count < (int)n ? a.entry_count : (int)n;
    int nf = 0;
    // phase -1: entry nodes; phases 0..iters-1: frontier expansion
    for (int it = -1; it < a.iters; ++it) {
      int raw_total;
      if (it < 0) {
        raw_total = entries;
      } else {
        // ---- frontier: first `beam` unexpanded pool entries, in pool order
        if (tid == 0) st.nf = 0;
        __syncthreads();
        for (int base = 0; base < P; base += kThreads) {
          const int pos = base + tid;
          const bool cand_f = pos < P && !(pool[pos] & 1ull);
          const unsigned bal = __ballot_sync(full, cand_f);
          if (lane == 0) st.warp_cnt[warp] = __popc(bal);
          __syncthreads();
          int before = st.nf;
          int total = 0;
#pragma unroll
          for (int w = 0; w < kWarps; ++w) {
            if (w < warp) before += st.warp_cnt[w];
            total += st.warp_cnt[w];
          }
          const int rank = before + __popc(bal & lt_mask);
          if (cand_f && rank < a.beam) {
            const uint64_t key = pool[pos];
            frontier[rank] = (uint32_t)(key >> 1) & 0x7FFFFFFFu;
            pool[pos] = key | 1ull;
          }
          __syncthreads();
          if (tid == 0) st.nf += total;
          __syncthreads();
          if (st.nf >= a.beam) break;
        }
        nf = st.nf < a.beam ? st.nf : a.beam;
        if (nf == 0) break;  // graph_index.cpp:160
        expanded += (uint64_t)nf;
        raw_total = nf * a.dg;
      }

      for (int cbase = 0; cbase < raw_total; cbase += kChunk) {
        const int rcount = raw_total - cbase < kChunk ? raw_total - cbase : kChunk;
        if (small && visited + (uint64_t)rcount > (uint64_t)(a.hsmall / 4 * 3)) {  // block-uniform
          // exact growth: rehash the small table's ids into the full one
          uint32_t* big = region + a.hsmall;
          for (int i = tid; i < a.hsize; i += kThreads) big[i] = kEmpty;
          __syncthreads();
          for (int i = tid; i < a.hsmall; i += kThreads) {
            const uint32_t v = table[i];
            if (v != kEmpty) visit_insert(big, (uint32_t)a.hsize - 1u, v);
          }
          __syncthreads();
          table = big;
          hmask = (uint32_t)a.hsize - 1u;
          small = false;
        }
        if (tid == 0) {
          st.ncand = 0;
          st.nsurv = 0;
        }
        // ---- gather raw ids (all loads first for MLP), then dedup
        uint32_t ids[kRawPerThread];
#pragma unroll
        for (int j = 0; j < kRawPerThread; ++j) {
          const int r = j * kThreads + tid;
          ids[j] = kEmpty;
          if (r < rcount) {
            const int g = cbase + r;
            if (it < 0) {
              ids[j] = __ldg(a.entry + row0 + g);
            } else {
              // g / dg by multiply-high with m = ceil(2^32/dg): exact while
              // g * (m*dg - 2^32) < 2^32, i.e. g < 2^24 and dg < 256 (host-checked);
              // dg == 1 overflows m, dg >= 256 takes the plain division
              const uint32_t f = a.dg == 1 ? (uint32_t)g
                               : (a.dg < 256 ? __umulhi((uint32_t)g, dg_magic) : (uint32_t)g / (uint32_t)a.dg);
              const uint32_t jj = (uint32_t)g - f * (uint32_t)a.dg;
              ids[j] = ldg_u32_stream(abase + (uint64_t)frontier[f] * (uint32_t)a.dg + jj);
            }
          }
        }
        __syncthreads();  // st.ncand reset visible
#pragma unroll
        for (int j = 0; j < kRawPerThread; ++j) {
          if (j * kThreads >= rcount) break;  // block-uniform
          const bool isnew = ids[j] != kEmpty && visit_insert(table, hmask, ids[j]);
          const unsigned bal = __ballot_sync(full, isnew);
          int base = 0;
          if (lane == 0 && bal) base = atomicAdd(&st.ncand, __popc(bal));
          base = __shfl_sync(full, base, 0);
          if (isnew) cand[base + __popc(bal & lt_mask)] = ids[j];
        }
        __syncthreads();
        const int M = st.ncand;
        visited += (uint64_t)M;

        // ---- score new candidates: warp per vector, U vectors in flight per warp
        for (int cb = warp * U; cb < M; cb += kWarps * U) {
          uint32_t ids_u[U];
          if constexpr (U >= 4) {
#pragma unroll
            for (int u4 = 0; u4 < U; u4 += 4) {
              const uint4 w4 = *reinterpret_cast<const uint4*>(cand + cb + u4);
              ids_u[u4] = w4.x; ids_u[u4 + 1] = w4.y; ids_u[u4 + 2] = w4.z; ids_u[u4 + 3] = w4.w;
            }
          } else {
#pragma unroll
            for (int u = 0; u < U; ++u) ids_u[u] = cand[cb + u];
          }
          float4 x[U8 ? 1 : U][VPL];
          uint32_t x8[U8 ? U : 1][VPL];
#pragma unroll
          for (int u = 0; u < U; ++u) {
            // past M: load row 0 (harmless, result discarded by the ci < M test)
            const uint32_t id = cb + u < M ? ids_u[u] : 0u;
#pragma unroll
            for (int v = 0; v < VPL; ++v) {
              const bool in = FULL || lane * 4 + 128 * v < a.dpad;
              if constexpr (U8) {
                x8[u][v] = in ? ldg_u8x4_raw(lbase8 + (uint64_t)id * rstride + 128 * v) : 0u;
              } else {
                x[u][v] = in ? ldg_f4(lbase + (uint64_t)id * rstride + 128 * v) : make_float4(0.f, 0.f, 0.f, 0.f);
              }
            }
          }
          ACC part[U];
#pragma unroll
          for (int u = 0; u < U; ++u) {
            ACC acc;
            if constexpr (U8) {
              acc = lane_partial<ACC, METRIC>(cvt_u8x4(x8[u][0]), q[0]);
#pragma unroll
              for (int v = 1; v < VPL; ++v) acc += lane_partial<ACC, METRIC>(cvt_u8x4(x8[u][v]), q[v]);
            } else {
              acc = lane_partial<ACC, METRIC>(x[u][0], q[0]);
#pragma unroll
              for (int v = 1; v < VPL; ++v) acc += lane_partial<ACC, METRIC>(x[u][v], q[v]);
            }
            part[u] = acc;
          }
          const ACC tot = transpose_reduce<U, ACC>(part, lane);
          constexpr int LU = ilog2(U);
          const int myu = (lane >> (5 - LU)) & (U - 1);
          const int ci = cb + myu;
          bool pass = false;
          uint64_t mykey = 0;
          if ((lane & ((32 >> LU) - 1)) == 0 && ci < M) {
            const float* qrow = a.queries + (uint64_t)qi * (uint64_t)a.dim;
            float dist;
            if constexpr (U8) dist = finish_dist<ACC, METRIC>(tot, vbase8 + (uint64_t)cand[ci] * rstride, qrow, a.dim);
            else dist = finish_dist<ACC, METRIC>(tot, vbase + (uint64_t)cand[ci] * rstride, qrow, a.dim);
            mykey = ((uint64_t)f2ord(dist) << 32) | ((uint64_t)cand[ci] << 1);
            pass = mykey < thresh;
          }
          const unsigned bal = __ballot_sync(full, pass);
          int base = 0;
          if (lane == 0 && bal) base = atomicAdd(&st.nsurv, __popc(bal));
          base = __shfl_sync(full, base, 0);
          if (pass) surv[base + __popc(bal & lt_mask)] = mykey;
        }
        __syncthreads();
        const int S = st.nsurv;
        __syncthreads();  // every thread has read the counters before the next reset
        if (S == 0) continue;  // block-uniform

        // ---- sort survivors, merge into the pool, truncate at cap
        sort_keys(surv, S, tid);
        const int outn = P + S < a.cap ? P + S : a.cap;
        merge_path(pool, P, surv, S, pool_alt, outn, tid);
        __syncthreads();
        {
          uint64_t* t = pool;
          pool = pool_alt;
          pool_alt = t;
        }
        P = P + S < a.cap ? P + S : a.cap;
        thresh = P == a.cap ? pool[a.cap - 1] : ~0ull;
      }
    }

    // ---- final: global ids, re-sorted by (dist, gid), first min(k, P)
    //      (graph_index.cpp:173-186).  Only entries whose dist ties the
    //      want-th can reorder, so sort the prefix up to the last such tie.
    const int want = a.k < P ? a.k : P;
    if (want > 0) {
      const uint32_t dk = (uint32_t)(pool[want - 1] >> 32);
      int lo = want, hi = P;  // first index with dist > dk
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if ((uint32_t)(pool[mid] >> 32) <= dk) lo = mid + 1; else hi = mid;
      }
      const int m = lo;
      for (int i = tid; i < m; i += kThreads) {
        const uint64_t key = pool[i];
        const uint32_t local = (uint32_t)(key >> 1) & 0x7FFFFFFFu;
        surv[i] = (key & 0xFFFFFFFF00000000ull) | (uint64_t)__ldg(a.gids + row0 + local);
      }
      __syncthreads();
      sort_keys(surv, m, tid);
      for (int i = tid; i < want; i += kThreads) {
        const uint64_t key = surv[i];
        a.out_ids[unit * (uint64_t)a.k + i] = (uint32_t)key;
        a.out_dists[unit * (uint64_t)a.k + i] = ord2f((uint32_t)(key >> 32));
      }
    }
    if (tid == 0) {
      a.out_count[unit] = (uint32_t)want;
      a.out_visited[unit] = visited;
      if (a.stats) {
        atomicAdd(a.stats + 0, 1ull);
        atomicAdd(a.stats + 1, (unsigned long long)visited);
        atomicAdd(a.stats + 2, (unsigned long long)expanded);
      }
    }
    __syncthreads();
  }
}

template <int VPL, typename ACC, int METRIC, bool FULL, bool U8 = false>
cudaError_t launch_t(const SearchArgs& a, int num_sms, int max_grid, cudaStream_t stream,
                     int* grid_out) {
  auto kern = search_kernel<VPL, ACC, METRIC, FULL, U8>;
  const size_t smem = search_smem_bytes(a.cap, a.chp, a.beam, a.hsize, a.hash_global == nullptr);
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int per_sm = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kThreads, smem);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) return cudaErrorInvalidConfiguration;
  uint64_t grid = (uint64_t)per_sm * (uint64_t)num_sms;
  if (grid > a.nunits) grid = a.nunits;
  if (max_grid > 0 && grid > (uint64_t)max_grid) grid = (uint64_t)max_grid;
  if (grid < 1) grid = 1;
  if (grid_out) *grid_out = (int)grid;
  kern<<<(unsigned)grid, kThreads, smem, stream>>>(a);
  return cudaGetLastError();
}

template <int VPL, bool U8>
cudaError_t launch_v(const SearchArgs& a, int metric, int accum, int num_sms, int mg,
                     cudaStream_t s, int* g) {
  const bool full = a.dpad == 128 * VPL;
  if (accum == 0) {
    if (metric == 0) return full ? launch_t<VPL, double, 0, true, U8>(a, num_sms, mg, s, g)
                                 : launch_t<VPL, double, 0, false, U8>(a, num_sms, mg, s, g);
    return full ? launch_t<VPL, double, 1, true, U8>(a, num_sms, mg, s, g)
                : launch_t<VPL, double, 1, false, U8>(a, num_sms, mg, s, g);
  }
  if (accum == 2) {
    if (metric == 0) return full ? launch_t<VPL, F2, 0, true, U8>(a, num_sms, mg, s, g)
                                 : launch_t<VPL, F2, 0, false, U8>(a, num_sms, mg, s, g);
    return full ? launch_t<VPL, F2, 1, true, U8>(a, num_sms, mg, s, g)
                : launch_t<VPL, F2, 1, false, U8>(a, num_sms, mg, s, g);
  }
  if (metric == 0) return full ? launch_t<VPL, float, 0, true, U8>(a, num_sms, mg, s, g)
                               : launch_t<VPL, float, 0, false, U8>(a, num_sms, mg, s, g);
  return full ? launch_t<VPL, float, 1, true, U8>(a, num_sms, mg, s, g)
              : launch_t<VPL, float, 1, false, U8>(a, num_sms, mg, s, g);
}

}  // namespace

size_t search_smem_bytes(int cap, int chp, int beam, int hsize, bool hash_in_smem) {
  size_t b = sizeof(uint64_t) * (2 * (size_t)cap + (size_t)chp);
  b += sizeof(uint32_t) * ((size_t)kChunk + (size_t)((beam + 3) & ~3));
  if (hash_in_smem) b += sizeof(uint32_t) * (size_t)hsize;
  return b;
}

cudaError_t launch_search(const SearchArgs& a, int metric, int accum, int num_sms,
                          int max_grid, cudaStream_t stream, int* grid_out) {
  const int vpl = (a.dpad + 127) / 128;
  if (a.vectors8) {  // byte storage: the rows of byte datasets (SIFT, Deep: dim <= 256)
    switch (vpl) {
      case 1: return launch_v<1, true>(a, metric, accum, num_sms, max_grid, stream, grid_out);
      case 2: return launch_v<2, true>(a, metric, accum, num_sms, max_grid, stream, grid_out);
      default: return cudaErrorInvalidValue;
    }
  }
  switch (vpl) {
    case 1: return launch_v<1, false>(a, metric, accum, num_sms, max_grid, stream, grid_out);
    case 2: return launch_v<2, false>(a, metric, accum, num_sms, max_grid, stream, grid_out);
    case 3:
    case 4: return launch_v<4, false>(a, metric, accum, num_sms, max_grid, stream, grid_out);
    case 5:
    case 6: return launch_v<6, false>(a, metric, accum, num_sms, max_grid, stream, grid_out);
    case 7:
    case 8: return launch_v<8, false>(a, metric, accum, num_sms, max_grid, stream, grid_out);
    default: return cudaErrorInvalidValue;
  }
}

namespace {
__global__ void to_u8_kernel(const float* __restrict__ x, uint64_t n, uint8_t* __restrict__ out, int* bad) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const float v = x[i];
    const bool ok = v >= 0.f && v <= 255.f && v == rintf(v);
    if (!ok) atomicOr(bad, 1);
    out[i] = ok ? (uint8_t)v : 0;
  }
}
}  // namespace

cudaError_t launch_to_u8(const float* x, uint64_t n, uint8_t* out, int* bad, cudaStream_t stream) {
  if (n == 0) return cudaSuccess;
  const uint64_t blocks = std::min<uint64_t>((n + 255) / 256, 148ull * 32);
  to_u8_kernel<<<(unsigned)blocks, 256, 0, stream>>>(x, n, out, bad);
  return cudaGetLastError();
}

}  // namespace dvsg
