// xchg_kernel.cu -- node-sharded search with a bulk-synchronous frontier
// exchange over NVLink peer memory (the multi-GPU layout of the north star).
//
// Semantics are exactly beam_search_stats (graph_index.cpp:105-187) over the
// UNSHARDED graph, as in K1 and the fused sharded kernel (shard_kernel.cu):
// the pool, visited set and frontier of a query live on its origin rank; only
// the rank that scores a candidate changes (node v's vector lives on rank
// v / S; adjacency, global ids and entry order are replicated).
//
// Instead of a per-CTA request/reply round trip (shard_kernel.cu, latency
// bound: ~40 us per trip, 7 trips per query), every query of the wave advances
// one phase at a time; per phase there are two kinds of work:
//
//   origin (expand_unit, CTA per query):
//     merge the keys the owners returned for the previous phase into the pool
//     (exact threshold filter, sort, merge path -- as K1), pick the frontier
//     (first w unexpanded, graph_index.cpp:156-161), gather its adjacency
//     rows, dedup against the visited hash (exact, per query in HBM), bucket
//     the new ids by owner, reserve a contiguous inbox range at each owner
//     (one peer atomic per owner) and write the requests there with
//     coalesced NVLink peer stores;
//   -- peer-flag barrier (xg_barrier) --
//   owner (score_warp_block, warp per 32 requests):
//     gather the rows (float4, 8 in flight per warp), score them exactly as
//     K1 (same lane partials and butterfly tree, so the same bits), and store
//     the 32 keys with one coalesced peer store into the origin's reply range
//     (same index as the inbox slot, so the origin needs no ids back);
//   -- peer-flag barrier --
//
// Two lanes (query waves) run half a phase apart and every xg_step launch
// carries one lane's origin items and the other lane's owner blocks, CTAs
// split by role, so latency-bound origin work and HBM-bound gathers share the
// SMs.  Phase 0 expands the entry nodes, phases 1..I the frontiers, and a
// last origin pass (phase I+1) merges the final replies and writes the
// (dist, gid)-sorted top-k (graph_index.cpp:173-186).  Traffic per remote
// candidate: 8 B request + 8 B key over NVLink instead of a 4*d-byte gather;
// load balance across ranks follows the (uniform) shard rule, not the query
// split.  Emulation (all ranks on one device) runs the same kernels with the
// barrier replaced by stream order; the NCCL baseline runs them over local
// slabs with host-driven ncclSend/ncclRecv in place of the peer stores.
#include <cstdint>
#include <cuda_runtime.h>

#include "dvsg_internal.h"
#include "k1_device.cuh"

#ifndef DVSG_XG_BATCH_PROBES
#define DVSG_XG_BATCH_PROBES 1
#endif
#ifndef DVSG_XG_SORT_RUNS
#define DVSG_XG_SORT_RUNS 1
#endif
#ifndef DVSG_UVEC
#define DVSG_UVEC 8  // vectors in flight per warp at VPL == 1 (as K1)
#endif

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

struct XgShared {
  uint64_t unit;
  int cnt[kXgMaxRanks];
  int fill[kXgMaxRanks];
  int off[kXgMaxRanks + 1];
  unsigned pos[kXgMaxRanks];
  uint2 meta[kXgMaxRanks];
};

// lane's slice of a dpad-strided query row (dims >= dim read as 0)
template <int VPL, bool FULL>
__device__ __forceinline__ void load_query(float4 (&q)[VPL], const float* qp, int lane, int dim) {
#pragma unroll
  for (int v = 0; v < VPL; ++v) {
    const int d0 = lane * 4 + 128 * v;
    if (FULL || d0 + 3 < dim) {
      q[v] = __ldcg(reinterpret_cast<const float4*>(qp + d0));
    } else {
      q[v].x = d0 + 0 < dim ? __ldcg(qp + d0 + 0) : 0.0f;
      q[v].y = d0 + 1 < dim ? __ldcg(qp + d0 + 1) : 0.0f;
      q[v].z = d0 + 2 < dim ? __ldcg(qp + d0 + 2) : 0.0f;
      q[v].w = d0 + 3 < dim ? __ldcg(qp + d0 + 3) : 0.0f;
    }
  }
}

// One query of the origin's wave: merge the previous phase's replies, then
// (phases <= iters) pick the frontier, dedup, push the requests, or
// (phase iters + 1) write the result.  Block-uniform call.
template <int VPL, typename ACC, int METRIC, bool FULL>
__device__ __forceinline__ void expand_unit(const XgArgs& a, const int rr, const uint32_t j,
                                            unsigned char* smem, BlockState& st, XgShared& xs) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int R = a.nranks;
  uint64_t* pool = reinterpret_cast<uint64_t*>(smem);
  uint64_t* pool_alt = pool + a.cap;
  uint64_t* surv = pool_alt + a.cap;
  uint32_t* cand = reinterpret_cast<uint32_t*>(surv + a.chp);
  uint32_t* buck = cand + a.maxraw;
  uint32_t* frontier = buck + a.maxraw;
  const uint32_t hmask = (uint32_t)a.hsize - 1u;
  const uint32_t dg_magic = (uint32_t)((0x100000000ull + (uint64_t)a.dg - 1) / (uint64_t)a.dg);
  const unsigned full = 0xFFFFFFFFu;
  const unsigned lt_mask = (1u << lane) - 1u;
  const bool entry_phase = a.phase == 0;
  const bool final_phase = a.phase > a.iters;
  const int slot = a.phase & 1;
  {
    const int me = a.rank_lo + rr;
    const uint64_t qs = (uint64_t)rr * a.wcap + j;
    uint32_t* table = a.hash + qs * (uint64_t)a.hsize;
    uint64_t* gpool = a.pool + qs * (uint64_t)a.cap;

    int P = 0;
    uint64_t visited = 0;
    uint32_t expanded = 0;
    if (entry_phase) {
      for (int i = tid; i < a.hsize; i += kThreads) table[i] = kEmpty;
    } else {
      P = (int)a.psize[qs];
      visited = a.visited[qs];
      expanded = a.expd[qs];
      for (int i = tid; i < P; i += kThreads) pool[i] = gpool[i];
      if (tid < R) xs.meta[tid] = a.meta[qs * (uint64_t)R + tid];
    }
    __syncthreads();
    uint64_t thresh = P == a.cap ? pool[a.cap - 1] : ~0ull;

    // ---- merge the keys the owners returned for the previous phase
    if (!entry_phase) {
      int off[kXgMaxRanks + 1];
      off[0] = 0;
#pragma unroll
      for (int r = 0; r < kXgMaxRanks; ++r) off[r + 1] = off[r] + (r < R ? (int)xs.meta[r].y : 0);
      const int tot = off[kXgMaxRanks];
      const uint64_t* rbase = a.views[me].reply;
      for (int cbase = 0; cbase < tot; cbase += kChunk) {
        const int rc = tot - cbase < kChunk ? tot - cbase : kChunk;
        if (tid == 0) st.nsurv = 0;
        __syncthreads();
        uint64_t keys[kRawPerThread];  // all loads in flight before the first use
#pragma unroll
        for (int jj = 0; jj < kRawPerThread; ++jj) {
          const int g = cbase + jj * kThreads + tid;
          keys[jj] = ~0ull;
          if (jj * kThreads + tid < rc) {
            int r = 0, offr = 0;
#pragma unroll
            for (int s = 1; s < kXgMaxRanks; ++s)
              if (g >= off[s]) {
                r = s;
                offr = off[s];
              }
            keys[jj] = __ldcg(rbase + (uint64_t)r * a.rstride + xs.meta[r].x + (uint32_t)(g - offr));
          }
        }
#pragma unroll
        for (int jj = 0; jj < kRawPerThread; ++jj) {
          const uint64_t key = keys[jj];
          const bool pass = jj * kThreads + tid < rc && key < thresh;
          const unsigned bal = __ballot_sync(full, pass);
          int base = 0;
          if (lane == 0 && bal) base = atomicAdd(&st.nsurv, __popc(bal));
          base = __shfl_sync(full, base, 0);
          if (pass) surv[base + __popc(bal & lt_mask)] = key;
        }
        __syncthreads();
        const int S = st.nsurv;
        __syncthreads();
        if (S == 0) continue;
#if DVSG_XG_SORT_RUNS
        // cand + buck (maxraw u64, unused until the dedup below) as the ping-pong buffer
        const uint64_t* sorted = sort_runs(surv, S, reinterpret_cast<uint64_t*>(cand), tid);
#else
        sort_keys(surv, S, tid);
        const uint64_t* sorted = surv;
#endif
        const int outn = P + S < a.cap ? P + S : a.cap;
        merge_path(pool, P, sorted, S, pool_alt, outn, tid);
        __syncthreads();
        uint64_t* t = pool;
        pool = pool_alt;
        pool_alt = t;
        P = outn;
        thresh = P == a.cap ? pool[a.cap - 1] : ~0ull;
      }
    }

    if (final_phase) {
      // ---- (dist, gid) order, first min(k, P) (graph_index.cpp:173-186)
      const uint64_t ob = (uint64_t)rr * a.out_stride + j;
      const int want = a.k < P ? a.k : P;
      if (want > 0) {
        const uint32_t dk = (uint32_t)(pool[want - 1] >> 32);
        int lo = want, hi = P;
        while (lo < hi) {
          const int mid = (lo + hi) >> 1;
          if ((uint32_t)(pool[mid] >> 32) <= dk) lo = mid + 1; else hi = mid;
        }
        const int m = lo;
        for (int i = tid; i < m; i += kThreads) {
          const uint64_t key = pool[i];
          const uint32_t local = (uint32_t)(key >> 1) & 0x7FFFFFFFu;
          surv[i] = (key & 0xFFFFFFFF00000000ull) | (uint64_t)__ldg(a.gids + local);
        }
        __syncthreads();
        sort_keys(surv, m, tid);
        for (int i = tid; i < want; i += kThreads) {
          const uint64_t key = surv[i];
          a.out_ids[ob * (uint64_t)a.k + i] = (uint32_t)key;
          a.out_dists[ob * (uint64_t)a.k + i] = ord2f((uint32_t)(key >> 32));
        }
      }
      if (tid == 0) {
        a.out_count[ob] = (uint32_t)want;
        a.out_visited[ob] = visited;
        if (a.stats) {
          atomicAdd(a.stats + 0, 1ull);
          atomicAdd(a.stats + 1, (unsigned long long)visited);
          atomicAdd(a.stats + 2, (unsigned long long)expanded);
        }
      }
      __syncthreads();
      return;
    }

    // ---- raw candidates: entry nodes, or the frontier's adjacency rows
    int raw_total = 0;
    if (entry_phase) {
      raw_total = a.entry_count < (int)a.n ? a.entry_count : (int)a.n;
    } else {
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
      const int nf = st.nf < a.beam ? st.nf : a.beam;
      expanded += (uint32_t)nf;
      raw_total = nf * a.dg;  // nf == 0: the search is over (graph_index.cpp:160)
    }

    // ---- exact dedup of all raw ids into cand[0..M)
    if (tid == 0) st.ncand = 0;
    if (tid < kXgMaxRanks) {
      xs.cnt[tid] = 0;
      xs.fill[tid] = 0;
    }
    __syncthreads();
    for (int cbase = 0; cbase < raw_total; cbase += kChunk) {
      const int rcount = raw_total - cbase < kChunk ? raw_total - cbase : kChunk;
      uint32_t ids[kRawPerThread];
#pragma unroll
      for (int jj = 0; jj < kRawPerThread; ++jj) {
        const int r = jj * kThreads + tid;
        ids[jj] = kEmpty;
        if (r < rcount) {
          const int g = cbase + r;
          if (entry_phase) {
            ids[jj] = __ldg(a.entry + g);
          } else {
            const uint32_t f = a.dg == 1 ? (uint32_t)g
                             : (a.dg < 256 ? __umulhi((uint32_t)g, dg_magic) : (uint32_t)g / (uint32_t)a.dg);
            const uint32_t col = (uint32_t)g - f * (uint32_t)a.dg;
            ids[jj] = ldg_u32_stream(a.adjacency + (uint64_t)frontier[f] * (uint32_t)a.dg + col);
          }
        }
      }
#if DVSG_XG_BATCH_PROBES
      // exact visited-set inserts for all 8 ids at once: every probe round
      // issues its 8 loads, then its CASes, before using any result (the table
      // is in HBM: latency, not bandwidth, bounds this loop)
      uint32_t hs[kRawPerThread];
      unsigned pend = 0, fresh = 0;
#pragma unroll
      for (int jj = 0; jj < kRawPerThread; ++jj) {
        hs[jj] = (hash_slot(ids[jj]) >> 7) & hmask;
        if (ids[jj] != kEmpty) pend |= 1u << jj;
      }
      while (pend) {
        uint32_t cur[kRawPerThread];
#pragma unroll
        for (int jj = 0; jj < kRawPerThread; ++jj) cur[jj] = (pend >> jj) & 1u ? table[hs[jj]] : 0u;
        // an empty slot is always CASed, so afterwards cur == kEmpty means "claimed"
#pragma unroll
        for (int jj = 0; jj < kRawPerThread; ++jj)
          if (((pend >> jj) & 1u) && cur[jj] == kEmpty) cur[jj] = atomicCAS(table + hs[jj], kEmpty, ids[jj]);
#pragma unroll
        for (int jj = 0; jj < kRawPerThread; ++jj) {
          if (!((pend >> jj) & 1u)) continue;
          if (cur[jj] == kEmpty) {  // claimed: new
            fresh |= 1u << jj;
            pend &= ~(1u << jj);
          } else if (cur[jj] == ids[jj]) {  // already visited
            pend &= ~(1u << jj);
          } else {  // another id: linear probe
            hs[jj] = (hs[jj] + 1u) & hmask;
          }
        }
      }
#endif
#pragma unroll
      for (int jj = 0; jj < kRawPerThread; ++jj) {
        if (jj * kThreads >= rcount) break;  // block-uniform
#if DVSG_XG_BATCH_PROBES
        const bool isnew = (fresh >> jj) & 1u;
#else
        const bool isnew = ids[jj] != kEmpty && visit_insert(table, hmask, ids[jj]);
#endif
        const unsigned bal = __ballot_sync(full, isnew);
        int base = 0;
        if (lane == 0 && bal) base = atomicAdd(&st.ncand, __popc(bal));
        base = __shfl_sync(full, base, 0);
        if (isnew) {
          cand[base + __popc(bal & lt_mask)] = ids[jj];
          atomicAdd(&xs.cnt[ids[jj] / a.shard_rows], 1);
        }
      }
    }
    __syncthreads();
    const int M = st.ncand;
    visited += (uint64_t)M;

    // ---- bucket by owner, reserve inbox ranges, push the requests
    if (tid == 0) {
      xs.off[0] = 0;
      for (int r = 0; r < kXgMaxRanks; ++r) xs.off[r + 1] = xs.off[r] + (r < R ? xs.cnt[r] : 0);
    }
    if (tid < R) {  // one peer atomic per owner reserves this query's inbox range
      const int c = xs.cnt[tid];
      xs.pos[tid] = c ? atomicAdd(a.views[tid].cursor + slot * R + me, (unsigned)c) : 0u;
    }
    __syncthreads();
    for (int i = tid; i < M; i += kThreads) {
      const uint32_t v = cand[i];
      const int o = (int)(v / a.shard_rows);
      buck[xs.off[o] + atomicAdd(&xs.fill[o], 1)] = v;
    }
    __syncthreads();
    for (int i = tid; i < M; i += kThreads) {
      int o = 0;
#pragma unroll
      for (int s = 1; s < kXgMaxRanks; ++s) o += i >= xs.off[s] ? 1 : 0;
      uint64_t* dst = a.views[o].inbox + (uint64_t)me * a.rstride + xs.pos[o] + (uint32_t)(i - xs.off[o]);
      *dst = ((uint64_t)j << 32) | buck[i];
    }
    if (tid < R)
      a.meta[qs * (uint64_t)R + tid] =
          make_uint2(xs.pos[tid], (unsigned)xs.cnt[tid]);
    for (int i = tid; i < P; i += kThreads) gpool[i] = pool[i];
    if (tid == 0) {
      a.psize[qs] = (uint32_t)P;
      a.visited[qs] = visited;
      a.expd[qs] = expanded;
    }
    __syncthreads();
  }
}

// Owner side, per phase: per-CTA table of the inbox segments (acting rank x
// origin) in 32-request warp blocks.
struct ScoreTable {
  uint64_t pref[kXgMaxRanks * kXgMaxRanks + 1];
  uint32_t cnt[kXgMaxRanks * kXgMaxRanks];
  int nseg;
};

__device__ __forceinline__ void score_table(const XgArgs& a, ScoreTable& t) {
  if (threadIdx.x == 0) {
    const int R = a.nranks, slot = a.phase & 1;
    t.nseg = a.rank_n * R;
    t.pref[0] = 0;
    for (int s = 0; s < t.nseg; ++s) {
      const int r = a.rank_lo + s / R, o = s % R;
      const uint32_t c = *a.err ? 0u : __ldcg(a.views[r].cursor + slot * R + o);
      t.cnt[s] = c;
      t.pref[s + 1] = t.pref[s] + (c + 31u) / 32u;
    }
  }
}

// Score warp block b (32 consecutive requests of one origin) and push the
// keys back into the origin's reply range.  Warp-collective.
template <int VPL, typename ACC, int METRIC, bool FULL>
__device__ __forceinline__ void score_warp_block(const XgArgs& a, const ScoreTable& t, uint64_t b,
                                                 uint64_t* wq, uint64_t* wk) {
  // rows in flight per warp: as K1 (search_kernel.cu), 4 (2 at VPL 8) for wide rows
  constexpr int U = VPL >= 4 ? (VPL >= 8 ? 2 : 4) : (VPL >= DVSG_UVEC ? 1 : (DVSG_UVEC / VPL));
  constexpr int LU = ilog2(U);
  const int lane = threadIdx.x & 31;
  const int R = a.nranks;
  int s = 0;
  while (b >= t.pref[s + 1]) ++s;
  const uint32_t* scnt = t.cnt;
  uint32_t cur_q = kEmpty;
  float4 q[VPL];
#pragma unroll
  for (int v = 0; v < VPL; ++v) q[v] = make_float4(0.f, 0.f, 0.f, 0.f);
  const uint64_t* pref = t.pref;
    const int r = a.rank_lo + s / R, o = s % R;
    const uint32_t e0 = (uint32_t)(b - pref[s]) * 32u;
    const int ne = (int)min(32u, scnt[s] - e0);
    const XgView& vr = a.views[r];
    const float* lbase = vr.vec + lane * 4;
    const uint32_t lo = (uint32_t)vr.lo;
    const float* qbase = vr.qall + (uint64_t)o * a.wcap * (uint64_t)a.dpad;
    // stage the 32 requests in smem; rounds read them back as broadcasts
    __syncwarp();  // previous block's readers are done with wq / wk
    wq[lane] = lane < ne ? __ldcg(vr.inbox + (uint64_t)o * a.rstride + e0 + lane) : (uint64_t)lo;
    __syncwarp();
#pragma unroll 1
    for (int round = 0; round < 32 / U; ++round) {
      if (round * U >= ne) break;  // warp-uniform
      uint64_t rq[U];
      if constexpr (U >= 2) {
#pragma unroll
        for (int u2 = 0; u2 < U; u2 += 2) {
          const ulonglong2 w2 = *reinterpret_cast<const ulonglong2*>(wq + round * U + u2);
          rq[u2] = w2.x;
          rq[u2 + 1] = w2.y;
        }
      } else {
        rq[0] = wq[round];
      }
      // one query for the whole round (the common case: requests are grouped
      // by query) -> reload it first, then all U gathers are in flight at once
      const uint32_t q0 = (uint32_t)(rq[0] >> 32);
      bool same = true;
#pragma unroll
      for (int u = 1; u < U; ++u) same &= round * U + u >= ne || (uint32_t)(rq[u] >> 32) == q0;
      if (q0 != cur_q) {
        cur_q = q0;
        load_query<VPL, FULL>(q, qbase + (uint64_t)q0 * (uint32_t)a.dpad, lane, a.dim);
      }
      ACC part[U];
      if (same) {
        float4 x[U][VPL];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          // past ne the slot holds node `lo` (row 0): harmless load, result unused
          const float* row = lbase + (uint64_t)((uint32_t)rq[u] - lo) * (uint32_t)a.dpad;
#pragma unroll
          for (int v = 0; v < VPL; ++v) {
            if (FULL || lane * 4 + 128 * v < a.dpad) x[u][v] = ldg_f4(row + 128 * v);
            else x[u][v] = make_float4(0.f, 0.f, 0.f, 0.f);
          }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          ACC acc = lane_partial<ACC, METRIC>(x[u][0], q[0]);
#pragma unroll
          for (int v = 1; v < VPL; ++v) acc += lane_partial<ACC, METRIC>(x[u][v], q[v]);
          part[u] = acc;
        }
      } else {  // the round spans a query boundary: one vector at a time
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const uint32_t qid = (uint32_t)(rq[u] >> 32);
          if (round * U + u < ne && qid != cur_q) {
            cur_q = qid;
            load_query<VPL, FULL>(q, qbase + (uint64_t)qid * (uint32_t)a.dpad, lane, a.dim);
          }
          const float* row = lbase + (uint64_t)((uint32_t)rq[u] - lo) * (uint32_t)a.dpad;
          ACC acc{};
#pragma unroll
          for (int v = 0; v < VPL; ++v) {
            const float4 xv = (FULL || lane * 4 + 128 * v < a.dpad) ? ldg_f4(row + 128 * v) : make_float4(0.f, 0.f, 0.f, 0.f);
            acc = v == 0 ? lane_partial<ACC, METRIC>(xv, q[0]) : acc + lane_partial<ACC, METRIC>(xv, q[v]);
          }
          part[u] = acc;
        }
      }
      const ACC tot = transpose_reduce<U, ACC>(part, lane);
      if ((lane & ((32 >> LU) - 1)) == 0) {
        const int e = round * U + ((lane >> (5 - LU)) & (U - 1));
        const uint64_t req = wq[e];
        const float dist = finish_dist<ACC, METRIC>(
            tot, lbase - lane * 4 + (uint64_t)((uint32_t)req - lo) * (uint32_t)a.dpad,
            qbase + (uint64_t)(uint32_t)(req >> 32) * (uint32_t)a.dpad, a.dim);
        wk[e] = ((uint64_t)f2ord(dist) << 32) | ((uint64_t)(uint32_t)req << 1);
      }
    }
    __syncwarp();
    if (lane < ne) a.views[o].reply[(uint64_t)r * a.rstride + e0 + lane] = wk[lane];
}

#ifndef DVSG_XG_MINB
#define DVSG_XG_MINB 4  // fp32: 64 registers (fp64 partials keep 3 CTAs/SM)
#endif
// One phase step: expand items of lane `ea` (do_e) and score items of lane
// `sa` (do_s) from one work counter, interleaved, so origin-side work
// (latency / issue bound) and owner-side gathers (HBM bound) share the SMs.
template <int VPL, typename ACC, int METRIC, bool FULL>
__global__ void __launch_bounds__(kThreads, VPL >= 4 ? 2 : sizeof(ACC) == 8 ? 3 : DVSG_XG_MINB)
xg_step(const XgArgs ea, const XgArgs sa, int do_e, int do_s, unsigned long long* counter) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ BlockState st;
  __shared__ XgShared xs;
  __shared__ ScoreTable tab;
  __shared__ __align__(16) uint64_t wreq[kThreads];
  __shared__ uint64_t wkey[kThreads];
  const int tid = threadIdx.x, warp = tid >> 5;
  if (do_s) score_table(sa, tab);
  __syncthreads();
  uint64_t nE = 0;
  if (do_e)
    for (int r = 0; r < ea.rank_n; ++r) nE += ea.wave_n[r];
  const uint64_t nwb = do_s ? tab.pref[tab.nseg] : 0;  // score warp blocks
  // CTAs alternate a preferred kind (so every SM runs both), then help with
  // the other kind; expand items are per CTA, score blocks per warp.
#ifndef DVSG_XG_S_EIGHTHS
#define DVSG_XG_S_EIGHTHS 4  // eighths of the CTAs that start on score blocks
#endif
  const bool prefer_s = do_s && (!do_e || (int)(blockIdx.x & 7) < DVSG_XG_S_EIGHTHS);
  for (int pass = 0; pass < 2; ++pass) {
    const bool s_mode = (pass == 0) == prefer_s;
    if (s_mode) {
      if (!do_s) continue;
      const int lane = tid & 31;
      for (;;) {
        uint64_t b = 0;
        if (lane == 0) b = *sa.err ? ~0ull : atomicAdd(counter + 1, 1ull);
        b = __shfl_sync(0xFFFFFFFFu, b, 0);
        if (b >= nwb) break;
        score_warp_block<VPL, ACC, METRIC, FULL>(sa, tab, b, wreq + warp * 32, wkey + warp * 32);
      }
      __syncthreads();  // every warp is done before the CTA claims expand items
    } else {
      if (!do_e) continue;
      for (;;) {
        if (tid == 0) {
          const uint64_t t = *ea.err ? ~0ull : atomicAdd(counter, 1ull);
          st.unit = t < nE ? t : ~0ull;
        }
        __syncthreads();
        uint64_t u = st.unit;
        __syncthreads();  // st is reused by expand_unit
        if (u == ~0ull) break;
        int rr = 0;
        while (u >= ea.wave_n[rr]) u -= ea.wave_n[rr++];
        expand_unit<VPL, ACC, METRIC, FULL>(ea, rr, (uint32_t)u, smem, st, xs);
      }
    }
  }
  __threadfence_system();  // release this CTA's peer stores before the barrier kernel
}

__global__ void xg_barrier(const XgView* views, int nranks, int me, unsigned epoch, int* err) {
  if (threadIdx.x != 0 || *reinterpret_cast<volatile int*>(err)) return;
  __threadfence_system();
  for (int r = 0; r < nranks; ++r) st_release_sys(views[r].flags + me, epoch);
  const unsigned* mine = views[me].flags;
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

template <int VPL, typename ACC, int METRIC, bool FULL>
cudaError_t launch_step_t(const XgArgs& ea, const XgArgs& sa, int do_e, int do_s,
                          unsigned long long* counter, int num_sms, cudaStream_t stream) {
  auto kern = xg_step<VPL, ACC, METRIC, FULL>;
  const size_t smem = xg_expand_smem_bytes(ea.cap, ea.chp, ea.beam, (int)ea.maxraw);
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int per_sm = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kThreads, smem);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) return cudaErrorInvalidConfiguration;
  kern<<<(unsigned)(per_sm * num_sms), kThreads, smem, stream>>>(ea, sa, do_e, do_s, counter);
  return cudaGetLastError();
}

template <int VPL>
cudaError_t launch_step_v(const XgArgs& ea, const XgArgs& sa, int do_e, int do_s, unsigned long long* ctr,
                          int metric, int accum, int num_sms, cudaStream_t s) {
  const bool full = ea.dpad == 128 * VPL;
  if (accum == 0) {
    if (metric == 0) return full ? launch_step_t<VPL, double, 0, true>(ea, sa, do_e, do_s, ctr, num_sms, s)
                                 : launch_step_t<VPL, double, 0, false>(ea, sa, do_e, do_s, ctr, num_sms, s);
    return full ? launch_step_t<VPL, double, 1, true>(ea, sa, do_e, do_s, ctr, num_sms, s)
                : launch_step_t<VPL, double, 1, false>(ea, sa, do_e, do_s, ctr, num_sms, s);
  }
  if (accum == 2) {
    if (metric == 0) return full ? launch_step_t<VPL, F2, 0, true>(ea, sa, do_e, do_s, ctr, num_sms, s)
                                 : launch_step_t<VPL, F2, 0, false>(ea, sa, do_e, do_s, ctr, num_sms, s);
    return full ? launch_step_t<VPL, F2, 1, true>(ea, sa, do_e, do_s, ctr, num_sms, s)
                : launch_step_t<VPL, F2, 1, false>(ea, sa, do_e, do_s, ctr, num_sms, s);
  }
  if (metric == 0) return full ? launch_step_t<VPL, float, 0, true>(ea, sa, do_e, do_s, ctr, num_sms, s)
                               : launch_step_t<VPL, float, 0, false>(ea, sa, do_e, do_s, ctr, num_sms, s);
  return full ? launch_step_t<VPL, float, 1, true>(ea, sa, do_e, do_s, ctr, num_sms, s)
              : launch_step_t<VPL, float, 1, false>(ea, sa, do_e, do_s, ctr, num_sms, s);
}

}  // namespace

size_t xg_expand_smem_bytes(int cap, int chp, int beam, int maxraw) {
  return sizeof(uint64_t) * (2 * (size_t)cap + (size_t)chp) +
         sizeof(uint32_t) * (2 * (size_t)maxraw + (size_t)((beam + 3) & ~3));
}

cudaError_t launch_xg_step(const XgArgs& ea, const XgArgs& sa, int do_e, int do_s,
                           unsigned long long* counter, int metric, int accum, int num_sms,
                           cudaStream_t s) {
  switch ((ea.dpad + 127) / 128) {
    case 1: return launch_step_v<1>(ea, sa, do_e, do_s, counter, metric, accum, num_sms, s);
    case 2: return launch_step_v<2>(ea, sa, do_e, do_s, counter, metric, accum, num_sms, s);
    case 3:
    case 4: return launch_step_v<4>(ea, sa, do_e, do_s, counter, metric, accum, num_sms, s);
    case 5:
    case 6: return launch_step_v<6>(ea, sa, do_e, do_s, counter, metric, accum, num_sms, s);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_xg_barrier(const XgView* views, int nranks, int me, unsigned epoch, int* err,
                              cudaStream_t stream) {
  xg_barrier<<<1, 32, 0, stream>>>(views, nranks, me, epoch, err);
  return cudaGetLastError();
}

}  // namespace dvsg
