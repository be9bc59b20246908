// shard_kernel.cu -- node-sharded K1: the north-star cross-partition frontier
// exchange, fused into the search kernel over peer memory.
//
// Semantics are exactly beam_search_stats (graph_index.cpp:105-187) over the
// UNSHARDED graph: the traversal, pool, visited set and tie rules are the
// origin CTA's, as in K1; only where a candidate's vector lives changes.
//
// Layout: vectors of node v live on rank owner(v) = v / S; adjacency, global
// ids and entry order are replicated on every rank (12.8 GB at 100M x 32 --
// affordable in 180 GB of HBM), so frontier expansion and dedup stay local.
//
// Per chunk of new candidates (after the exact dedup at the origin):
//   * own-shard ids  -> scored locally, exactly as K1;
//   * remote ids     -> pushed with warp-coalesced NVLink peer stores into the
//                       owner's mailbox for this (origin rank, CTA), with the
//                       query vector, then a doorbell entry in the owner's ring
//                       (peer atomicAdd + store, system-scope release);
//   * the origin CTA scores its local ids, then waits for the owners' replies
//     -- serving its own rank's doorbell ring while it waits, so every waiting
//     CTA is also a server and no rank can starve another (deadlock-free with
//     all CTAs co-resident: the grid is one persistent wave);
//   * owners score the pushed ids against their local rows and push the keys
//     (ord(dist) << 32 | id << 1) back into the origin's reply box, then publish
//     the request's sequence number;
//   * the origin applies the same exact cap-th-key filter to remote keys and
//     merges them with the local survivors: bit-identical to the unsharded K1.
// Traffic per remote candidate: 4 B id out, 8 B key back (+ one query per
// request), instead of a 4*d-byte vector gather over NVLink.
// Termination: a rank is done when all its CTAs finished their units; CTAs
// keep serving until every rank is done (a done rank has no pending requests).
#include <cstdint>
#include <cuda_runtime.h>

#include "dvsg_internal.h"
#include "k1_device.cuh"

namespace dvsg {
namespace {

#ifndef DVSG_SHARD_FENCE_ALL
#define DVSG_SHARD_FENCE_ALL 0  // 1: every storing thread fences (conservative)
#endif

static_assert(kChunk == 2048, "shard_mail_stride/shard_reply_stride assume kChunk == 2048");

__device__ __forceinline__ uint32_t ld_cg_u32(const void* p) {
  return __ldcg(reinterpret_cast<const unsigned int*>(p));
}
__device__ __forceinline__ unsigned ld_volatile(const unsigned* p) {
  return *reinterpret_cast<const volatile unsigned*>(p);
}

struct ShardState {
  int dcnt[8];    // remote ids pushed per destination rank this chunk
  int job;        // doorbell entry being served (-1: none)
  int ready;      // all expected replies arrived
};

// Score ids cand[0..M) (smem) against query q with local rows vloc[id - lo];
// sink(valid, ci, key) is called by every lane (warp-collective).
template <int VPL, typename ACC, int METRIC, typename Sink>
__device__ __forceinline__ void score_ids(const uint32_t* cand, int M, const float4 (&q)[VPL],
                                          const float* qrow, int dim, const float* vloc, uint32_t lo,
                                          int dpad, int lane, int warp, Sink&& sink) {
  constexpr int U = VPL >= 8 ? 1 : (8 / VPL);
  constexpr int LU = ilog2(U);
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
    float4 x[U][VPL];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const bool valid = cb + u < M;
      const float* row = vloc + (uint64_t)(ids_u[u] - lo) * (uint64_t)dpad;
#pragma unroll
      for (int v = 0; v < VPL; ++v) {
        const int b = lane * 4 + 128 * v;
        if (valid && b < dpad) x[u][v] = ldg_f4(row + b);
        else x[u][v] = make_float4(0.f, 0.f, 0.f, 0.f);
      }
    }
    ACC part[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      ACC acc = lane_partial<ACC, METRIC>(x[u][0], q[0]);
#pragma unroll
      for (int v = 1; v < VPL; ++v) acc += lane_partial<ACC, METRIC>(x[u][v], q[v]);
      part[u] = acc;
    }
    const ACC tot = transpose_reduce<U, ACC>(part, lane);
    const int myu = (lane >> (5 - LU)) & (U - 1);
    const int ci = cb + myu;
    const bool valid = (lane & ((32 >> LU) - 1)) == 0 && ci < M;
    uint64_t key = 0;
    if (valid) {
      const float dist = finish_dist<ACC, METRIC>(tot, vloc + (uint64_t)(cand[ci] - lo) * (uint64_t)dpad, qrow, dim);
      key = ((uint64_t)f2ord(dist) << 32) | ((uint64_t)cand[ci] << 1);
    }
    sink(valid, ci, key);
  }
}

// Claim one doorbell entry of rank `me` (thread 0 only); -1 if the ring is empty.
__device__ __forceinline__ int try_claim(const ShardView& v, uint32_t ring_mask) {
  const unsigned h = ld_volatile(v.ring_head);
  const unsigned t = ld_volatile(v.ring_tail);
  if ((int)(t - h) <= 0) return -1;
  if (atomicCAS(v.ring_head, h, h + 1) != h) return -1;
  volatile uint32_t* slot = v.ring + (h & ring_mask);
  uint32_t e;
  while ((e = *slot) == 0u) __nanosleep(32);  // producer reserved, not yet written
  *slot = 0u;
  __threadfence_system();  // acquire: mailbox contents written before the doorbell
  return (int)(e - 1u);
}

// Serve one request (whole CTA): score the pushed ids against this rank's rows
// and push the keys back into the origin's reply box.  Uses `cand` as scratch.
template <int VPL, typename ACC, int METRIC>
__device__ void serve_request(const ShardArgs& sh, int me, int job, uint32_t* cand, int dim,
                              int dpad, uint32_t lo, int tid, int lane, int warp) {
  const int o = job >> 16, c = job & 0xFFFF;
  const ShardView& mine = sh.views[me];
  const unsigned char* mb = mine.mail + ((size_t)o * sh.gpr + c) * sh.mail_stride;
  const uint32_t seq = ld_cg_u32(mb);
  const int cnt = (int)ld_cg_u32(mb + 4);
  const float* qsrc = reinterpret_cast<const float*>(mb + 16);
  const uint32_t* isrc = reinterpret_cast<const uint32_t*>(mb + 16 + 4 * dpad);
  float4 qs[VPL];
#pragma unroll
  for (int v = 0; v < VPL; ++v) {
    const int b = lane * 4 + 128 * v;
    qs[v] = b < dpad ? __ldcg(reinterpret_cast<const float4*>(qsrc + b))
                     : make_float4(0.f, 0.f, 0.f, 0.f);
  }
  for (int i = tid; i < cnt; i += kThreads) cand[i] = __ldcg(isrc + i);
  __syncthreads();
  unsigned char* rb = sh.views[o].reply + ((size_t)c * sh.nranks + me) * sh.reply_stride;
  uint64_t* keys = reinterpret_cast<uint64_t*>(rb + 16);
  score_ids<VPL, ACC, METRIC>(cand, cnt, qs, qsrc, dim, mine.vec, lo, dpad, lane, warp,
                              [&](bool valid, int ci, uint64_t key) {
                                if (valid) keys[ci] = key;  // NVLink peer store
                              });
#if DVSG_SHARD_FENCE_ALL
  __threadfence_system();
#endif
  __syncthreads();
  if (tid == 0) {
    __threadfence_system();  // release the whole CTA's key stores (cumulative after the barrier)
    volatile uint32_t* hdr = reinterpret_cast<volatile uint32_t*>(rb);
    hdr[1] = (uint32_t)cnt;
    __threadfence_system();
    hdr[0] = seq;  // release: the origin polls this
  }
  __syncthreads();
  (void)dim;
}

struct ShardBlockState {
  BlockState b;
  ShardState s;
};

template <int VPL, typename ACC, int METRIC>
__global__ void __launch_bounds__(kThreads, 4)
    search_sharded_kernel(const SearchArgs a, const ShardArgs sh) {
  constexpr int U = VPL >= 8 ? 1 : (8 / VPL);
  (void)U;
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ ShardBlockState sst;
  BlockState& st = sst.b;
  ShardState& ss = sst.s;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int me = sh.rank_self >= 0 ? sh.rank_self : (int)(blockIdx.x / sh.gpr);
  const int cta = sh.rank_self >= 0 ? (int)blockIdx.x : (int)(blockIdx.x % sh.gpr);
  const ShardView& mine = sh.views[me];
  const uint32_t lo = (uint32_t)((uint64_t)me * sh.shard_rows);
  const uint64_t shard_rows = sh.shard_rows;

  uint64_t* pool = reinterpret_cast<uint64_t*>(smem);
  uint64_t* pool_alt = pool + a.cap;
  uint64_t* surv = pool_alt + a.cap;
  uint32_t* cand = reinterpret_cast<uint32_t*>(surv + a.chp);
  uint32_t* frontier = cand + kChunk;
  uint32_t* table = a.hash_global + (size_t)blockIdx.x * (size_t)a.hsize;
  const uint32_t hmask = (uint32_t)a.hsize - 1u;
  const unsigned full = 0xFFFFFFFFu;
  const unsigned lt_mask = (1u << lane) - 1u;

  const uint64_t ulo = sh.rank_self >= 0 ? 0 : (uint64_t)me * sh.units_per_rank;
  uint64_t uhi = sh.rank_self >= 0 ? a.nunits : ulo + sh.units_per_rank;
  if (uhi > a.nunits) uhi = a.nunits;
  uint32_t myseq = 0;

  // dedicated servers skip the search loop and drain the ring from the start
  for (; cta < sh.origin_ctas;) {
    if (tid == 0) st.unit = ulo + atomicAdd(mine.work, 1ull);
    __syncthreads();
    const uint64_t unit = st.unit;
    if (unit >= uhi) break;

    const uint32_t qi = a.unit_query[unit];
    const uint32_t n = a.parts[0].n;  // the whole (unsharded) graph
#ifdef DVSG_SHARD_PROFILE
    const long long t_unit0 = clock64();
#endif

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
    for (int i = tid; i < a.hsize; i += kThreads) table[i] = kEmpty;
    __syncthreads();

    int P = 0;
    uint64_t thresh = ~0ull;
    uint64_t visited = 0;
    uint64_t expanded = 0;
    const int entries = a.entry_count < (int)n ? a.entry_count : (int)n;
    int nf = 0;
    for (int it = -1; it < a.iters; ++it) {
      int raw_total;
      if (it < 0) {
        raw_total = entries;
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
        nf = st.nf < a.beam ? st.nf : a.beam;
        if (nf == 0) break;
        expanded += (uint64_t)nf;
        raw_total = nf * a.dg;
      }

      for (int cbase = 0; cbase < raw_total; cbase += kChunk) {
        const int rcount = raw_total - cbase < kChunk ? raw_total - cbase : kChunk;
        if (tid == 0) {
          st.ncand = 0;
          st.nsurv = 0;
        }
        if (tid < 8) ss.dcnt[tid] = 0;
        uint32_t ids[kRawPerThread];
#pragma unroll
        for (int j = 0; j < kRawPerThread; ++j) {
          const int r = j * kThreads + tid;
          ids[j] = kEmpty;
          if (r < rcount) {
            const int g = cbase + r;
            if (it < 0) {
              ids[j] = __ldg(a.entry + g);
            } else {
              const int f = g / a.dg, jj = g - f * a.dg;
              ids[j] = __ldg(a.adjacency + (uint64_t)frontier[f] * (uint64_t)a.dg + jj);
            }
          }
        }
        __syncthreads();
        // ---- exact dedup; new own-shard ids -> cand, remote ids -> owner mailboxes
        bool pushed = false;
#pragma unroll
        for (int j = 0; j < kRawPerThread; ++j) {
          if (j * kThreads >= rcount) break;  // block-uniform
          const bool isnew = ids[j] != kEmpty && visit_insert(table, hmask, ids[j]);
          const int owner = isnew ? (int)(ids[j] / shard_rows) : -1;
          const bool local = isnew && owner == me;
          unsigned bal = __ballot_sync(full, local);
          int base = 0;
          if (lane == 0 && bal) base = atomicAdd(&st.ncand, __popc(bal));
          base = __shfl_sync(full, base, 0);
          if (local) cand[base + __popc(bal & lt_mask)] = ids[j];
          const unsigned remote_bal = __ballot_sync(full, isnew && !local);
          if (remote_bal) {
            for (int d = 0; d < sh.nranks; ++d) {
              if (d == me) continue;
              bal = __ballot_sync(full, owner == d && !local);
              if (!bal) continue;
              int b2 = 0;
              if (lane == 0) b2 = atomicAdd(&ss.dcnt[d], __popc(bal));
              b2 = __shfl_sync(full, b2, 0);
              if (owner == d && !local) {
                unsigned char* mb = sh.views[d].mail + ((size_t)me * sh.gpr + cta) * sh.mail_stride;
                reinterpret_cast<uint32_t*>(mb + 16 + 4 * a.dpad)[b2 + __popc(bal & lt_mask)] = ids[j];
                pushed = true;
              }
            }
          }
        }
        __syncthreads();
        const int M = st.ncand;
        int nremote = 0;
        unsigned expect = 0;
        for (int d = 0; d < sh.nranks; ++d) {
          const int cdd = ss.dcnt[d];
          nremote += cdd;
          if (cdd > 0) expect |= 1u << d;
        }
        visited += (uint64_t)(M + nremote);
        if (expect) {
          ++myseq;
          // query vector + header into every destination mailbox, then the doorbell
          if (warp == 0) {
            for (int d = 0; d < sh.nranks; ++d) {
              if (!(expect >> d & 1u)) continue;
              unsigned char* mb = sh.views[d].mail + ((size_t)me * sh.gpr + cta) * sh.mail_stride;
              float* qdst = reinterpret_cast<float*>(mb + 16);
#pragma unroll
              for (int v = 0; v < VPL; ++v) {
                const int b = lane * 4 + 128 * v;
                if (b < a.dpad) *reinterpret_cast<float4*>(qdst + b) = q[v];
              }
              if (lane == 0) {
                reinterpret_cast<uint32_t*>(mb)[0] = myseq;
                reinterpret_cast<uint32_t*>(mb)[1] = (uint32_t)ss.dcnt[d];
              }
            }
            pushed = true;
          }
#if DVSG_SHARD_FENCE_ALL
          if (pushed) __threadfence_system();  // release this thread's peer stores
#endif
          __syncthreads();
          if (tid < sh.nranks && (expect >> tid & 1u)) {
            // release (cumulative fence after the CTA barrier, as in grid sync):
            // every thread's mailbox stores are ordered before the doorbell
            __threadfence_system();
            const ShardView& dst = sh.views[tid];
            const unsigned slot = atomicAdd(dst.ring_tail, 1u);
            reinterpret_cast<volatile uint32_t*>(dst.ring)[slot & sh.ring_mask] =
                ((uint32_t)me << 16 | (uint32_t)cta) + 1u;
          }
        }

        // ---- score own-shard candidates (as K1)
        score_ids<VPL, ACC, METRIC>(cand, M, q, a.queries + (uint64_t)qi * (uint64_t)a.dim, a.dim, mine.vec, lo,
                                    a.dpad, lane, warp,
                                    [&](bool valid, int, uint64_t key) {
                                      const bool pass = valid && key < thresh;
                                      const unsigned b = __ballot_sync(full, pass);
                                      int base = 0;
                                      if (lane == 0 && b) base = atomicAdd(&st.nsurv, __popc(b));
                                      base = __shfl_sync(full, base, 0);
                                      if (pass) surv[base + __popc(b & lt_mask)] = key;
                                    });
        if (expect) {
          // ---- wait for the owners' keys, serving our own ring meanwhile
#ifdef DVSG_SHARD_PROFILE
          const long long t_wait0 = clock64();
          long long t_serve = 0;
#endif
          for (;;) {
            __syncthreads();
            if (tid == 0) {
              bool all = true;
              for (int d = 0; d < sh.nranks; ++d) {
                if (!(expect >> d & 1u)) continue;
                const unsigned char* rb = mine.reply + ((size_t)cta * sh.nranks + d) * sh.reply_stride;
                if (ld_volatile(reinterpret_cast<const unsigned*>(rb)) != myseq) all = false;
              }
              if (all) __threadfence_system();  // acquire the keys
              ss.ready = all;
              ss.job = all ? -1 : try_claim(mine, sh.ring_mask);
            }
            __syncthreads();
            if (ss.ready) break;
            if (ss.job >= 0) {
#ifdef DVSG_SHARD_PROFILE
              const long long t0 = clock64();
#endif
              serve_request<VPL, ACC, METRIC>(sh, me, ss.job, cand, a.dim, a.dpad, lo, tid, lane,
                                              warp);
#ifdef DVSG_SHARD_PROFILE
              t_serve += clock64() - t0;
#endif
            } else if (tid == 0) {
              __nanosleep(64);
            }
          }
#ifdef DVSG_SHARD_PROFILE
          if (tid == 0 && a.stats) {
            atomicAdd(a.stats + 3, (unsigned long long)(clock64() - t_wait0 - t_serve));
            atomicAdd(a.stats + 4, (unsigned long long)t_serve);
            atomicAdd(a.stats + 5, 1ull);
          }
#endif
          // remote keys through the same exact cap-th-key filter
          for (int d = 0; d < sh.nranks; ++d) {
            if (!(expect >> d & 1u)) continue;
            const unsigned char* rb = mine.reply + ((size_t)cta * sh.nranks + d) * sh.reply_stride;
            const int cnt = (int)ld_cg_u32(rb + 4);
            const uint64_t* keys = reinterpret_cast<const uint64_t*>(rb + 16);
            for (int b0 = 0; b0 < cnt; b0 += kThreads) {
              const int i = b0 + tid;
              const uint64_t key = i < cnt ? __ldcg(keys + i) : ~0ull;
              const bool pass = i < cnt && key < thresh;
              const unsigned b = __ballot_sync(full, pass);
              int base = 0;
              if (lane == 0 && b) base = atomicAdd(&st.nsurv, __popc(b));
              base = __shfl_sync(full, base, 0);
              if (pass) surv[base + __popc(b & lt_mask)] = key;
            }
          }
        }
        __syncthreads();
        const int S = st.nsurv;
        __syncthreads();
        if (S == 0) continue;
        sort_keys(surv, S, tid);
        const int outn = P + S < a.cap ? P + S : a.cap;
        merge_path(pool, P, surv, S, pool_alt, outn, tid);
        __syncthreads();
        {
          uint64_t* t = pool;
          pool = pool_alt;
          pool_alt = t;
        }
        P = outn;
        thresh = P == a.cap ? pool[a.cap - 1] : ~0ull;
      }
    }

    const int want = a.k < P ? a.k : P;
    if (want > 0) {
      const uint32_t dk = (uint32_t)(pool[want - 1] >> 32);
      int lo2 = want, hi2 = P;
      while (lo2 < hi2) {
        const int mid = (lo2 + hi2) >> 1;
        if ((uint32_t)(pool[mid] >> 32) <= dk) lo2 = mid + 1; else hi2 = mid;
      }
      const int m = lo2;
      for (int i = tid; i < m; i += kThreads) {
        const uint64_t key = pool[i];
        const uint32_t local = (uint32_t)(key >> 1) & 0x7FFFFFFFu;
        surv[i] = (key & 0xFFFFFFFF00000000ull) | (uint64_t)__ldg(a.gids + local);
      }
      __syncthreads();
      sort_keys(surv, m, tid);
      for (int i = tid; i < want; i += kThreads) {
        const uint64_t key = surv[i];
        a.out_ids[unit * (uint64_t)a.k + i] = (uint32_t)key;
        a.out_dists[unit * (uint64_t)a.k + i] = ord2f((uint32_t)(key >> 32));
      }
    }
#ifdef DVSG_SHARD_PROFILE
    if (tid == 0 && a.stats) atomicAdd(a.stats + 6, (unsigned long long)(clock64() - t_unit0));
#endif
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

  // ---- this CTA's units are done: announce, then serve until every rank is done
  if (tid == 0) {
    __threadfence_system();
    const unsigned prev = atomicAdd(mine.finished, 1u);
    if (prev == (unsigned)sh.gpr - 1u)
      for (int d = 0; d < sh.nranks; ++d) atomicAdd(sh.views[d].done, 1u);
  }
  for (;;) {
    __syncthreads();
    if (tid == 0) {
      ss.ready = ld_volatile(mine.done) >= (unsigned)sh.nranks;
      ss.job = ss.ready ? -1 : try_claim(mine, sh.ring_mask);
    }
    __syncthreads();
    if (ss.ready) break;
    if (ss.job >= 0) {
      serve_request<VPL, ACC, METRIC>(sh, me, ss.job, cand, a.dim, a.dpad, lo, tid, lane, warp);
    } else if (tid == 0) {
      __nanosleep(128);
    }
  }
}

template <int VPL, typename ACC, int METRIC>
cudaError_t launch_sh_t(const SearchArgs& a, const ShardArgs& sh, int num_sms, cudaStream_t stream,
                        int* grid_out, int* gpr_out, int* per_sm_out) {
  auto kern = search_sharded_kernel<VPL, ACC, METRIC>;
  const size_t smem = search_smem_bytes(a.cap, a.chp, a.beam, a.hsize, false);
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int per_sm = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kThreads, smem);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) return cudaErrorInvalidConfiguration;
  if (per_sm_out) {
    *per_sm_out = per_sm;
    return cudaSuccess;
  }
  // one persistent wave: every CTA must be co-resident (they wait on each other)
  const int resident = per_sm * num_sms;
  int gpr = sh.gpr;
  const int ranks_here = sh.rank_self >= 0 ? 1 : sh.nranks;
  if (gpr * ranks_here > resident || gpr < 1) return cudaErrorInvalidConfiguration;
  if (grid_out) *grid_out = gpr * ranks_here;
  if (gpr_out) *gpr_out = gpr;
  kern<<<(unsigned)(gpr * ranks_here), kThreads, smem, stream>>>(a, sh);
  return cudaGetLastError();
}

template <int VPL>
cudaError_t launch_sh_v(const SearchArgs& a, const ShardArgs& sh, int metric, int accum, int num_sms,
                        cudaStream_t s, int* g, int* gpr, int* per_sm) {
  if (accum == 0) {
    return metric == 0 ? launch_sh_t<VPL, double, 0>(a, sh, num_sms, s, g, gpr, per_sm)
                       : launch_sh_t<VPL, double, 1>(a, sh, num_sms, s, g, gpr, per_sm);
  }
  if (accum == 2) {
    return metric == 0 ? launch_sh_t<VPL, F2, 0>(a, sh, num_sms, s, g, gpr, per_sm)
                       : launch_sh_t<VPL, F2, 1>(a, sh, num_sms, s, g, gpr, per_sm);
  }
  return metric == 0 ? launch_sh_t<VPL, float, 0>(a, sh, num_sms, s, g, gpr, per_sm)
                     : launch_sh_t<VPL, float, 1>(a, sh, num_sms, s, g, gpr, per_sm);
}

cudaError_t dispatch_sh(const SearchArgs& a, const ShardArgs& sh, int metric, int accum,
                        int num_sms, cudaStream_t stream, int* g, int* gpr, int* per_sm) {
  switch ((a.dpad + 127) / 128) {
    case 1: return launch_sh_v<1>(a, sh, metric, accum, num_sms, stream, g, gpr, per_sm);
    case 2: return launch_sh_v<2>(a, sh, metric, accum, num_sms, stream, g, gpr, per_sm);
    case 3:
    case 4: return launch_sh_v<4>(a, sh, metric, accum, num_sms, stream, g, gpr, per_sm);
    case 5:
    case 6: return launch_sh_v<6>(a, sh, metric, accum, num_sms, stream, g, gpr, per_sm);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace

int search_sharded_blocks_per_sm(const SearchArgs& a, int metric, int accum) {
  ShardArgs dummy{};
  int per_sm = 0;
  if (dispatch_sh(a, dummy, metric, accum, 1, nullptr, nullptr, nullptr, &per_sm) != cudaSuccess)
    return 0;
  return per_sm;
}

cudaError_t launch_search_sharded(const SearchArgs& a, const ShardArgs& sh, int metric, int accum,
                                  int num_sms, cudaStream_t stream, int* grid_out, int* gpr_out) {
  if (sh.nranks < 1 || sh.nranks > 8) return cudaErrorInvalidValue;
  return dispatch_sh(a, sh, metric, accum, num_sms, stream, grid_out, gpr_out, nullptr);
}

}  // namespace dvsg
