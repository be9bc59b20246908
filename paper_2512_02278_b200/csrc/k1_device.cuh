// k1_device.cuh -- device helpers shared by K1 (search_kernel.cu) and the
// node-sharded K1 (shard_kernel.cu).  Included inside each .cu translation
// unit (internal linkage), not a public header.
#pragma once
#include <cstdint>
#include <type_traits>
#include <cuda_runtime.h>

#include "dvsg_internal.h"

namespace dvsg {
namespace {

constexpr int kRawPerThread = kChunk / kThreads;  // 8

__device__ __forceinline__ uint32_t f2ord(float f) {
  if (f == 0.0f) f = 0.0f;  // -0.0 == +0.0 in the reference's comparisons
  const uint32_t u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

__device__ __forceinline__ float ord2f(uint32_t o) {
  const uint32_t u = (o & 0x80000000u) ? (o & 0x7FFFFFFFu) : ~o;
  return __uint_as_float(u);
}

__device__ __forceinline__ uint32_t hash_slot(uint32_t id) { return id * 0x9E3779B1u; }

// Exact insert; returns true when `id` was not present.
#ifndef DVSG_HASH_CAS_FIRST
#define DVSG_HASH_CAS_FIRST 0  // measured: CAS-first -10% (the plain probe loads hit L1)
#endif
__device__ __forceinline__ bool visit_insert(uint32_t* table, uint32_t mask, uint32_t id) {
  uint32_t h = (hash_slot(id) >> 7) & mask;
  for (;;) {
#if DVSG_HASH_CAS_FIRST
    const uint32_t cur = atomicCAS(table + h, kEmpty, id);  // claims the slot or returns its id
    if (cur == kEmpty) return true;
    if (cur == id) return false;
#else
    uint32_t cur = table[h];
    if (cur == id) return false;
    if (cur == kEmpty) {
      cur = atomicCAS(table + h, kEmpty, id);
      if (cur == kEmpty) return true;
      if (cur == id) return false;
    }
#endif
    h = (h + 1) & mask;
  }
}

constexpr unsigned kFull = 0xFFFFFFFFu;

#ifndef DVSG_SORT_ROLLED
#define DVSG_SORT_ROLLED 1  // measured: rolled stage loops beat full unroll (I-cache)
#endif
#ifndef DVSG_SORT_NOINLINE
#define DVSG_SORT_NOINLINE 0
#endif
#ifndef DVSG_SCORE_ROLLED
#define DVSG_SCORE_ROLLED 0
#endif

__host__ __device__ constexpr int ilog2(int x) { return x <= 1 ? 0 : 1 + ilog2(x >> 1); }

__device__ __forceinline__ uint64_t umin64(uint64_t a, uint64_t b) { return a < b ? a : b; }
__device__ __forceinline__ uint64_t umax64(uint64_t a, uint64_t b) { return a < b ? b : a; }

// Register-tiled bitonic sort of N = KPT * NT keys, ascending.  Element
// e = t * KPT + r lives in x[r] of thread t.  Partners closer than KPT are in
// the same thread (register compare-swap), closer than 32 * KPT in the same
// warp (shuffles); only the remaining stages go through shared memory
// (r-major, conflict-free) with barriers.  Fully unrolled, but sort_keys is
// __noinline__ so each kernel carries one copy of each network.
// Element e = t*KPT + r with t*KPT a multiple of KPT, so the direction bit
// (e & k) is (r & k) for k < KPT (a compile-time constant per register) and
// (t*KPT & k) for k >= KPT (one bit per stage, shared by all r).
template <int J, int KPT>
__device__ __forceinline__ void cmpswap_regs(uint64_t (&x)[KPT], int e0, int k) {
  const bool up_hi = (e0 & k) == 0;
#pragma unroll
  for (int r = 0; r < KPT; ++r) {
    const int r2 = r ^ J;
    if (r2 > r) {
      const bool up = k < KPT ? ((r & k) == 0) : up_hi;
      const uint64_t a = x[r], b = x[r2];
      const bool sw = (b < a) == up;  // keys unique: never equal
      x[r] = sw ? b : a;
      x[r2] = sw ? a : b;
    }
  }
}

template <int KPT, int NT>
__device__ __forceinline__ void bitonic_regs(uint64_t (&x)[KPT], int t, uint64_t* s) {
  constexpr int LOGN = ilog2(KPT * NT);
  const int e0 = t * KPT;
#if DVSG_SORT_ROLLED
#pragma unroll 1
#else
#pragma unroll
#endif
  for (int lk = 1; lk <= LOGN; ++lk) {
    const int k = 1 << lk;
    const bool up_stage = (e0 & k) == 0;  // valid for every stage with k >= KPT
#if DVSG_SORT_ROLLED
#pragma unroll 1
#else
#pragma unroll
#endif
    for (int lj = lk - 1; lj >= 0; --lj) {
      const int j = 1 << lj;
      if (j < KPT) {
        if (j == 1) cmpswap_regs<1, KPT>(x, e0, k);
        if (KPT > 2 && j == 2) cmpswap_regs<(KPT > 2 ? 2 : 1), KPT>(x, e0, k);
        if (KPT > 4 && j == 4) cmpswap_regs<(KPT > 4 ? 4 : 1), KPT>(x, e0, k);
      } else if (j < KPT * 32) {
        const int lm = j / KPT;
        const bool keep_min = ((t & lm) == 0) == up_stage;
#pragma unroll
        for (int r = 0; r < KPT; ++r) {
          const uint64_t o = __shfl_xor_sync(kFull, x[r], lm);
          x[r] = ((o < x[r]) == keep_min) ? o : x[r];
        }
      } else {
        const int tm = j / KPT;
        const bool keep_min = ((t & tm) == 0) == up_stage;
#pragma unroll
        for (int r = 0; r < KPT; ++r) s[r * NT + t] = x[r];
        __syncthreads();
#pragma unroll
        for (int r = 0; r < KPT; ++r) {
          const uint64_t o = s[r * NT + (t ^ tm)];
          x[r] = ((o < x[r]) == keep_min) ? o : x[r];
        }
        __syncthreads();
      }
    }
  }
}

template <int KPT>
__device__ __forceinline__ void sort_block(uint64_t* s, int n, int tid) {
  uint64_t x[KPT];
#pragma unroll
  for (int r = 0; r < KPT; ++r) {
    const int e = tid * KPT + r;
    x[r] = e < n ? s[e] : ~0ull;
  }
  __syncthreads();
  bitonic_regs<KPT, kThreads>(x, tid, s);
#pragma unroll
  for (int r = 0; r < KPT; ++r) {
    const int e = tid * KPT + r;
    if (e < n) s[e] = x[r];
  }
  __syncthreads();
}

template <int KPT>
__device__ __forceinline__ void sort_warp0(uint64_t* s, int n, int tid) {
  if (tid < 32) {
    uint64_t x[KPT];
#pragma unroll
    for (int r = 0; r < KPT; ++r) {
      const int e = tid * KPT + r;
      x[r] = e < n ? s[e] : ~0ull;
    }
    bitonic_regs<KPT, 32>(x, tid, nullptr);
#pragma unroll
    for (int r = 0; r < KPT; ++r) {
      const int e = tid * KPT + r;
      if (e < n) s[e] = x[r];
    }
  }
  __syncthreads();
}

// Plain shared-memory bitonic for the rare n > 2048 (final sort when cap > 2048).
__device__ void sort_smem_large(uint64_t* s, int n, int tid) {
  int np = 1;
  while (np < n) np <<= 1;
  for (int i = n + tid; i < np; i += kThreads) s[i] = ~0ull;
  __syncthreads();
  for (int k = 2; k <= np; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int p = tid; p < (np >> 1); p += kThreads) {
        const int i = ((p & ~(j - 1)) << 1) | (p & (j - 1));
        const int ixj = i | j;
        const uint64_t a = s[i], b = s[ixj];
        const bool up = (i & k) == 0;
        if ((a > b) == up) {
          s[i] = b;
          s[ixj] = a;
        }
      }
      __syncthreads();
    }
  }
}

// Sort s[0..n) ascending in place (block-uniform call; s holds >= pow2(n)).
#if DVSG_SORT_NOINLINE
__device__ __noinline__
#else
__device__ __forceinline__
#endif
void sort_keys(uint64_t* s, int n, int tid) {
  if (n <= 1) return;
  if (n <= 32) return sort_warp0<1>(s, n, tid);
  if (n <= 64) return sort_warp0<2>(s, n, tid);
  if (n <= 128) return sort_warp0<4>(s, n, tid);
  if (n <= 256) return sort_block<1>(s, n, tid);
  if (n <= 512) return sort_block<2>(s, n, tid);
  if (n <= 1024) return sort_block<4>(s, n, tid);
  if (n <= 2048) return sort_block<8>(s, n, tid);
  return sort_smem_large(s, n, tid);
}

// out[0..outn) = first outn of merge(A[0..na), B[0..nb)); keys unique.
// Merge path: each of nthreads threads owns a contiguous slice of the output.
__device__ __forceinline__ void merge_path(const uint64_t* A, int na, const uint64_t* B, int nb,
                                           uint64_t* out, int outn, int tid, int nthreads = kThreads) {
  const int per = (outn + nthreads - 1) / nthreads;
  const int o0 = min(tid * per, outn), o1 = min(o0 + per, outn);
  if (o0 >= o1) return;
  int lo = max(0, o0 - nb), hi = min(o0, na);
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (A[mid] < B[o0 - mid - 1]) lo = mid + 1; else hi = mid;
  }
  int ia = lo, ib = o0 - lo;
  for (int o = o0; o < o1; ++o) {
    const bool takeA = ib >= nb || (ia < na && A[ia] < B[ib]);
    out[o] = takeA ? A[ia++] : B[ib++];
  }
}

// One warp sorts s[0..n) (n <= 32 * KPT) in registers; no block barrier.
template <int KPT>
__device__ __forceinline__ void warp_sort_slice(uint64_t* s, int n, int lane) {
  uint64_t x[KPT];
#pragma unroll
  for (int r = 0; r < KPT; ++r) {
    const int e = lane * KPT + r;
    x[r] = e < n ? s[e] : ~0ull;
  }
  bitonic_regs<KPT, 32>(x, lane, nullptr);
#pragma unroll
  for (int r = 0; r < KPT; ++r) {
    const int e = lane * KPT + r;
    if (e < n) s[e] = x[r];
  }
}

// Sort s[0..n) (n <= 2048, block-uniform call): every warp sorts one eighth
// in registers (bitonic, shuffles only), then three merge-path levels
// ping-pong between s and tmp (>= n entries).  O(n log n) compare work
// instead of the full block bitonic's O(n log^2 n) with smem stages.
// Returns the buffer holding the sorted keys.
__device__ __forceinline__ uint64_t* sort_runs(uint64_t* s, int n, uint64_t* tmp, int tid) {
  if (n <= 128) {
    sort_keys(s, n, tid);
    return s;
  }
  const int lane = tid & 31, warp = tid >> 5;
  const int L = (n + kWarps - 1) / kWarps;  // <= 256
  const int base = warp * L;
  const int cnt = n - base < 0 ? 0 : (n - base < L ? n - base : L);
  if (L <= 64) warp_sort_slice<2>(s + base, cnt, lane);
  else if (L <= 128) warp_sort_slice<4>(s + base, cnt, lane);
  else warp_sort_slice<8>(s + base, cnt, lane);
  __syncthreads();
  uint64_t* src = s;
  uint64_t* dst = tmp;
  int Lr = L;
#pragma unroll 1
  for (int pairs = kWarps / 2; pairs >= 1; pairs >>= 1) {
    const int tpp = kThreads / pairs;
    const int i = tid / tpp, t = tid - i * tpp;
    const int a0 = i * 2 * Lr;
    const int na = n - a0 < 0 ? 0 : (n - a0 < Lr ? n - a0 : Lr);
    const int b0 = a0 + Lr;
    const int nb = n - b0 < 0 ? 0 : (n - b0 < Lr ? n - b0 : Lr);
    merge_path(src + a0, na, src + b0, nb, dst + a0, na + nb, t, tpp);
    __syncthreads();
    uint64_t* x = src;
    src = dst;
    dst = x;
    Lr *= 2;
  }
  return src;
}

// Compensated f32 accumulator (DVSG_ACCUM_F32C): hi carries the running
// TwoSum of the rounded terms, lo the sum of every rounding error (TwoSum,
// FMA TwoProd, and for L2 the exact-difference error).  ~48-bit effective
// mantissa: agrees with the fp64 sum after the final f32 rounding except
// within ~2^-24 ulp of a rounding boundary (an id-identity mode, not parity).
struct F2 {
  float hi, lo;
};
__device__ __forceinline__ F2 f2_add(F2 a, F2 b) {
  const float s = __fadd_rn(a.hi, b.hi);
  const float bb = __fsub_rn(s, a.hi);
  const float e = __fadd_rn(__fsub_rn(a.hi, __fsub_rn(s, bb)), __fsub_rn(b.hi, bb));
  return F2{s, __fadd_rn(e, __fadd_rn(a.lo, b.lo))};
}
__device__ __forceinline__ F2 operator+(F2 a, F2 b) { return f2_add(a, b); }
__device__ __forceinline__ F2& operator+=(F2& a, F2 b) {
  a = f2_add(a, b);
  return a;
}
__device__ __forceinline__ float shfl_xor(float v, int off) { return __shfl_xor_sync(kFull, v, off); }
__device__ __forceinline__ double shfl_xor(double v, int off) { return __shfl_xor_sync(kFull, v, off); }
__device__ __forceinline__ F2 shfl_xor(F2 v, int off) {
  return F2{__shfl_xor_sync(kFull, v.hi, off), __shfl_xor_sync(kFull, v.lo, off)};
}
// the accumulated sum rounded once to f32 (graph_index/distance.cpp: the
// fp64 sum cast to float); negation commutes with round-to-nearest-even
__device__ __forceinline__ float acc_to_f32(float v) { return v; }
__device__ __forceinline__ float acc_to_f32(double v) { return (float)v; }
__device__ __forceinline__ float acc_to_f32(F2 v) { return __fadd_rn(v.hi, v.lo); }

// f64 mode, squared L2: exact by construction.  The lanes add the same fp64
// terms ((double)x - (double)q)^2 as squared_l2 (distance.cpp:19-27), in a tree
// instead of i = 0..d-1; both sums lie within (d-1) 2^-53 S of the exact sum of
// those terms (all >= 0), so the two differ by at most e = (2d+2) 2^-53 tot.
// If [tot - e, tot + e] holds no f32 rounding midpoint, both round to the same
// float; otherwise (about one distance in 10^6-10^7) one lane redoes the sum in
// the reference's order from the row and the query in memory.
template <typename VT>
__device__ __noinline__ float l2_f64_sequential(const VT* __restrict__ row, const float* __restrict__ qrow,
                                                int dim) {
  double s = 0.0;
  for (int i = 0; i < dim; ++i) {
    const double t = __dsub_rn((double)row[i], (double)qrow[i]);
    s = __dadd_rn(s, __dmul_rn(t, t));
  }
  return (float)s;
}
template <typename VT>
__device__ __forceinline__ float l2_f64_exact(double tot, const VT* row, const float* qrow, int dim) {
  const float f = (float)tot;
  const double fd = (double)f;
  const double up = (double)__uint_as_float(__float_as_uint(f) + 1u);  // next float up (f >= 0)
  const double dn = f > 0.f ? (double)__uint_as_float(__float_as_uint(f) - 1u) : -1.0;
  const double e = (double)(2 * dim + 2) * 0x1p-53 * tot;
  if (tot + e < 0.5 * (fd + up) && tot - e > 0.5 * (fd + dn)) return f;
  return l2_f64_sequential(row, qrow, dim);
}
#ifndef DVSG_F64_GUARD
#define DVSG_F64_GUARD 1  // 0: round the tree sum unconditionally (A/B of the guard only)
#endif
// key distance of a finished accumulator (the one rounding point of every mode)
template <typename ACC, int METRIC, typename VT = float>
__device__ __forceinline__ float finish_dist(const ACC& tot, const VT* row, const float* qrow, int dim) {
  if constexpr (std::is_same<ACC, double>::value && METRIC == 0 && DVSG_F64_GUARD) {
    return l2_f64_exact(tot, row, qrow, dim);
  } else {
    (void)row; (void)qrow; (void)dim;
    return METRIC == 0 ? acc_to_f32(tot) : -acc_to_f32(tot);
  }
}

// U partial sums per lane -> lane holds the full sum of vector
// (lane >> (5 - log2 U)) & (U - 1): log2(U) "transpose" stages that halve the
// live values, then a plain butterfly (U - 1 + 5 - log2 U shuffles instead of 5U).
template <int U, typename ACC>
__device__ __forceinline__ ACC transpose_reduce(ACC (&p)[U], int lane) {
  constexpr int LU = ilog2(U);
#pragma unroll
  for (int st = 0; st < LU; ++st) {
    const int half = U >> (st + 1);
    const int off = 16 >> st;
    const bool upper = (lane & off) != 0;
#pragma unroll
    for (int i = 0; i < half; ++i) {
      const ACC send = upper ? p[i] : p[i + half];
      const ACC keep = upper ? p[i + half] : p[i];
      p[i] = keep + shfl_xor(send, off);
    }
  }
  ACC v = p[0];
#pragma unroll
  for (int off = 16 >> LU; off > 0; off >>= 1) v += shfl_xor(v, off);
  return v;
}

template <typename ACC, int METRIC>
__device__ __forceinline__ ACC lane_partial(const float4& x, const float4& q);

template <>
__device__ __forceinline__ double lane_partial<double, 0>(const float4& x, const float4& q) {
  // sequential within the lane, no contraction: (x-q)^2 rounded then added
  const double d0 = (double)x.x - (double)q.x, d1 = (double)x.y - (double)q.y;
  const double d2 = (double)x.z - (double)q.z, d3 = (double)x.w - (double)q.w;
  double acc = __dmul_rn(d0, d0);
  acc = __dadd_rn(acc, __dmul_rn(d1, d1));
  acc = __dadd_rn(acc, __dmul_rn(d2, d2));
  acc = __dadd_rn(acc, __dmul_rn(d3, d3));
  return acc;
}
template <>
__device__ __forceinline__ double lane_partial<double, 1>(const float4& x, const float4& q) {
  double acc = __dmul_rn((double)x.x, (double)q.x);
  acc = __dadd_rn(acc, __dmul_rn((double)x.y, (double)q.y));
  acc = __dadd_rn(acc, __dmul_rn((double)x.z, (double)q.z));
  acc = __dadd_rn(acc, __dmul_rn((double)x.w, (double)q.w));
  return acc;
}
// exact x - q as d + de (TwoSum), d^2 as p + pe (FMA TwoProd), the 2*d*de
// cross term into lo (de^2 is below lo's own rounding)
__device__ __forceinline__ void f2_sq_diff(float x, float q, F2& acc) {
  const float d = __fsub_rn(x, q);
  const float bb = __fsub_rn(d, x);
  const float de = __fadd_rn(__fsub_rn(x, __fsub_rn(d, bb)), __fsub_rn(-q, bb));
  const float p = __fmul_rn(d, d);
  float lo = __fmaf_rn(d, d, -p);
  lo = __fmaf_rn(__fmul_rn(2.0f, d), de, lo);
  // both addends >= 0: FastTwoSum on (max, min) is error-free
  const float a = fmaxf(acc.hi, p), b = fminf(acc.hi, p);
  const float s = __fadd_rn(a, b);
  const float e = __fsub_rn(b, __fsub_rn(s, a));
  acc = F2{s, __fadd_rn(acc.lo, __fadd_rn(e, lo))};
}
__device__ __forceinline__ void f2_prod(float x, float q, F2& acc) {
  const float p = __fmul_rn(x, q);
  acc = f2_add(acc, F2{p, __fmaf_rn(x, q, -p)});
}
template <>
__device__ __forceinline__ F2 lane_partial<F2, 0>(const float4& x, const float4& q) {
  F2 acc{0.f, 0.f};
  f2_sq_diff(x.x, q.x, acc);
  f2_sq_diff(x.y, q.y, acc);
  f2_sq_diff(x.z, q.z, acc);
  f2_sq_diff(x.w, q.w, acc);
  return acc;
}
template <>
__device__ __forceinline__ F2 lane_partial<F2, 1>(const float4& x, const float4& q) {
  F2 acc{0.f, 0.f};
  f2_prod(x.x, q.x, acc);
  f2_prod(x.y, q.y, acc);
  f2_prod(x.z, q.z, acc);
  f2_prod(x.w, q.w, acc);
  return acc;
}
template <>
__device__ __forceinline__ float lane_partial<float, 0>(const float4& x, const float4& q) {
  const float d0 = x.x - q.x, d1 = x.y - q.y, d2 = x.z - q.z, d3 = x.w - q.w;
  float acc = d0 * d0;
  acc = fmaf(d1, d1, acc);
  acc = fmaf(d2, d2, acc);
  acc = fmaf(d3, d3, acc);
  return acc;
}
template <>
__device__ __forceinline__ float lane_partial<float, 1>(const float4& x, const float4& q) {
  float acc = x.x * q.x;
  acc = fmaf(x.y, q.y, acc);
  acc = fmaf(x.z, q.z, acc);
  acc = fmaf(x.w, q.w, acc);
  return acc;
}

#ifndef DVSG_GATHER_NO_L1
#define DVSG_GATHER_NO_L1 2  // 1: vector rows bypass L1 (+5%), 2: adjacency rows too (+1%)
#endif
// Vector rows are streamed (little L1 reuse): optionally keep them out of L1
// so the CTA's visited-table lines stay cached there.
__device__ __forceinline__ float4 ldg_f4(const float* p) {
#if DVSG_GATHER_NO_L1
  float4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w) : "l"(p));
  return r;
#else
  return __ldg(reinterpret_cast<const float4*>(p));
#endif
}

// 4 byte-stored coordinates (U8 vector storage): raw word, then -> float4 (exact)
__device__ __forceinline__ uint32_t ldg_u8x4_raw(const uint8_t* p) {
  uint32_t w;
  asm volatile("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(w) : "l"(p));
  return w;
}
__device__ __forceinline__ float4 cvt_u8x4(uint32_t w) {
  return make_float4((float)(w & 0xFFu), (float)((w >> 8) & 0xFFu), (float)((w >> 16) & 0xFFu), (float)(w >> 24));
}

__device__ __forceinline__ uint32_t ldg_u32_stream(const uint32_t* p) {
#if DVSG_GATHER_NO_L1 >= 2
  uint32_t r;
  asm volatile("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(r) : "l"(p));
  return r;
#else
  return __ldg(p);
#endif
}

struct BlockState {
  uint64_t unit;
  int ncand;
  int nsurv;
  int nf;
  int warp_cnt[kWarps];
};

}  // namespace
}  // namespace dvsg
