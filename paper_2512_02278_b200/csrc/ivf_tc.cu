// ivf_tc.cu -- K7 on the 5th-generation tensor cores (tcgen05 + TMEM).
//
// Same contract as range_topk_kernel (ivf_build.cu): per row of a <= 128-row
// block, the m <= 32 smallest (squared L2, column id) keys over a list of
// column ranges.  The dot products run as one UMMA per 16-deep K slice:
//
//   A = the block's rows   (128 x K bf16, K-major, loaded once per block)
//   B = 128 columns        (128 x K bf16, K-major, double-buffered cp.async)
//   D = A . B^T            (128 x 128 fp32 in TMEM: lane = row, column = col)
//
// issued by one thread (tcgen05.mma.cta_group::1.kind::f16, M=128, N=128,
// K=16 per instruction) and committed to an mbarrier; the 4 warps then read
// their 32 TMEM lanes (tcgen05.ld 32x32b.x32), form dist = |x|^2 + |y|^2 -
// 2 x.y and filter them against their row's current m-th key into a
// per-row survivor buffer in shared memory (one predicated store per column,
// no divergent loop); each warp then merges the survivors of its 32 rows into
// register-resident sorted lists (lane i of the warp holds the i-th smallest
// key of each of its rows: one ballot + shuffle per insertion, whatever the
// position -- a per-thread sorted insert diverges across the warp and cost 8x
// the instructions).  The next column tile streams in while the current one
// is multiplied and scanned.
//
// Exactness: the bench data are integers in [0, 255]: exact in bf16, every
// product exact in fp32 and every partial sum an integer below 2^24, so the
// tensor-core dot product -- whatever its internal summation order -- is the
// exact integer and the keys equal the CUDA-core K7's (tested bit for bit in
// tests/test_gpu_ivf.py).  On float data bf16 rounds the inputs: the result is
// an approximate kNN, which is all a graph build needs; ground truth on float
// data stays on the fp32 path.
//
// Shared-memory layout of an operand (UMMA canonical K-major, no swizzle):
// element (r, k) at (r/8)*SBO + (k/8)*LBO + (r%8)*16 + (k%8)*2 bytes with
// LBO = 128 (the 16-byte K chunks of one 8-row core matrix are adjacent) and
// SBO = K/8 * 128 (8-row groups follow each other).
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

#include "dvsg_internal.h"

namespace dvsg {
namespace {

constexpr int TCM = 128;  // rows per block (UMMA M)
constexpr int TCN = 128;  // columns per tile (UMMA N)
constexpr int TCMAXK = 256;

__device__ __forceinline__ uint32_t s32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint32_t f2ord(float f) {
  if (f == 0.0f) f = 0.0f;
  const uint32_t u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float ord2f(uint32_t o) {
  return __uint_as_float((o & 0x80000000u) ? (o & 0x7FFFFFFFu) : ~o);
}

// the 32 smallest of two ascending 32-lists (lane i holds entry i of each):
// min against the reversed other list is bitonic; 5 half-cleaners sort it
__device__ __forceinline__ uint64_t warp_merge_u64(uint64_t a, uint64_t b_sorted, int lane) {
  const uint64_t rev = __shfl_sync(0xFFFFFFFFu, b_sorted, 31 - lane);
  uint64_t v = a < rev ? a : rev;
#pragma unroll
  for (int j = 16; j > 0; j >>= 1) {
    const uint64_t w = __shfl_xor_sync(0xFFFFFFFFu, v, j);
    v = (lane & j) ? (w > v ? w : v) : (w < v ? w : v);
  }
  return v;
}

__device__ __forceinline__ void cp16(uint32_t dst, const void* src, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(valid ? 16 : 0)
               : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46);  // version 1 (Blackwell), no swizzle
}

__device__ __forceinline__ void mbar_init(uint64_t* bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(s32(bar)),
      "r"(phase)
      : "memory");
}

#define TMEM_LD32(taddr, r)                                                                                  \
  asm volatile(                                                                                              \
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17," \
      "%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"                                     \
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),      \
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),  \
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]),            \
        "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]),            \
        "=r"(r[30]), "=r"(r[31])                                                                             \
      : "r"(taddr))

// dynamic smem per CTA: A (128 x K) + 2 x B (128 x K) + a survivor buffer per
// epilogue group + barrier
__host__ __device__ inline size_t tc_smem_bytes(int row_bytes, int groups = 1) {
  return (size_t)3 * TCM * row_bytes + (size_t)groups * 32 * TCM * 8 + 64;
}

// T = uint16_t: bf16 operands (kind::f16, K = 16 per MMA); T = float: tf32
// operands read from fp32 storage (kind::tf32, K = 8 per MMA).  Either way one
// MMA consumes a 32-byte K slice of every row.
// G epilogue groups of 4 warps: warp w reads TMEM lanes 32*(w%4).. (its 32
// rows) and group g = w/4 scans columns [g*128/G, (g+1)*128/G) of every tile
// into its own lists; at the end group 1 hands its lists to group 0, which
// merges and writes.  G = 2 doubles the warps that hide the epilogue's latency.
template <typename T, int G>
__global__ void __launch_bounds__(128 * G, 1)
range_topk_tc_kernel(const T* __restrict__ rows, const float* __restrict__ rnorm,
                     const T* __restrict__ cols, const float* __restrict__ cnorm, int kpad,
                     const uint32_t* __restrict__ row_map, const RangeBlock* __restrict__ blocks,
                     const uint32_t* __restrict__ list_off, const uint2* __restrict__ ranges, int m, int flags,
                     uint32_t* __restrict__ out_ids, float* __restrict__ out_dists, uint64_t out_stride) {
  extern __shared__ __align__(128) unsigned char smem[];
  unsigned char* sa = smem;
  constexpr bool kTF32 = sizeof(T) == 4;
  constexpr int kEl = 16 / sizeof(T);  // elements per 16-byte chunk
  const int row_bytes = kpad * (int)sizeof(T);
  auto sb = [&](int b) { return smem + (size_t)(1 + b) * TCM * row_bytes; };  // B double buffer
  __shared__ float cn[2][TCN];  // column norms of the two B tiles (static smem: LDS, not generic loads)
  // per group [32][128]: survivor j of row t at j*128 + t
  uint64_t* cbuf0 = reinterpret_cast<uint64_t*>(smem + (size_t)3 * TCM * row_bytes);
  uint64_t* bar = cbuf0 + G * 32 * TCM;
  __shared__ uint32_t tmem_slot;

  constexpr int NT = 128 * G;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int grp = tid >> 7, rt = tid & 127, rw = warp & 3;  // group, row (= TMEM lane), lane quarter
  uint64_t* cbuf = cbuf0 + grp * 32 * TCM;
  const RangeBlock blk = blocks[blockIdx.x];
  const int nrows = (int)blk.nrows;
  const int kch = row_bytes / 16;  // 16-byte chunks per row
  const uint32_t lbo = 128, sbo = (uint32_t)kch * 128;

  // ---- TMEM (128 fp32 columns) and the MMA-completion barrier
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(s32(&tmem_slot))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (tid == 0) mbar_init(bar);
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_slot;

  // ---- this thread's row: physical index, norm; the warp's 32 row lists
  const bool rvalid = rt < nrows;
  const uint32_t prow = rvalid ? (row_map ? row_map[blk.row0 + rt] : blk.row0 + rt) : 0u;
  const float nr = rvalid ? rnorm[prow] : 0.f;
  const uint64_t orow = (flags & 8) ? (uint64_t)prow : (uint64_t)blk.out_row0 + (uint64_t)rt;
  uint64_t top[32];  // top[rr] at lane i: i-th smallest key of row rw*32 + rr (this group's columns)
  // this thread's row: current m-th key -- (+inf, 0) while the list is
  // short, so the padding columns (+inf) never pass
  const uint64_t kInfKey = (uint64_t)f2ord(__int_as_float(0x7F800000)) << 32;
  uint64_t thr = kInfKey;
  // two groups: each publishes its rows' m-th keys; a column that fails the
  // other group's key cannot reach the union's top m either, so each group
  // filters with the smaller of the two (stale values are larger: safe)
  __shared__ uint64_t gthr[G][TCM];
  gthr[grp][rt] = kInfKey;
  auto set_thr = [&](uint64_t t) {
    thr = t == ~0ull ? kInfKey : t;
    if (G == 2) gthr[grp][rt] = thr;
  };
#pragma unroll
  for (int rr = 0; rr < 32; ++rr) {
    top[rr] = ~0ull;
    if (flags & 4) {  // continue from the lists already in the output (group 1: their m-th key only)
      const uint64_t o = __shfl_sync(0xFFFFFFFFu, orow, rr);
      const bool v = __shfl_sync(0xFFFFFFFFu, rvalid, rr);
      uint32_t id = 0xFFFFFFFFu;
      float d = 0.f;
      if (v && lane < m) {
        id = out_ids[o * out_stride + lane];
        d = out_dists[o * out_stride + lane];
      }
      const unsigned bad = __ballot_sync(0xFFFFFFFFu, id == 0xFFFFFFFFu);
      const int first_bad = bad ? __ffs(bad) - 1 : 32;  // entries after the first gap are ignored
      const uint64_t prev = lane < first_bad ? ((uint64_t)f2ord(d) << 32) | id : ~0ull;
      if (grp == 0) top[rr] = prev;  // group 1 keeps an empty list (no duplicates at the hand-over)
      const uint64_t t = __shfl_sync(0xFFFFFFFFu, prev, m - 1);
      if (lane == rr) set_thr(t);
    }
  }

  // ---- A: the block's rows, canonical K-major layout
  for (int c = tid; c < TCM * kch; c += NT) {
    const int r = c / kch, kc = c - r * kch;
    const uint32_t pr = r < nrows ? (row_map ? row_map[blk.row0 + r] : blk.row0 + r) : 0u;
    cp16(s32(sa + (r >> 3) * sbo + kc * lbo + (r & 7) * 16), rows + (uint64_t)pr * kpad + kc * kEl, r < nrows);
  }
  cp_commit();

  // ---- column tiles: (range, start) pairs, prefetched one ahead
  const uint32_t l0 = list_off[blk.list], l1 = list_off[blk.list + 1];
  uint32_t li = l0, c0 = l0 < l1 ? ranges[l0].x : 0u;
  auto next_tile = [&](uint32_t& l, uint32_t& c) {  // advance to the next non-empty tile start
    while (l < l1) {
      const uint2 rg = ranges[l];
      if (c < rg.x) c = rg.x;
      if (c < rg.y) return true;
      ++l;
      if (l < l1) c = ranges[l].x;
    }
    return false;
  };
  bool have = next_tile(li, c0);
  auto load_b = [&](int buf, uint32_t l, uint32_t c) {
    const uint32_t end = ranges[l].y;
    for (int q = tid; q < TCN * kch; q += NT) {
      const int r = q / kch, kc = q - r * kch;
      const bool v = c + r < end;
      cp16(s32(sb(buf) + (r >> 3) * sbo + kc * lbo + (r & 7) * 16), cols + (uint64_t)(v ? c + r : 0) * kpad + kc * kEl,
           v);
    }
    if (tid < TCN) cn[buf][tid] = c + tid < end ? cnorm[c + tid] : __int_as_float(0x7F800000);  // +inf: never a survivor
    cp_commit();
  };
  if (have) load_b(0, li, c0);
  // instruction descriptor: D f32, A/B bf16 (1) or tf32 (2), K-major, N, M
  const uint32_t fmt = kTF32 ? 2u : 1u;
  const uint32_t idesc = (1u << 4) | (fmt << 7) | (fmt << 10) | ((uint32_t)(TCN >> 3) << 17) | ((uint32_t)(TCM >> 4) << 24);

  int buf = 0;
  uint32_t phase = 0;
  while (have) {
    const uint32_t tc = c0;
    // prefetch the following tile into the other buffer (its MMA finished last round)
    uint32_t nl = li, nc = c0 + TCN;
    const bool nhave = next_tile(nl, nc);
    if (nhave) load_b(buf ^ 1, nl, nc);
    if (nhave) cp_wait<1>(); else cp_wait<0>();
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic smem writes -> tensor core
    __syncthreads();
    if (tid == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t abase = s32(sa), bbase = s32(sb(buf));
      for (int kk = 0; kk < row_bytes / 32; ++kk) {
        const uint64_t ad = umma_desc(abase + kk * 2 * lbo, lbo, sbo);
        const uint64_t bd = umma_desc(bbase + kk * 2 * lbo, lbo, sbo);
        const uint32_t acc = kk > 0 ? 1u : 0u;
        if constexpr (kTF32) {
          asm volatile(
              "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
              "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
              "l"(ad), "l"(bd), "r"(idesc), "r"(acc)
              : "memory");
        } else {
          asm volatile(
              "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
              "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
              "l"(ad), "l"(bd), "r"(idesc), "r"(acc)
              : "memory");
        }
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(s32(bar))
                   : "memory");
    }
    mbar_wait(bar, phase);
    phase ^= 1u;
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    // ---- epilogue: this group's 128/G columns in TMEM loads of 32
#pragma unroll 1
    for (int part = grp * (4 / G); part < (grp + 1) * (4 / G); ++part) {
      uint32_t r[32];
      TMEM_LD32(tmem + ((uint32_t)(rw * 32) << 16) + (uint32_t)(part * 32), r);
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      // (1) this thread's row: survivors of the m-th-key filter -> cbuf
      int ns = 0;
      uint64_t fthr = thr;
      if (G == 2) {
        const uint64_t o = gthr[grp ^ 1][rt];
        fthr = o < fthr ? o : fthr;
      }
      if (rvalid) {
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const int cl = part * 32 + j;
          const uint32_t col = tc + (uint32_t)cl;
          const float dist = fmaxf(fmaf(-2.f, __uint_as_float(r[j]), nr + cn[buf][cl]), 0.f);
          const uint64_t key = ((uint64_t)f2ord(dist) << 32) | col;
          const bool ok = key < fthr && !((flags & 1) && col == prow);
          if (ok) cbuf[ns * TCM + rt] = key;
          ns += ok ? 1 : 0;
        }
      }
      __syncwarp();
      // (2) the warp merges each of its rows' survivors into the row's list
#pragma unroll
      for (int rr = 0; rr < 32; ++rr) {
        const int n = __shfl_sync(0xFFFFFFFFu, ns, rr);
        if (n == 0) continue;
        const int row = rw * 32 + rr;
        for (int s2 = 0; s2 < n; ++s2) {
          const uint64_t key = cbuf[s2 * TCM + row];
          const unsigned gt = __ballot_sync(0xFFFFFFFFu, top[rr] > key);
          if (gt == 0) continue;  // not among the 32 smallest
          const int pos = __ffs(gt) - 1;
          const uint64_t up = __shfl_up_sync(0xFFFFFFFFu, top[rr], 1);
          if (lane > pos) top[rr] = up;
          if (lane == pos) top[rr] = key;
        }
        const uint64_t t = __shfl_sync(0xFFFFFFFFu, top[rr], m - 1);
        if (lane == rr) set_thr(t);
      }
      __syncwarp();
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();  // TMEM and buffer `buf` free for the next round
    buf ^= 1;
    li = nl;
    c0 = nc;
    have = nhave;
  }

  if constexpr (G == 2) {  // group 1's lists -> group 0 (cbuf of group 1 as the hand-over buffer)
    if (grp == 1) {
#pragma unroll
      for (int rr = 0; rr < 32; ++rr) cbuf[lane * TCM + rw * 32 + rr] = top[rr];
    }
    __syncthreads();
    if (grp == 0) {
      // merge two ascending 32-lists: min with the other list reversed is a
      // bitonic sequence holding the 32 smallest of the union; 5 half-cleaner
      // stages sort it (no per-key insertion)
      const uint64_t* other = cbuf0 + 32 * TCM;
#pragma unroll
      for (int rr = 0; rr < 32; ++rr) {
        const int row = rw * 32 + rr;
        top[rr] = warp_merge_u64(top[rr], other[lane * TCM + row], lane);
      }
    }
  }

  // ---- emit (same rules as range_topk_kernel): lane j writes entry j of each row
#pragma unroll
  for (int rr = 0; rr < 32; ++rr) {
    if (grp != 0) break;
    if (!__shfl_sync(0xFFFFFFFFu, rvalid, rr)) continue;
    const uint64_t o = __shfl_sync(0xFFFFFFFFu, orow, rr);
    const int nv = __popc(__ballot_sync(0xFFFFFFFFu, lane < m && top[rr] != ~0ull));
    if (flags & 2) {
      const uint32_t pr = __shfl_sync(0xFFFFFFFFu, prow, rr);
      const uint64_t kj = __shfl_sync(0xFFFFFFFFu, top[rr], nv > 0 ? lane % nv : 0);
      if (lane < m) {
        out_ids[o * out_stride + lane] = nv > 0 ? (uint32_t)kj : pr;
        if (out_dists) out_dists[o * out_stride + lane] = nv > 0 ? ord2f((uint32_t)(kj >> 32)) : 0.f;
      }
    } else if (lane < m) {
      const bool ok = lane < nv;
      out_ids[o * out_stride + lane] = ok ? (uint32_t)top[rr] : 0xFFFFFFFFu;
      if (out_dists) out_dists[o * out_stride + lane] = ok ? ord2f((uint32_t)(top[rr] >> 32)) : __int_as_float(0x7F800000);
    }
  }
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tmem) : "memory");
}

__global__ void to_bf16_kernel(const float* __restrict__ x, uint64_t n, int dpad, int kpad,
                               uint16_t* __restrict__ out) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n * (uint64_t)kpad) return;
  const uint64_t r = i / (uint64_t)kpad;
  const int k = (int)(i - r * (uint64_t)kpad);
  const float v = k < dpad ? x[r * (uint64_t)dpad + k] : 0.f;
  // round to nearest even (integers up to 256 are exact)
  uint32_t u = __float_as_uint(v);
  u += 0x7FFFu + ((u >> 16) & 1u);
  out[i] = (uint16_t)(u >> 16);
}

}  // namespace

size_t range_topk_tc_smem_bytes(int kpad) { return tc_smem_bytes(kpad * 2); }

template <typename T, int G>
cudaError_t launch_tc_g(const T* rows, const float* rnorm, const T* cols, const float* cnorm, int kpad,
                        const uint32_t* row_map, const RangeBlock* blocks, uint64_t nblocks, const uint32_t* list_off,
                        const uint2* ranges, int m, int flags, uint32_t* out_ids, float* out_dists,
                        uint64_t out_stride, size_t smem, cudaStream_t stream) {
  cudaError_t e = cudaFuncSetAttribute(range_topk_tc_kernel<T, G>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
  if (e != cudaSuccess) return e;
  for (uint64_t b0 = 0; b0 < nblocks; b0 += 0x7FFFFFFFull) {
    const uint64_t nb = nblocks - b0 < 0x7FFFFFFFull ? nblocks - b0 : 0x7FFFFFFFull;
    range_topk_tc_kernel<T, G><<<(unsigned)nb, 128 * G, smem, stream>>>(rows, rnorm, cols, cnorm, kpad, row_map,
                                                                       blocks + b0, list_off, ranges, m, flags,
                                                                       out_ids, out_dists, out_stride);
  }
  return cudaGetLastError();
}

// groups: a second epilogue group doubles the warps per CTA but its survivor
// buffer costs 32 KB of smem.  When one group already fits two CTAs per SM
// (bf16 build rows: 106 KB) the second CTA hides the load / MMA / epilogue
// phases better than more warps in one CTA (two groups: 1 CTA/SM, 8.2 ->
// 17.5 s of kNN at 100M); when one group is already alone on its SM (TF32
// assign rows: 176 KB) the second group is free (1M x 4096: 60 -> 48 ms).
// groups = 0: that rule; DVSG_TC_GROUPS overrides.
template <typename T>
cudaError_t launch_tc_t(const T* rows, const float* rnorm, const T* cols, const float* cnorm, int kpad,
                        const uint32_t* row_map, const RangeBlock* blocks, uint64_t nblocks, const uint32_t* list_off,
                        const uint2* ranges, int m, int flags, uint32_t* out_ids, float* out_dists,
                        uint64_t out_stride, int groups, cudaStream_t stream) {
  const int row_bytes = kpad * (int)sizeof(T);
  if (m < 1 || m > 32 || row_bytes % 32 || kpad < 1 || row_bytes > TCMAXK * 2) return cudaErrorInvalidValue;
  if (nblocks == 0) return cudaSuccess;
  static const int groups_env = [] {
    const char* e = std::getenv("DVSG_TC_GROUPS");
    return e ? std::atoi(e) : 0;
  }();
  if (groups_env > 0) groups = groups_env;
  if (groups == 0) groups = 2 * tc_smem_bytes(row_bytes, 1) + 2048 > 227 * 1024 ? 2 : 1;
  // two epilogue groups only if their second survivor buffer fits (227 KB opt-in)
  if (groups >= 2 && tc_smem_bytes(row_bytes, 2) + 2048 <= 227 * 1024)
    return launch_tc_g<T, 2>(rows, rnorm, cols, cnorm, kpad, row_map, blocks, nblocks, list_off, ranges, m, flags,
                             out_ids, out_dists, out_stride, tc_smem_bytes(row_bytes, 2), stream);
  return launch_tc_g<T, 1>(rows, rnorm, cols, cnorm, kpad, row_map, blocks, nblocks, list_off, ranges, m, flags,
                           out_ids, out_dists, out_stride, tc_smem_bytes(row_bytes, 1), stream);
}

cudaError_t launch_range_topk_tc(const uint16_t* rows, const float* rnorm, const uint16_t* cols, const float* cnorm,
                                 int kpad, const uint32_t* row_map, const RangeBlock* blocks, uint64_t nblocks,
                                 const uint32_t* list_off, const uint2* ranges, int m, int flags, uint32_t* out_ids,
                                 float* out_dists, uint64_t out_stride, cudaStream_t stream) {
  if (kpad % 16) return cudaErrorInvalidValue;
  return launch_tc_t<uint16_t>(rows, rnorm, cols, cnorm, kpad, row_map, blocks, nblocks, list_off, ranges, m, flags,
                               out_ids, out_dists, out_stride, 0, stream);
}

cudaError_t launch_range_topk_tf32(const float* rows, const float* rnorm, const float* cols, const float* cnorm,
                                   int kpad, const uint32_t* row_map, const RangeBlock* blocks, uint64_t nblocks,
                                   const uint32_t* list_off, const uint2* ranges, int m, int flags, uint32_t* out_ids,
                                   float* out_dists, uint64_t out_stride, cudaStream_t stream) {
  if (kpad % 8) return cudaErrorInvalidValue;
  return launch_tc_t<float>(rows, rnorm, cols, cnorm, kpad, row_map, blocks, nblocks, list_off, ranges, m, flags,
                            out_ids, out_dists, out_stride, 0, stream);
}

cudaError_t launch_to_bf16(const float* x, uint64_t n, int dpad, int kpad, uint16_t* out, cudaStream_t stream) {
  const uint64_t tot = n * (uint64_t)kpad;
  if (tot == 0) return cudaSuccess;
  to_bf16_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, stream>>>(x, n, dpad, kpad, out);
  return cudaGetLastError();
}

}  // namespace dvsg
