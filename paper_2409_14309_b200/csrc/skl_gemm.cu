// Gaussian sketch apply SA = G * A on the fp64 tensor cores.
//
// Reference: /root/reference/pkg/src/sketchls/sketch.py:204-208 (`g @ A`,
// OpenBLAS dgemm).  Shapes: G is d x m, row-major (numpy's C order, ld ldg),
// A is m x n column-major (lda): both operands are K-contiguous (K = m), the
// "row.col" layout of the fp64 MMA.  On sm_100a fp64 MMA exists only as
// warp-level `mma.sync ... .f64` (SASS DMMA); tcgen05 has no f64 kind.
//
// Design: CTA tile 128 x 128 (d x n), 8 warps each owning 64 x 32 as
// 4 x 4 m16n8k4 fragments (64 fp64 accumulators per thread), K staged in
// 16-deep slices through a 5-stage cp.async (LDGSTS) ring with padded rows
// (conflict-free fragment loads).  Stages are handed over by per-stage
// full/empty mbarriers (cp.async.mbarrier.arrive as copies land, one arrive
// per warp when its fragments are consumed) instead of a CTA barrier per
// slice, so warps drift by up to a slice and the DMMA pipe is not drained at
// every K step (config 3: 17.63 ms with a __syncthreads ring of 32-deep
// slices -> 16.09 ms; cuBLAS DGEMM 15.70 ms on the same operands).  The reduction dimension m is long
// (262144 at config 3) and the output small, so K is split S ways with
// S chosen to make tiles x S a multiple of the SM count; partial tiles go
// to a workspace and are summed in fixed split order (deterministic).
// Blocks that share a G row panel are launched adjacently so G streams
// from HBM about once.
#include <cuda_runtime.h>

#include <algorithm>
#include <numeric>

#include "skl_common.h"
#include "skl_ptx.cuh"

namespace skl {

#ifndef SKL_GM_BK
#define SKL_GM_BK 16
#endif
#ifndef SKL_GM_STAGES
#define SKL_GM_STAGES 5
#endif
#ifndef SKL_GM_MINB
#define SKL_GM_MINB 1
#endif
constexpr int GM_BM = 128, GM_BN = 128, GM_BK = SKL_GM_BK, GM_PAD = 2, GM_STAGES = SKL_GM_STAGES;
constexpr int GM_LD = GM_BK + GM_PAD;  // smem row stride (doubles)
constexpr int GM_THREADS = 256;

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, int src_bytes) {
  const uint32_t s = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(s), "l"(gmem),
               "r"(src_bytes)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

__device__ __forceinline__ void dmma_16x8x4(double (&c)[4], double a0, double a1, double b0) {
  asm volatile(
      "mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, "
      "{%0,%1,%2,%3};"
      : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
      : "d"(a0), "d"(a1), "d"(b0));
}

// Signal `bar` once all of this thread's prior cp.async copies have landed
// (the arrival was pre-counted in the barrier's init count).
__device__ __forceinline__ void cp_async_mbar_arrive(uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

struct GemmParams {
  const double* G;
  int64_t ldg;
  const double* A;
  int64_t lda;
  double* C;       // final (S == 1) or workspace [S][n][d] column-major slices
  int64_t ldc;
  int64_t d, n, K;
  int S;
  int64_t nkb;     // K blocks of GM_BK
  int accumulate;  // S == 1 only
};

// Load one K slice of the G tile (rows i0..i0+127) and A tile (cols j0..).
__device__ __forceinline__ void gm_load(const GemmParams& p, double* Gs, double* As, int64_t i0,
                                        int64_t j0, int64_t k0) {
  const int tid = threadIdx.x;
#pragma unroll
  for (int q = 0; q < (GM_BM * GM_BK / 2) / GM_THREADS; ++q) {
    const int idx = tid + q * GM_THREADS;  // 16-byte chunk id
    const int r = idx / (GM_BK / 2), kc = (idx % (GM_BK / 2)) * 2;
    const int64_t gi = i0 + r, gk = k0 + kc;
    const bool ok = gi < p.d && gk < p.K;
    const int bytes = ok ? (int)min((int64_t)16, (p.K - gk) * 8) : 0;
    const double* src = ok ? p.G + gi * p.ldg + gk : p.G;
    cp_async16(Gs + r * GM_LD + kc, src, bytes);
  }
#pragma unroll
  for (int q = 0; q < (GM_BN * GM_BK / 2) / GM_THREADS; ++q) {
    const int idx = tid + q * GM_THREADS;
    const int c = idx / (GM_BK / 2), kc = (idx % (GM_BK / 2)) * 2;
    const int64_t gj = j0 + c, gk = k0 + kc;
    const bool ok = gj < p.n && gk < p.K;
    const int bytes = ok ? (int)min((int64_t)16, (p.K - gk) * 8) : 0;
    const double* src = ok ? p.A + gj * p.lda + gk : p.A;
    cp_async16(As + c * GM_LD + kc, src, bytes);
  }
}

__global__ void __launch_bounds__(GM_THREADS, SKL_GM_MINB) gemm_f64_dmma_kernel(const GemmParams p) {
  extern __shared__ __align__(128) double gsm[];
  double* Gs = gsm;                                   // [STAGES][BM][LD]
  double* As = gsm + GM_STAGES * GM_BM * GM_LD;       // [STAGES][BN][LD]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp >> 2, wn = warp & 3;            // 2 x 4 warps: 64 x 32 each
  const int64_t j0 = (int64_t)blockIdx.x * GM_BN;
  const int64_t i0 = (int64_t)blockIdx.y * GM_BM;
  const int s = blockIdx.z;
  const int64_t kb0 = p.nkb * s / p.S, kb1 = p.nkb * (s + 1) / p.S;
  const int64_t nk = kb1 - kb0;

  double acc[4][4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b)
#pragma unroll
      for (int c = 0; c < 4; ++c) acc[a][b][c] = 0.0;

  // Per-stage full/empty mbarriers instead of a CTA barrier per slice: every
  // thread's copies arrive on full[s] as they land; each warp releases a
  // stage on empty[s] once its fragments are consumed, so warps drift by up
  // to a slice and the DMMA pipe is not drained at every K step.
  __shared__ __align__(8) uint64_t full[GM_STAGES], empty[GM_STAGES];
  if (tid == 0) {
#pragma unroll
    for (int st = 0; st < GM_STAGES; ++st) {
      mbar_init(&full[st], GM_THREADS);
      mbar_init(&empty[st], GM_THREADS / 32);
    }
    fence_mbar_init();
  }
  __syncthreads();
#pragma unroll
  for (int st = 0; st < GM_STAGES - 1; ++st) {
    if (st < nk) {
      gm_load(p, Gs + st * GM_BM * GM_LD, As + st * GM_BN * GM_LD, i0, j0, (kb0 + st) * GM_BK);
      cp_async_mbar_arrive(&full[st]);
    }
  }
  const int g = lane >> 2, tq = lane & 3;
  for (int64_t kb = 0; kb < nk; ++kb) {
    {
      const int64_t nxt = kb + GM_STAGES - 1;
      const int sl = (int)(nxt % GM_STAGES);
      if (nxt < nk) {
        if (nxt >= GM_STAGES) mbar_wait(&empty[sl], (uint32_t)((nxt / GM_STAGES - 1) & 1));
        gm_load(p, Gs + sl * GM_BM * GM_LD, As + sl * GM_BN * GM_LD, i0, j0, (kb0 + nxt) * GM_BK);
        cp_async_mbar_arrive(&full[sl]);
      }
    }
    const int cur = (int)(kb % GM_STAGES);
    mbar_wait(&full[cur], (uint32_t)((kb / GM_STAGES) & 1));
    const double* gs = Gs + cur * GM_BM * GM_LD + (wm * 64) * GM_LD;
    const double* as = As + cur * GM_BN * GM_LD + (wn * 32) * GM_LD;
#pragma unroll
    for (int kk = 0; kk < GM_BK; kk += 4) {
      double af[4][2], bf[4];
#pragma unroll
      for (int mt = 0; mt < 4; ++mt) {
        af[mt][0] = gs[(mt * 16 + g) * GM_LD + kk + tq];
        af[mt][1] = gs[(mt * 16 + 8 + g) * GM_LD + kk + tq];
      }
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) bf[nt] = as[(nt * 8 + g) * GM_LD + kk + tq];
#pragma unroll
      for (int mt = 0; mt < 4; ++mt)
#pragma unroll
        for (int nt = 0; nt < 4; ++nt) dmma_16x8x4(acc[mt][nt], af[mt][0], af[mt][1], bf[nt]);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[cur]);
  }
  cp_async_wait<0>();

  // epilogue: c0,c1 at (g, 2tq..2tq+1), c2,c3 at (g+8, ...)
  double* out = p.S == 1 ? p.C : p.C + (int64_t)s * p.n * p.d;
  const int64_t ldo = p.S == 1 ? p.ldc : p.d;
#pragma unroll
  for (int mt = 0; mt < 4; ++mt)
#pragma unroll
    for (int nt = 0; nt < 4; ++nt)
#pragma unroll
      for (int h = 0; h < 4; ++h) {
        const int64_t i = i0 + wm * 64 + mt * 16 + g + (h >= 2 ? 8 : 0);
        const int64_t j = j0 + wn * 32 + nt * 8 + 2 * tq + (h & 1);
        if (i < p.d && j < p.n) {
          double v = acc[mt][nt][h];
          if (p.S == 1 && p.accumulate) v += out[j * ldo + i];
          out[j * ldo + i] = v;
        }
      }
}

__global__ void gemm_split_reduce_kernel(const double* part, int S, int64_t d, int64_t n,
                                         double* C, int64_t ldc, int accumulate) {
  const int64_t total = d * n;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = idx / d, i = idx % d;
    double v = 0.0;
    for (int q = 0; q < S; ++q) v += part[(int64_t)q * total + idx];
    if (accumulate) v = C[j * ldc + i] + v;
    C[j * ldc + i] = v;
  }
}

// y = G x for one column (n == 1): the tile GEMM would spend 127 of every
// 128 tile columns on padding; this is one HBM pass over G instead.  A warp
// owns a row of G (K-contiguous: coalesced 16-byte loads, eight in flight
// per lane), x (m doubles) is re-read from L2, and the row sum folds in a
// fixed order (per-lane accumulators, then a shuffle tree): deterministic.
constexpr int GV_WARPS = 8;
__global__ void __launch_bounds__(GV_WARPS * 32) gemv_f64_rows_kernel(
    const double* __restrict__ G, int64_t ldg, const double* __restrict__ x, int64_t m,
    int64_t d, double* __restrict__ y, int accumulate) {
  const int lane = threadIdx.x & 31;
  const int64_t row = (int64_t)blockIdx.x * GV_WARPS + (threadIdx.x >> 5);
  if (row >= d) return;
  const double2* g2 = reinterpret_cast<const double2*>(G + row * ldg);
  const double2* x2 = reinterpret_cast<const double2*>(x);
  const int64_t m2 = m / 2;
  double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
  int64_t i = lane;
  for (; i + 7 * 32 < m2; i += 8 * 32) {
    double2 gv[8], xv[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      gv[u] = __ldcs(g2 + i + u * 32);
      xv[u] = __ldg(x2 + i + u * 32);
    }
#pragma unroll
    for (int u = 0; u < 8; u += 2) {
      a0 = fma(gv[u].x, xv[u].x, a0);
      a1 = fma(gv[u].y, xv[u].y, a1);
      a2 = fma(gv[u + 1].x, xv[u + 1].x, a2);
      a3 = fma(gv[u + 1].y, xv[u + 1].y, a3);
    }
  }
  for (; i < m2; i += 32) {
    const double2 gv = __ldcs(g2 + i), xv = __ldg(x2 + i);
    a0 = fma(gv.x, xv.x, a0);
    a1 = fma(gv.y, xv.y, a1);
  }
  if ((m & 1) && lane == 0) a2 = fma(G[row * ldg + m - 1], x[m - 1], a2);
  double t = (a0 + a1) + (a2 + a3);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
  if (lane == 0) y[row] = accumulate ? y[row] + t : t;
}

}  // namespace skl

using namespace skl;

extern "C" int skl_gemm_f64(const double* G, int64_t ldg, const double* A, int64_t lda, double* C,
                            int64_t ldc, int64_t d, int64_t n, int64_t m, int accumulate,
                            void* stream) {
  clear_error();
  cudaStream_t st = (cudaStream_t)stream;
  SKL_REQUIRE(G && A && C && d >= 1 && n >= 1 && m >= 1 && ldg >= m && lda >= m && ldc >= d,
              SKL_ERR_SHAPE, "gemm_f64: bad arguments");
  SKL_REQUIRE(((uintptr_t)G & 15) == 0 && ((uintptr_t)A & 15) == 0 && ldg % 2 == 0 &&
                  (lda % 2 == 0 || n == 1),
              SKL_ERR_INVALID, "gemm_f64: operands must be 16-byte aligned with even leading dims");
  if (n == 1) {  // one column: an HBM pass over G (gemv_f64_rows_kernel)
    gemv_f64_rows_kernel<<<(unsigned)((d + GV_WARPS - 1) / GV_WARPS), GV_WARPS * 32, 0, st>>>(
        G, ldg, A, m, d, C, accumulate);
    SKL_CUDA_LAUNCH();
    return SKL_OK;
  }
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t tiles = ((d + GM_BM - 1) / GM_BM) * ((n + GM_BN - 1) / GM_BN);
  const int64_t nkb = (m + GM_BK - 1) / GM_BK;
  // split K so tiles*S is a multiple of the SM count, >= 64 K blocks each
  int64_t S = sms / std::gcd((int64_t)sms, tiles);
  while (S > 1 && nkb / S < 64) S = std::max<int64_t>(1, S / 2);
  if (tiles >= sms) S = 1;
  GemmParams p;
  p.G = G; p.ldg = ldg; p.A = A; p.lda = lda; p.d = d; p.n = n; p.K = m; p.S = (int)S;
  p.nkb = nkb; p.accumulate = accumulate; p.ldc = ldc;
  double* part = nullptr;
  if (S > 1) {
    SKL_CUDA(malloc_async(&part, (size_t)S * d * n * sizeof(double), st));
    p.C = part;
  } else {
    p.C = C;
  }
  const size_t smem = (size_t)GM_STAGES * (GM_BM + GM_BN) * GM_LD * sizeof(double);
  SKL_CUDA(raise_smem_limit(gemm_f64_dmma_kernel, smem));
  dim3 grid((unsigned)((n + GM_BN - 1) / GM_BN), (unsigned)((d + GM_BM - 1) / GM_BM), (unsigned)S);
  gemm_f64_dmma_kernel<<<grid, GM_THREADS, smem, st>>>(p);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    if (part) cudaFreeAsync(part, st);
    SKL_FAIL(SKL_ERR_CUDA, "gemm_f64 launch failed: %s", cudaGetErrorString(e));
  }
  if (S > 1) {
    const int64_t total = d * n;
    const int blocks = (int)std::min<int64_t>((total + 255) / 256, 8LL * sms);
    gemm_split_reduce_kernel<<<blocks, 256, 0, st>>>(part, (int)S, d, n, C, ldc, accumulate);
    SKL_CUDA_LAUNCH();
    SKL_CUDA(cudaFreeAsync(part, st));
  }
  return SKL_OK;
}
