// Reduced solve of the sketch-and-apply path: Cholesky-based, two paths
// picked on the device, each with one corrected semi-normal step.
//
// Reference: /root/reference/pkg/src/sketchls/solvers.py:296-320 and
// linalg.py:166-192, 214-218 -- x = R^{-1} Q^T Sb from the economy QR of SA
// (numpy/LAPACK Householder), diag(R) >= 0, rank check
// |R[c,c]| < 1e-14 ||SA||_F.  The R factor with a positive diagonal is
// unique, so any backward-stable QR gives the reference's R and x to
// rounding, and x is the least-squares minimiser either way; this file
// computes it with far fewer dependent steps than a column-by-column
// Householder sweep (skl_qr_blocked.cu: 257 dependent column steps across a
// thread-block cluster for config 2's 2048 x 257):
//
//   M  = [SA | Sb]                     (d x N, N = n + 1, never copied)
//   G1 = M^T M                          gram kernel, fp64 tensor cores (DMMA)
//   R1s = chol(G1 + s I)                cluster Cholesky, s = 11 (dN + N(N+1)) u ||M||_F^2,
//   R1u = chol(G1)                      and the unshifted variant in a second cluster
//   pick (cqr_pick_kernel): R1u held and its diagonal spans < 1e3 ->
//     semi-normal path: R1u^{-1} explicitly (dataflow TRSM on I),
//       x = R11^{-1} r12 (normal equations, ~kappa^2 u), one corrected
//       semi-normal step (~kappa u; Householder hand-over if it does not contract)
//   else shifted CholeskyQR2 (Fukaya, Kannan, Nakatsukasa, Yamamoto,
//   Yanagisawa 2020):
//     Q1 = M R1s^{-1}                   row-block dataflow TRSM (DMMA)
//     G2 = Q1^T Q1, R2 = chol(G2), R = R2 R1s
//     x  = R[:n,:n]^{-1} R[:n, n]       (the augmented column carries Q^T Sb)
//     x += R^{-1} R^{-T} SA^T (Sb - SA x) when R's diagonal spans > 1e3
//   The kernels of the path not taken return at once on the pick's flag.
//
// The refinement step brings the x error on config 2 (kappa = 1e8) to the
// spread of two Householder QRs of the same system (measured in numpy on the
// full-size sketched system: 4-6e-9 vs the Householder spread of 3-6e-9).
// A non-positive or non-finite Cholesky pivot of the chosen variant
// (numerically rank deficient or kappa beyond ~1e15) sets a flag; the caller
// then falls back to the Householder factorisation, which also produces the
// reference's error.
//
// Layouts: Gram, R and the diagonal-block inverses of R are kept as 32 x 32
// column-major tiles ("tile layout"), upper tiles (I <= J) packed column by
// column: tile (I, J) at index J (J + 1) / 2 + I.  Rows / columns past N are
// padded with the identity.
//
// Kernels (one stream, programmatic dependent launch between them):
//   cqr_gram_kernel   one CTA per (upper tile, row slice); 4 warps each own
//                     the whole 32 x 32 tile over a quarter of the slice's
//                     16-row chunks (DMMA m16n8k4, operands straight from
//                     HBM/L2 with 32-byte vector loads); the last CTA of a
//                     tile folds the slices in fixed order (deterministic).
//   cqr_chol_kernel   one cluster of nb CTAs, CTA J owns block column J in
//                     shared memory.  Step K: CTA K factors its diagonal
//                     tile (LDL^T in one warp: the dependent chain per pivot
//                     is a shuffle, a reciprocal and two FMAs); every CTA
//                     J > K solves its tile (K, J) against it (forward
//                     substitution, U_KK read over DSMEM); CTA K+1 updates
//                     and factors the next diagonal tile while the others
//                     apply the rank-32 update to the rest of their column
//                     (DMMA, R(K, I) read over DSMEM).  Two split cluster
//                     barriers per step.
//   cqr_trsm_df_kernel  Q = M R^{-1}, 16 rows per CTA, right-looking as a
//                     dataflow over the warps (see the kernel); the blocked
//                     Cholesky's block-row solves run through it too.
//   cqr_solve_*       rank check, y, the triangular solves (one CTA), the
//                     residual and SA^T r (multi-CTA GEMVs).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>

#include "skl_common.h"
#include "skl_ptx.cuh"

namespace skl {

constexpr int CQ_LD = 33;                 // shared-memory tile stride (doubles)
constexpr int CQ_TILE = 32 * CQ_LD;       // doubles per shared-memory tile
constexpr int CQ_MAXNB = 16;              // block columns (= cluster CTAs): N <= 512
constexpr int CQ_CHOL_NT = 256;
constexpr int CQ_TRSM_ROWS = 16;
constexpr int CQ_QLD = 20;                // row stride of the TRSM's Q block (conflict-free frags)
constexpr double CQ_RANK_TOL = 1e-14;     // linalg.py RANK_TOL
// Above this ratio of R's largest to smallest diagonal entry (a lower bound
// of kappa(SA), 25-40x below it on log-spaced spectra) the corrected
// semi-normal step is no longer reliable (it needs kappa^2 u well below 1):
// the solve hands over to Householder.  Config 2 (kappa = 1e8) sits at
// 4.3e6.
constexpr double CQ_DIAG_RATIO_MAX = 2e7;
// Below this diagonal ratio (kappa ~< 4e4) CholeskyQR2's own x is accurate
// to ~kappa u and the corrected semi-normal step is skipped (its kernels
// return at once).
constexpr double CQ_REFINE_RATIO = 1e3;

__host__ __device__ __forceinline__ int64_t cq_tile(int I, int J) {
  return (int64_t)J * (J + 1) / 2 + I;
}

// Columns of M: column c < n of A (ld lda), column n = b (when b != null).
struct CqCols {
  const double* A;
  int64_t lda;
  const double* b;
  int64_t n;  // columns taken from A
  int64_t d;  // rows
};
// The CholeskyQR2 kernels after the pick (TRSM, second Gram, second
// factorisation) return at once when *stop: the unshifted first factor was
// picked and the solve is the semi-normal one (cqr_pick_kernel).
__device__ __forceinline__ bool cq_stopped(const int* stop) { return stop != nullptr && *stop != 0; }

__device__ __forceinline__ const double* cq_col(const CqCols& X, int64_t c) {
  return c < X.n ? X.A + c * X.lda : X.b;
}

__device__ __forceinline__ void cq_dmma(double (&c)[4], double a0, double a1, double b0) {
  asm volatile(
      "mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, "
      "{%0,%1,%2,%3};"
      : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
      : "d"(a0), "d"(a1), "d"(b0));
}

__device__ __forceinline__ uint32_t cq_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cq_arrive() {
  asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
}
__device__ __forceinline__ void cq_wait() {
  asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// Remote shared-memory load (ordering from the cluster barrier before use).
__device__ __forceinline__ double cq_ld_remote(const double* local, uint32_t cta) {
  const uint32_t a = static_cast<uint32_t>(__cvta_generic_to_shared(local));
  uint32_t ra;
  asm("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(a), "r"(cta));
  double v;
  asm("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(ra));
  return v;
}

// Instrumented builds (SKL_NVCC_DEFINES=-DSKL_CQR_PROBE): thread 0 of every
// Cholesky CTA records %globaltimer at phase boundaries (skl_cqr_probe_dump).
#ifdef SKL_CQR_PROBE
__device__ long long g_cqr_probe[2][CQ_MAXNB][72];
__device__ int g_cqr_probe_call;
__device__ __forceinline__ long long cq_now() {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define CQ_PROBE(slot)                                                                   \
  do {                                                                                   \
    if (threadIdx.x == 0) g_cqr_probe[p.shift_coef > 0.0 ? 0 : 1][J][(slot)] = cq_now(); \
  } while (0)
#else
#define CQ_PROBE(slot) \
  do {                 \
  } while (0)
#endif

// ------------------------------------------------------------------ Gram
struct GramParams {
  CqCols X;
  int64_t N;
  uint32_t nchunk;    // 16-row chunks of d
  uint32_t U;         // work units: upper tiles x chunks, tile-major (U * P < 2^32)
  uint32_t P;         // CTAs (<= U): CTA c takes units [U c / P, U (c + 1) / P)
  int SEG;            // partial slots per CTA (>= tiles any CTA touches)
  double* part;       // [P][SEG][1024]
  double* Gt;         // [ntiles][1024]
  unsigned* cnt;      // [ntiles], zero on entry, left zero
  double* Gt2;        // optional second copy of the Gram (unshifted variant)
  const int* skip;    // cq_stopped: return at once
};

__device__ __forceinline__ uint32_t cq_unit_lo(const GramParams& p, uint32_t c) { return p.U * c / p.P; }

__device__ __forceinline__ void cq_tile_ij(int t, int& I, int& J) {
  J = (int)((sqrtf(8.0f * t + 1.0f) - 1.0f) * 0.5f);
  while ((J + 1) * (J + 2) / 2 <= t) ++J;
  while (J * (J + 1) / 2 > t) --J;
  I = t - J * (J + 1) / 2;
}

// Rows k .. k+3 of the lane's 8 columns (4 of block I, 4 of block J).
template <bool VEC>
__device__ __forceinline__ void cq_gram_load(const double* const (&pc)[8], int64_t k, int64_t d,
                                             bool ragged, double (&v)[8][4]) {
  if (VEC && !ragged) {
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const double2 x0 = __ldg(reinterpret_cast<const double2*>(pc[q] + k));
      const double2 x1 = __ldg(reinterpret_cast<const double2*>(pc[q] + k + 2));
      v[q][0] = x0.x; v[q][1] = x0.y; v[q][2] = x1.x; v[q][3] = x1.y;
    }
  } else {
#pragma unroll
    for (int q = 0; q < 8; ++q)
#pragma unroll
      for (int j = 0; j < 4; ++j) v[q][j] = (k + j < d) ? __ldg(pc[q] + k + j) : 0.0;
  }
}

__device__ __forceinline__ void cq_gram_mma(double (&acc)[2][4][4], const double (&v)[8][4]) {
#pragma unroll
  for (int j = 0; j < 4; ++j)
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) cq_dmma(acc[mt][nt], v[mt * 2][j], v[mt * 2 + 1][j], v[4 + nt][j]);
}

// G = X^T X on the fp64 tensor cores, stream-K: one wave of CTAs, each
// taking an equal contiguous range of (upper tile, 16-row chunk) units, so
// the load is balanced to a chunk whatever the tile count.  Within a tile
// segment the 4 warps split the chunks round-robin (each owns the whole
// 32 x 32 tile: 2 x 4 m16n8k4 fragments; lane (g, tq) reads rows
// k0 + 4 tq .. + 3 of its 8 columns with 32-byte vector loads, two chunks in
// flight in ping-pong registers; MMA step j takes k = k0 + 4 tq + j, the
// same permutation of k for both operands).  Columns past N read column
// N - 1 instead (the Cholesky ignores those Gram entries).  Every segment
// leaves a partial tile; the last CTA to finish a tile folds the partials
// of the CTAs that cover it in CTA order (deterministic).
template <bool VEC>
__global__ void __launch_bounds__(128) cqr_gram_kernel(const GramParams p) {
  pdl_enter();
  if (cq_stopped(p.skip)) return;
  __shared__ double red[4][1024];
  __shared__ int is_last;
  const uint32_t c = blockIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, tq = lane & 3;
  const int64_t d = p.X.d;
  const uint32_t last_chunk = (d % 16) ? p.nchunk - 1 : 0xffffffffu;  // ragged: bounds checks
  const uint32_t u0 = cq_unit_lo(p, c), u1 = cq_unit_lo(p, c + 1);
  const int t_first = (int)(u0 / p.nchunk);
  for (uint32_t ua = u0; ua < u1;) {
    const int t = (int)(ua / p.nchunk);
    const uint32_t tbase = (uint32_t)t * p.nchunk;
    const uint32_t ub = min(u1, tbase + p.nchunk);
    int I, J;
    cq_tile_ij(t, I, J);
    const double* pc[8];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int64_t ca = (int64_t)I * 32 + (q >> 1) * 16 + (q & 1) * 8 + g;
      pc[q] = cq_col(p.X, min(ca, p.N - 1));
      const int64_t cb = (int64_t)J * 32 + q * 8 + g;
      pc[4 + q] = cq_col(p.X, min(cb, p.N - 1));
    }
    double acc[2][4][4];
#pragma unroll
    for (int a2 = 0; a2 < 2; ++a2)
#pragma unroll
      for (int b2 = 0; b2 < 4; ++b2)
#pragma unroll
        for (int c2 = 0; c2 < 4; ++c2) acc[a2][b2][c2] = 0.0;
    const uint32_t ch1 = ub - tbase;
    uint32_t ch = ua - tbase + warp;
    double v0[8][4], v1[8][4];
    if (ch < ch1) cq_gram_load<VEC>(pc, (int64_t)ch * 16 + 4 * tq, d, ch == last_chunk, v0);
    while (ch < ch1) {
      if (ch + 4 < ch1) cq_gram_load<VEC>(pc, (int64_t)(ch + 4) * 16 + 4 * tq, d, ch + 4 == last_chunk, v1);
      cq_gram_mma(acc, v0);
      ch += 4;
      if (ch >= ch1) break;
      if (ch + 4 < ch1) cq_gram_load<VEC>(pc, (int64_t)(ch + 4) * 16 + 4 * tq, d, ch + 4 == last_chunk, v0);
      cq_gram_mma(acc, v1);
      ch += 4;
    }
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
      for (int nt = 0; nt < 4; ++nt)
#pragma unroll
        for (int h = 0; h < 4; ++h) {
          const int r = mt * 16 + g + (h >= 2 ? 8 : 0), cc = nt * 8 + 2 * tq + (h & 1);
          red[warp][cc * 32 + r] = acc[mt][nt][h];
        }
    __syncthreads();
    double* out = p.part + ((int64_t)c * p.SEG + (t - t_first)) * 1024;
    for (int e = threadIdx.x; e < 1024; e += 128)
      out[e] = ((red[0][e] + red[1][e]) + red[2][e]) + red[3][e];
    // CTAs covering tile t: the last one to finish folds their partials
    const uint32_t A = tbase, B = A + p.nchunk;
    uint32_t cf = A * p.P / p.U, cl = (B - 1) * p.P / p.U;
    while (cf > 0 && cq_unit_lo(p, cf) > A) --cf;
    while (cq_unit_lo(p, cf + 1) <= A) ++cf;
    while (cl + 1 < p.P && cq_unit_lo(p, cl + 1) < B) ++cl;
    while (cq_unit_lo(p, cl) >= B) --cl;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) is_last = atomicAdd(&p.cnt[t], 1u) == cl - cf;
    __syncthreads();
    if (is_last) {
      __threadfence();
      double v[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) v[i] = 0.0;
      for (uint32_t q = cf; q <= cl; ++q) {
        const int jq = t - (int)(cq_unit_lo(p, q) / p.nchunk);
        const double* src = p.part + ((int64_t)q * p.SEG + jq) * 1024 + threadIdx.x;
        double w[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) w[i] = __ldcg(src + i * 128);
#pragma unroll
        for (int i = 0; i < 8; ++i) v[i] += w[i];
      }
#pragma unroll
      for (int i = 0; i < 8; ++i) p.Gt[(int64_t)t * 1024 + threadIdx.x + i * 128] = v[i];
      if (p.Gt2 != nullptr)
#pragma unroll
        for (int i = 0; i < 8; ++i) p.Gt2[(int64_t)t * 1024 + threadIdx.x + i * 128] = v[i];
      if (threadIdx.x == 0) p.cnt[t] = 0u;
    }
    __syncthreads();  // red reused by the next segment
    ua = ub;
  }
}

// -------------------------------------------------------------- Cholesky
struct CholParams {
  const double* Gt;    // Gram, upper tiles
  int nb;              // block columns of this factorisation (= cluster CTAs)
  int64_t N;
  double shift_coef;   // > 0: G += shift_coef * trace(G) * I (first iteration; to == 0, all tiles)
  double* Rt;          // R, upper tiles
  double* Rinv;        // inverses of R's diagonal tiles [nb][1024]
  int* flag;           // set on a non-positive / non-finite pivot
  int to;              // tile offset: this cluster factors diagonal block [to, to + nb)
  // blockIdx.y = 1: the unshifted variant (Gt + vs_g, Rt + vs_r, Rinv + vs_i,
  // flag + 1, no shift), factored beside the shifted one
  int64_t vs_g, vs_r, vs_i;
  const int* skip;  // second factorisation: not run (cq_stopped)
};

#ifdef CQ_FACTOR_CLOCKS
__device__ long long cq_factor_clocks[17];
#endif
__device__ __forceinline__ double cq_rcp(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  r = fma(r, fma(-x, r, 1.0), r);  // two Newton steps: ~1 ulp
  return fma(r, fma(-x, r, 1.0), r);
}

// LDL^T of the 32 x 32 tile T (shared, column-major, stride CQ_LD) by one
// warp, lane j holding column j.  On return T holds U (unit upper, 1 on the
// diagonal, 0 below), disq[k] = 1 / sqrt(d_k) (disq is the 32 doubles right
// after T: the pair is pushed to the other CTAs as one block), and Rg
// (global tile, ld 32) R = D^{1/2} U.
//
// Two pivots per pass: with a = G[k][k], b = G[k][k+1], e = G[k+1][k+1],
// l = b / a and d1 = e - b l, lane j forms U[k][j] = G[k][j] / a, the
// eliminated row G'[k+1][j] = G[k+1][j] - l G[k][j] and U[k+1][j] =
// G'[k+1][j] / d1, the two rows are exchanged once through shared memory
// (one 16-byte store and 15 16-byte broadcast loads per lane) and the
// window c[i] = G[k + i][j] of the lane's column takes the rank-2 update
// while shifting by two rows, so the loop body has static register indices
// (rolled loop: the routine runs once per CTA per factorisation, from a cold
// instruction cache).  The next pivot block (lanes k+2, k+3) is formed from
// the lanes' own registers plus one broadcast pair before the bulk update,
// and its first reciprocal is in flight while the update issues.  The whole
// tile is updated (lower entries too: the Gram tiles are symmetric), which
// keeps the loop free of per-lane predicates.  s2[64..127] stay zero, so
// rows past the tile update as no-ops.  A non-positive or non-finite pivot
// only sets the flag (the caller then falls back to Householder).
__device__ __noinline__ void cq_factor(double* T, double* s2, double* Rg, int* flag) {
  const int lane = threadIdx.x & 31;
  double* disq = T + CQ_TILE;
  double c[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) c[i] = T[lane * CQ_LD + i];
  reinterpret_cast<double2*>(s2)[32 + lane] = make_double2(0.0, 0.0);
  double a = __shfl_sync(0xffffffffu, c[0], 0);
  double b = __shfl_sync(0xffffffffu, c[0], 1);
  double e = __shfl_sync(0xffffffffu, c[1], 1);
  double ra = cq_rcp(a);
  bool bad = false;
  double myd = 1.0;
#pragma unroll 1
  for (int k = 0; k < 32; k += 2) {
#ifdef CQ_FACTOR_CLOCKS
    if (lane == 0) cq_factor_clocks[k >> 1] = clock64();
#endif
    const double l = b * ra;
    const double d1 = fma(-b, l, e);
    const double gk = c[0], gk1 = c[1];
    const double u0 = gk * ra;             // U[k][lane]   (lane > k)
    const double gk1p = fma(-l, gk, gk1);  // G'[k+1][lane]
    const bool hi = lane > k + 1;
    reinterpret_cast<double2*>(s2)[lane] = hi ? make_double2(gk, gk1p) : make_double2(0.0, 0.0);
    const double r1 = cq_rcp(d1);
    const double u1 = gk1p * r1;           // U[k+1][lane] (lane > k+1)
    if (lane > k) T[lane * CQ_LD + k] = u0;
    if (hi) T[lane * CQ_LD + k + 1] = u1;
    if (lane == k) myd = a;
    if (lane == k + 1) myd = d1;
    bad |= !(a > 0.0) || !(a < INFINITY) || !(d1 > 0.0) || !(d1 < INFINITY);
    __syncwarp();
    const double2* sr = reinterpret_cast<const double2*>(s2) + k + 2;
    // the next pivot block first: a' on lane k+2, b' and e' on lane k+3
    const double2 v2 = sr[0];
    const double pa = fma(-gk1p, u1, fma(-gk, u0, c[2]));
    const double pe = fma(-gk1p, u1, fma(-gk, u0, c[3]));
    const double pb = fma(-v2.y, u1, fma(-v2.x, u0, c[2]));
    const double an = __shfl_sync(0xffffffffu, pa, (k + 2) & 31);
    const double bn = __shfl_sync(0xffffffffu, pb, (k + 3) & 31);
    const double en = __shfl_sync(0xffffffffu, pe, (k + 3) & 31);
    double rn;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(rn) : "d"(an));
    // rank-2 update of the window, shifted by two rows
#pragma unroll
    for (int i = 0; i < 30; ++i) {
      const double2 v = sr[i];
      c[i] = fma(-v.y, u1, fma(-v.x, u0, c[i + 2]));
    }
    c[30] = 0.0;
    c[31] = 0.0;
    rn = fma(rn, fma(-an, rn, 1.0), rn);
    rn = fma(rn, fma(-an, rn, 1.0), rn);
    __syncwarp();
    a = an;
    b = bn;
    e = en;
    ra = rn;
  }
#ifdef CQ_FACTOR_CLOCKS
  if (lane == 0) cq_factor_clocks[16] = clock64();
#endif
  const double sq = sqrt(myd);
  s2[lane] = sq;
  disq[lane] = 1.0 / sq;
  __syncwarp();
  double uk[32];
#pragma unroll
  for (int k = 0; k < 32; ++k) uk[k] = T[lane * CQ_LD + k];
#pragma unroll
  for (int k = 0; k < 32; ++k) uk[k] = k < lane ? uk[k] : (k == lane ? 1.0 : 0.0);
  __syncwarp();
#pragma unroll
  for (int k = 0; k < 32; ++k) T[lane * CQ_LD + k] = uk[k];
  __syncwarp();
  // R = D^{1/2} U, written coalesced: lane = row, one column per store
#pragma unroll
  for (int cc = 0; cc < 32; ++cc) Rg[cc * 32 + lane] = sq * T[cc * CQ_LD + lane];
  if (bad && lane == 0) atomicExch(flag, 1);
  __syncwarp();
}

// R(K, J) = D_K^{-1/2} U_KK^{-T} G(K, J) in place (T: the tile, shared), one
// warp, lane = column: forward substitution with U broadcast from Us (the
// pushed block: U then 1/sqrt(d)).
__device__ __noinline__ void cq_rowsolve(double* T, const double* Us, double* Rg) {
  const int lane = threadIdx.x & 31;
  const double* isq = Us + CQ_TILE;
  double g[32], sc[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) {
    g[i] = T[lane * CQ_LD + i];
    sc[i] = isq[i];
  }
#pragma unroll
  for (int k = 0; k < 31; ++k)
#pragma unroll
    for (int m = k + 1; m < 32; ++m) g[m] = fma(-Us[m * CQ_LD + k], g[k], g[m]);
  __syncwarp();  // all loads of T done before it is overwritten
#pragma unroll
  for (int k = 0; k < 32; ++k) g[k] *= sc[k];
#pragma unroll
  for (int k = 0; k < 32; ++k) T[lane * CQ_LD + k] = g[k];
  __syncwarp();
#pragma unroll
  for (int cc = 0; cc < 32; ++cc) Rg[cc * 32 + lane] = T[cc * CQ_LD + lane];  // coalesced
}

// C -= A^T B for 32 x 32 tiles (shared, stride CQ_LD): A = R(K, I) (local or
// in CTA `acta` of the cluster), B = R(K, J) local.  The m16n8 fragments
// [MT0, MT0 + NMT) x [NT0, NT0 + NNT).
template <int NMT, int NNT>
__device__ __noinline__ void cq_tile_update(double* C, const double* A, bool a_remote,
                                            uint32_t acta, const double* B, int mt0, int nt0) {
  const int lane = threadIdx.x & 31, g = lane >> 2, tq = lane & 3;
  double acc[NMT][NNT][4];
#pragma unroll
  for (int a = 0; a < NMT; ++a)
#pragma unroll
    for (int b = 0; b < NNT; ++b)
#pragma unroll
      for (int c = 0; c < 4; ++c) acc[a][b][c] = 0.0;
  double af[8][NMT][2];
#pragma unroll
  for (int ks = 0; ks < 8; ++ks)
#pragma unroll
    for (int mt = 0; mt < NMT; ++mt)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const double* src = A + ((mt0 + mt) * 16 + h * 8 + g) * CQ_LD + ks * 4 + tq;
        af[ks][mt][h] = a_remote ? cq_ld_remote(src, acta) : *src;
      }
#pragma unroll
  for (int ks = 0; ks < 8; ++ks)
#pragma unroll
    for (int nt = 0; nt < NNT; ++nt) {
      const double b0 = B[((nt0 + nt) * 8 + g) * CQ_LD + ks * 4 + tq];
#pragma unroll
      for (int mt = 0; mt < NMT; ++mt) cq_dmma(acc[mt][nt], af[ks][mt][0], af[ks][mt][1], b0);
    }
#pragma unroll
  for (int mt = 0; mt < NMT; ++mt)
#pragma unroll
    for (int nt = 0; nt < NNT; ++nt)
#pragma unroll
      for (int h = 0; h < 4; ++h) {
        const int r = (mt0 + mt) * 16 + g + (h >= 2 ? 8 : 0), c = (nt0 + nt) * 8 + 2 * tq + (h & 1);
        C[c * CQ_LD + r] -= acc[mt][nt][h];
      }
}

// Inverse of the diagonal tile R_JJ = D^{1/2} U (U in T, unit upper):
// R^{-1} = U^{-1} D^{-1/2}; lane j builds column j of U^{-1} upward.
__device__ __noinline__ void cq_diag_inverse(const double* T, double* out, double* scratch) {
  const int lane = threadIdx.x & 31;
  const double* disq = T + CQ_TILE;
  double acc[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) acc[i] = 0.0;
  double x[32];
#pragma unroll
  for (int m = 31; m >= 0; --m) {
    const double xm = m == lane ? 1.0 : (m < lane ? -acc[m] : 0.0);
    x[m] = xm;
#pragma unroll
    for (int i = 0; i < m; ++i) acc[i] = fma(T[m * CQ_LD + i], xm, acc[i]);
  }
  // out (column-major, ld 32) = X diag(disq): lane j holds column j; go
  // through shared memory (the first 33 x 32 doubles of `scratch`) so the
  // global stores are coalesced
  const double sc = disq[lane];
#pragma unroll
  for (int i = 0; i < 32; ++i) scratch[i * CQ_LD + lane] = x[i] * sc;
  __syncwarp();
#pragma unroll
  for (int cc = 0; cc < 32; ++cc) out[cc * 32 + lane] = scratch[lane * CQ_LD + cc];
}

constexpr uint32_t CQ_PUSH_BYTES = (CQ_TILE + 32) * sizeof(double);

// The owner of a freshly factored diagonal tile pushes U and 1/sqrt(d) (one
// contiguous block) into buffer `buf` of every CTA that still needs it,
// completing on that CTA's mbarrier.
__device__ __forceinline__ void cq_push(const double* blk, int from, int nb, double (*Us)[CQ_TILE + 32],
                                        uint64_t* mbar, int buf) {
  fence_proxy_async_smem();
  __syncwarp();
  if ((threadIdx.x & 31) == 0)
    for (int dst = from + 1; dst < nb; ++dst)
      bulk_s2cluster(mapa_u32(smem_u32(&Us[buf][0]), (uint32_t)dst), blk, CQ_PUSH_BYTES,
                     mapa_u32(smem_u32(&mbar[buf]), (uint32_t)dst));
}

__global__ void __launch_bounds__(CQ_CHOL_NT, 1) cqr_chol_kernel(const CholParams p0) {
  CholParams p = p0;
  if (blockIdx.y) {
    p.Gt += p.vs_g;
    p.Rt += p.vs_r;
    p.Rinv += p.vs_i;
    p.flag += 1;
    p.shift_coef = 0.0;
  }
  // tiles (I, J) of my block column, I = 0..J, then 32 doubles (1/sqrt of
  // my pivots) right after my diagonal tile
  extern __shared__ __align__(16) double csm[];
  __shared__ __align__(16) double Us[2][CQ_TILE + 32];  // pushed U_KK | 1/sqrt(d_K)
  __shared__ __align__(8) uint64_t mbar[2];
  __shared__ __align__(16) double srow[128];
  const int J = (int)cq_rank();
  const int nb = p.nb;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  double* T = csm;
  auto tile = [&](int I) { return T + I * CQ_TILE; };
  if (tid == 0) {
    mbar_init(&mbar[0], 1);
    mbar_init(&mbar[1], 1);
    fence_mbar_init();
    // arm the first two receptions (steps 0 and 1)
    if (J > 0) mbar_arrive_expect_tx(&mbar[0], CQ_PUSH_BYTES);
    if (J > 1) mbar_arrive_expect_tx(&mbar[1], CQ_PUSH_BYTES);
  }
  pdl_enter();
  if (cq_stopped(p.skip)) return;  // every CTA of the cluster alike
  CQ_PROBE(0);
  // my column's Gram tiles, all copies in flight at once (8-byte cp.async;
  // past N: zero-filled, identity on the diagonal below)
  for (int I = 0; I <= J; ++I) {
    const double* src = p.Gt + cq_tile(I + p.to, J + p.to) * 1024;
    double* dst = tile(I);
    for (int e = tid; e < 1024; e += CQ_CHOL_NT) {
      const int r = e & 31, c = e >> 5;
      const bool ok = (int64_t)(I + p.to) * 32 + r < p.N && (int64_t)(J + p.to) * 32 + c < p.N;
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(smem_u32(dst + c * CQ_LD + r)),
                   "l"(src + e), "r"(ok ? 8 : 0)
                   : "memory");
    }
  }
  asm volatile("cp.async.commit_group;\n\tcp.async.wait_all;" ::: "memory");
  __syncthreads();
  if (warp == 0) {
    const int64_t gi = (int64_t)(J + p.to) * 32 + lane;
    if (gi >= p.N) tile(J)[lane * (CQ_LD + 1)] = 1.0;
    if (p.shift_coef > 0.0) {
      // the same fixed-order trace in every CTA
      double s = 0.0;
      for (int b = 0; b < nb; ++b)
        if ((int64_t)b * 32 + lane < p.N) s += p.Gt[cq_tile(b, b) * 1024 + lane * 33];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if (gi < p.N) tile(J)[lane * (CQ_LD + 1)] += p.shift_coef * s;
    }
  }
  __syncthreads();
  CQ_PROBE(1);
  // every CTA's mbarriers are initialised before the first push
  cq_arrive();
  cq_wait();
  if (J == 0 && warp == 0) {
    cq_factor(tile(0), srow, p.Rt + cq_tile(p.to, p.to) * 1024, p.flag);
    cq_push(tile(0), 0, nb, Us, mbar, 0);
  }
  for (int K = 0; K < nb - 1; ++K) {
    const int buf = K & 1;
    if (J > K) {
      // U_KK pushed by CTA K, then R(K, J)
      mbar_wait_cluster(&mbar[buf], (uint32_t)((K >> 1) & 1));
      CQ_PROBE(2 + 4 * K);
      if (warp == 0) cq_rowsolve(tile(K), Us[buf], p.Rt + cq_tile(K + p.to, J + p.to) * 1024);
      __syncthreads();
      if (tid == 0 && K + 2 < J) mbar_arrive_expect_tx(&mbar[buf], CQ_PUSH_BYTES);
    }
    CQ_PROBE(3 + 4 * K);
    cq_arrive();  // R(K, J) published
    if (J == K + 1) {
      // the next diagonal tile: its update is local; factor and push it
      // while the other CTAs wait for the barrier
      if (warp < 4)
        cq_tile_update<1, 2>(tile(J), tile(K), false, 0, tile(K), warp >> 1, (warp & 1) * 2);
      __syncthreads();
      if (warp == 0) {
        cq_factor(tile(J), srow, p.Rt + cq_tile(J + p.to, J + p.to) * 1024, p.flag);
        cq_push(tile(J), J, nb, Us, mbar, (K + 1) & 1);
      }
    }
    cq_wait();
    CQ_PROBE(4 + 4 * K);
    if (J > K + 1) {
      // tiles (I, J), K < I <= J: T_I -= R(K, I)^T R(K, J), one warp each
      for (int I = K + 1 + warp; I <= J; I += CQ_CHOL_NT / 32)
        cq_tile_update<2, 4>(tile(I), tile(K), I != J, (uint32_t)I, tile(K), 0, 0);
      __syncthreads();
    }
    CQ_PROBE(5 + 4 * K);
  }
  if (warp == 0) cq_diag_inverse(tile(J), p.Rinv + (int64_t)(J + p.to) * 1024, Us[0]);
  CQ_PROBE(70);
  // shared memory stays alive until every remote reader is done
  cq_arrive();
  cq_wait();
}

// ------------------------------------------- Cholesky beyond 16 block columns
// N > 512: right-looking over super-blocks of up to 16 tiles.  For the
// super-block [to, to + nbs): the cluster kernel factors its diagonal block,
// the block row R(to.., J) = R11^{-T} G(to.., J) of every later tile column
// J is the TRSM of G^T by R11 (cqr_trsm_df_kernel<true>), cqr_syrk_kernel applies
// G(I, J) -= sum_K R(K, I)^T R(K, J) to the trailing tiles.  The shift of
// the first factorisation is applied once beforehand (cqr_shift_kernel),
// because the trailing updates change the later diagonal tiles.
constexpr int CQ_MAXNB_BIG = 33;  // N <= 1056

// acc += A^T B for 32 x 32 global tiles (column-major, ld 32), one warp.
__device__ __forceinline__ void cq_gtile_mma_tn(double (&acc)[2][4][4], const double* A,
                                                const double* B) {
  const int lane = threadIdx.x & 31, g = lane >> 2, tq = lane & 3;
  double af[8][2][2], bf[8][4];
#pragma unroll
  for (int ks = 0; ks < 8; ++ks) {
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
      for (int h = 0; h < 2; ++h) af[ks][mt][h] = __ldcg(A + (mt * 16 + h * 8 + g) * 32 + ks * 4 + tq);
#pragma unroll
    for (int nt = 0; nt < 4; ++nt) bf[ks][nt] = __ldcg(B + (nt * 8 + g) * 32 + ks * 4 + tq);
  }
#pragma unroll
  for (int ks = 0; ks < 8; ++ks)
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) cq_dmma(acc[mt][nt], af[ks][mt][0], af[ks][mt][1], bf[ks][nt]);
}

// Fixed-order fold of 8 warps' accumulators into red[0..3] -> sum tile (column-major).
__device__ __forceinline__ void cq_fold8(double (&acc)[2][4][4], double (*red)[1024]) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, tq = lane & 3;
  auto spill = [&](int w, bool add) {
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
      for (int nt = 0; nt < 4; ++nt)
#pragma unroll
        for (int h = 0; h < 4; ++h) {
          double& r = red[w][(nt * 8 + 2 * tq + (h & 1)) * 32 + mt * 16 + g + (h >= 2 ? 8 : 0)];
          r = add ? r + acc[mt][nt][h] : acc[mt][nt][h];
        }
  };
  if (warp >= 4) spill(warp - 4, false);
  __syncthreads();
  if (warp < 4) spill(warp, true);
  __syncthreads();
}

struct TriParams {
  double* Gt;         // Gram (updated), tile layout
  double* Rt;         // R tiles (diagonal block [to, to+nbs) factored)
  const double* Rinv; // inverses of R's diagonal tiles
  int to, nbs, nb;
  int64_t vs_g, vs_r;  // blockIdx.y = 1: the unshifted variant's buffers
  const int* skip;
};

__global__ void __launch_bounds__(256) cqr_syrk_kernel(const TriParams p0) {
  __shared__ double red[4][1024];
  TriParams p = p0;
  if (blockIdx.y) {
    p.Gt += p.vs_g;
    p.Rt += p.vs_r;
  }
  pdl_enter();
  if (cq_stopped(p.skip)) return;
  int jj = (int)((sqrtf(8.0f * blockIdx.x + 1.0f) - 1.0f) * 0.5f);
  while ((jj + 1) * (jj + 2) / 2 <= (int)blockIdx.x) ++jj;
  while (jj * (jj + 1) / 2 > (int)blockIdx.x) --jj;
  const int ii = (int)blockIdx.x - jj * (jj + 1) / 2;
  const int base = p.to + p.nbs, I = base + ii, J = base + jj;
  const int warp = threadIdx.x >> 5;
  double acc[2][4][4];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b)
#pragma unroll
      for (int c = 0; c < 4; ++c) acc[a][b][c] = 0.0;
  for (int K = p.to + warp; K < p.to + p.nbs; K += 8)
    cq_gtile_mma_tn(acc, p.Rt + cq_tile(K, I) * 1024, p.Rt + cq_tile(K, J) * 1024);
  cq_fold8(acc, red);
  double* gij = p.Gt + cq_tile(I, J) * 1024;
  for (int e = threadIdx.x; e < 1024; e += 256)
    gij[e] = __ldcg(gij + e) - (((red[0][e] + red[1][e]) + red[2][e]) + red[3][e]);
}

// G += shift_coef * trace(G) * I over the first N diagonal entries, and
// fro2 = ||SA||_F^2 (the first n diagonal entries of the unshifted G), both
// in a fixed order.  One CTA.
__global__ void __launch_bounds__(1024) cqr_shift_kernel(double* Gt, int64_t N, int64_t n,
                                                         double shift_coef, double* fro2) {
  __shared__ double red[2][32];
  pdl_enter();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double t = 0.0, f = 0.0;
  for (int64_t i = tid; i < N; i += 1024) {
    const double v = Gt[cq_tile((int)(i >> 5), (int)(i >> 5)) * 1024 + (i & 31) * 33];
    t += v;
    if (i < n) f += v;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    t += __shfl_xor_sync(0xffffffffu, t, o);
    f += __shfl_xor_sync(0xffffffffu, f, o);
  }
  if (lane == 0) {
    red[0][warp] = t;
    red[1][warp] = f;
  }
  __syncthreads();
  double tr = 0.0, fr = 0.0;
  for (int w = 0; w < 32; ++w) {
    tr += red[0][w];
    fr += red[1][w];
  }
  if (tid == 0) *fro2 = fr;
  for (int64_t i = tid; i < N; i += 1024)
    Gt[cq_tile((int)(i >> 5), (int)(i >> 5)) * 1024 + (i & 31) * 33] += shift_coef * tr;
}

// ------------------------------------------------------------------ TRSM
struct TrsmParams {
  CqCols X;
  int64_t N;
  int nb;
  const double* Rt;
  const double* Rinv;
  double* Q;
  int64_t ldq;
  const double* Rf;   // R's tiles in B-fragment order (cqr_rfrag_kernel)
  const double* Rfi;  // the diagonal tiles' inverses, same order
  // block-row solve of the blocked Cholesky (GT): X = G(to.., J0..)^T, R and
  // Rinv tiles offset by `to`, the result R(to.., J0..) written as tiles
  const double* G;
  double* Rout;
  int to, J0;
  int64_t vs_g, vs_r, vs_i;  // GT, blockIdx.y = 1: the unshifted variant (G, Rout and Rf, Rfi)
  const int* skip;           // cq_stopped: return at once
  // X = I (the rows r0.. of the identity): Q = R^{-1}, rows r0.. (block
  // columns before r0's start out and stay zero); run only when *need
  int ident;
  const int* need;
  // X from the rows of R's tile layout: X(r, c) = R(r, to * 32 + c) (the
  // off-diagonal block of the 2 x 2 split of R^{-1}); nullptr: X as above
  const double* XR;
};

constexpr int CQ_TRSM_WARPS = 8;
constexpr int CQ_TRSM_NT = CQ_TRSM_WARPS * 32;

// R tiles re-laid in the order the DMMA B fragments consume them: for each
// tile, 16 rows of 32 double2 (q = ks * 2 + np holds bf[ks][2np], bf[ks][2np+1]
// of every lane), so a warp's fetch of a tile is 16 fully used 512-byte loads
// instead of 32 loads touching 8 separate 128-byte lines each -- the TRSM
// streams all of R once per 16-row block, and the scattered loads made it
// bound by the L1 wavefront rate rather than by the fp64 tensor pipe.
// Blocks [0, nbs (nbs + 1) / 2): the upper tiles of the diagonal block that
// starts at tile `to`; the next nbs blocks: its diagonal tiles' inverses.
// The pick after the first factorisation: take the unshifted variant (1)
// when it did not break down and its R's diagonal over the n columns of SA
// spans less than CQ_REFINE_RATIO.  Its R1 is then the Cholesky factor of
// the normal equations of a well-conditioned SA, x = R1^{-1} R1^{-T} SA^T Sb
// is within ~kappa^2 u, and one corrected semi-normal step brings it to
// ~kappa u (the error contracts by ~kappa^2 u per step): the CholeskyQR2
// kernels after the pick return at once.  The shifted variant (0,
// CholeskyQR2) otherwise.  Block-wide (every CTA of the kernel that makes
// it reaches the same answer); the result in every thread.
__device__ __noinline__ int cq_pick(const double* R1u, int64_t n, const int* flag) {
  __shared__ double red[2][32];
  __shared__ int res;
  double lo = INFINITY, hi = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    const double v = R1u[cq_tile((int)(i >> 5), (int)(i >> 5)) * 1024 + (i & 31) * 33];
    const bool ok = v > 0.0 && v < INFINITY;
    lo = ok ? fmin(lo, v) : -1.0;
    hi = ok ? fmax(hi, v) : INFINITY;
    if (!ok) break;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, o));
    hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, o));
  }
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    red[0][w] = lo;
    red[1][w] = hi;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int k = 0; k < (int)(blockDim.x >> 5); ++k) {
      lo = fmin(lo, red[0][k]);
      hi = fmax(hi, red[1][k]);
    }
    res = (flag[1] == 0 && lo > 0.0 && hi < CQ_REFINE_RATIO * lo) ? 1 : 0;
  }
  __syncthreads();
  return res;
}

// Variant blockIdx.y (buffers of variant 1 at + vs_r / + vs_i).
struct FragParams {
  const double* Rt;
  const double* Rinv;
  double* Rf;
  double* Rfi;
  int to, nbs;
  int64_t vs_r, vs_i;
  const int* skip;  // cq_stopped: return at once
  const int* need;  // run only when *need
  // pick != nullptr (after the first factorisation): every CTA makes the
  // pick (cq_pick, R1u's diagonal = Rt + vs_r), takes that variant as the
  // source, and CTA 0 records it (pick[2]; pick[0] = 0 when the unshifted
  // variant is taken: the flag then describes the chosen variant)
  int* pick;
  int64_t n;
};

__global__ void __launch_bounds__(256) cqr_rfrag_kernel(const FragParams fp) {
  pdl_enter();
  if (cq_stopped(fp.skip) || (fp.need != nullptr && *fp.need == 0)) return;
  int vs = (int)blockIdx.y;
  const int vd = (int)blockIdx.y;
  if (fp.pick != nullptr) {
    vs = cq_pick(fp.Rt + fp.vs_r, fp.n, fp.pick);
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      fp.pick[2] = vs;
      if (vs) fp.pick[0] = 0;
    }
  }
  const double* Rt = fp.Rt + vs * fp.vs_r;
  const double* Rinv = fp.Rinv + vs * fp.vs_i;
  double* Rf = fp.Rf + vd * fp.vs_r;
  double* Rfi = fp.Rfi + vd * fp.vs_i;
  const int to = fp.to, nbs = fp.nbs;
  const int t = blockIdx.x, ntl = nbs * (nbs + 1) / 2;
  const double* src;
  double* dst;
  if (t < ntl) {
    int J = (int)((sqrtf(8.0f * t + 1.0f) - 1.0f) * 0.5f);
    while ((J + 1) * (J + 2) / 2 <= t) ++J;
    while (J * (J + 1) / 2 > t) --J;
    const int64_t base = cq_tile(to + t - J * (J + 1) / 2, to + J) * 1024;
    src = Rt + base;
    dst = Rf + base;
  } else {
    const int64_t base = (int64_t)(to + t - ntl) * 1024;
    src = Rinv + base;
    dst = Rfi + base;
  }
#pragma unroll
  for (int q4 = 0; q4 < 4; ++q4) {
    const int o = threadIdx.x + q4 * 256;
    const int pr = o >> 1, lane = pr & 31, q = pr >> 5;
    const int ks = q >> 1, nt = 2 * (q & 1) + (o & 1), g = lane >> 2, tq = lane & 3;
    dst[o] = __ldg(src + (nt * 8 + g) * 32 + ks * 4 + tq);
  }
}

__device__ __forceinline__ void cq_trsm_fetch_rf(const double* rf, double (&bf)[8][4]) {
  const double2* f = reinterpret_cast<const double2*>(rf) + (threadIdx.x & 31);
#pragma unroll
  for (int ks = 0; ks < 8; ++ks)
#pragma unroll
    for (int np = 0; np < 2; ++np) {
      const double2 v = __ldg(f + (ks * 2 + np) * 32);
      bf[ks][2 * np] = v.x;
      bf[ks][2 * np + 1] = v.y;
    }
}

// Q_L = T_L Rinv_LL (bi), stored over T_L and to the output, then released.
template <bool GT>
__device__ __forceinline__ void cq_df_form_q(const TrsmParams& p, double* tsm, int L, int Jt, int rb,
                                             int64_t r0, const double (&bi)[8][4], uint64_t* bar) {
  const int lane = threadIdx.x & 31, g = lane >> 2, tq = lane & 3;
  __syncwarp();  // the warp's updates of T_L visible to all its lanes
  double qa[2][4][4];  // ks halves: half the dependent DMMA depth
#pragma unroll
  for (int s2 = 0; s2 < 2; ++s2)
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) qa[s2][a][b] = 0.0;
#pragma unroll
  for (int ks = 0; ks < 8; ++ks) {
    const int k = L * 32 + ks * 4 + tq;
    const double a0 = tsm[k * CQ_QLD + g], a1 = tsm[k * CQ_QLD + g + 8];
#pragma unroll
    for (int nt = 0; nt < 4; ++nt) cq_dmma(qa[ks >> 2][nt], a0, a1, bi[ks][nt]);
  }
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) qa[0][a][b] += qa[1][a][b];
  __syncwarp();  // every lane's reads of T_L done
  double* out = GT ? p.Rout + cq_tile(p.to + L, Jt) * 1024 : nullptr;
#pragma unroll
  for (int nt = 0; nt < 4; ++nt)
#pragma unroll
    for (int h = 0; h < 4; ++h) {
      const int r = g + (h >= 2 ? 8 : 0), c = nt * 8 + 2 * tq + (h & 1);
      tsm[(L * 32 + c) * CQ_QLD + r] = qa[0][nt][h];
      if (GT) {
        out[(rb + r) * 32 + c] = qa[0][nt][h];
      } else {
        const int64_t gc = (int64_t)L * 32 + c, gr = r0 + r;
        if (gc < p.N && gr < p.X.d) p.Q[gc * p.ldq + gr] = qa[0][nt][h];
      }
    }
  mbar_arrive(bar);
}

// T_L -= Q_J R(J, L), R(J, L) in bf.  CHAIN (the link that makes T_L final):
// two accumulator sets over ks halves (half the dependent DMMA depth), no
// prefetch; else the fragments of my next tile (L + 8) are fetched into bn
// before the product issues.
template <bool CHAIN>
__device__ __forceinline__ void cq_df_update(const TrsmParams& p, double* tsm, int J, int L,
                                             const double (&qf0)[8], const double (&qf1)[8],
                                             const double (&bf)[8][4], double (&bn)[8][4]) {
  const int lane = threadIdx.x & 31, g = lane >> 2, tq = lane & 3;
  if (!CHAIN && L + CQ_TRSM_WARPS < p.nb)
    cq_trsm_fetch_rf(p.Rf + cq_tile(p.to + J, p.to + L + CQ_TRSM_WARPS) * 1024, bn);
  constexpr int NS = CHAIN ? 2 : 1;
  double acc[NS][4][4];
#pragma unroll
  for (int s2 = 0; s2 < NS; ++s2)
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) acc[s2][a][b] = 0.0;
#pragma unroll
  for (int ks = 0; ks < 8; ++ks)
#pragma unroll
    for (int nt = 0; nt < 4; ++nt) cq_dmma(acc[CHAIN ? ks >> 2 : 0][nt], qf0[ks], qf1[ks], bf[ks][nt]);
#pragma unroll
  for (int nt = 0; nt < 4; ++nt)
#pragma unroll
    for (int h = 0; h < 4; ++h) {
      const int r = g + (h >= 2 ? 8 : 0), c = nt * 8 + 2 * tq + (h & 1);
      tsm[(L * 32 + c) * CQ_QLD + r] -= CHAIN ? acc[0][nt][h] + acc[NS - 1][nt][h] : acc[0][nt][h];
    }
}

__device__ __forceinline__ void cq_copy_frags(double (&dst)[8][4], const double (&src)[8][4]) {
#pragma unroll
  for (int ks = 0; ks < 8; ++ks)
#pragma unroll
    for (int nt = 0; nt < 4; ++nt) dst[ks][nt] = src[ks][nt];
}

template <bool GT>
__device__ __forceinline__ void cq_df_body(const TrsmParams& p0, int blk) {
  extern __shared__ __align__(16) double tsm[];  // T[c * CQ_QLD + r]; becomes Q
  __shared__ __align__(8) uint64_t qbar[CQ_MAXNB_BIG];
  TrsmParams p = p0;
  if (GT && blockIdx.y) {
    p.G += p.vs_g;
    p.Rout += p.vs_r;
    p.Rf += p.vs_r;
    p.Rfi += p.vs_i;
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, tq = lane & 3;
  const int64_t r0 = (int64_t)blk * CQ_TRSM_ROWS;
  const int64_t d = p.X.d;
  const int nb = p.nb, ncol = nb * 32;
  const int Jt = p.J0 + (int)(r0 >> 5), rb = (int)(r0 & 31);
  if (threadIdx.x < nb) mbar_init(&qbar[threadIdx.x], 32);
  pdl_enter();
  if (cq_stopped(p.skip) || (p.need != nullptr && *p.need == 0)) return;
  const int Js = (!GT && p.ident) ? (int)(r0 >> 5) : 0;  // first nonzero block column
  // T = X: every 8-byte copy in flight at once (zero-filled past N and d)
  if (!GT && p.ident) {
    for (int e = threadIdx.x; e < ncol * CQ_TRSM_ROWS; e += CQ_TRSM_NT)
      tsm[(e >> 4) * CQ_QLD + (e & 15)] = (r0 + (e & 15) == (e >> 4)) ? 1.0 : 0.0;
  } else if (GT) {  // X(r, c) = G(c, r): 16 contiguous rows of 32 in each tile
    for (int e = threadIdx.x; e < ncol * CQ_TRSM_ROWS; e += CQ_TRSM_NT) {
      const int ci = e & 31, r = (e >> 5) & 15, cI = e >> 9;
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(
                       smem_u32(tsm + (cI * 32 + ci) * CQ_QLD + r)),
                   "l"(p.G + cq_tile(p.to + cI, Jt) * 1024 + (rb + r) * 32 + ci)
                   : "memory");
    }
  } else if (p.XR != nullptr) {  // X(r, c) = R(r0 + r, to * 32 + c): 16 contiguous doubles per column
    for (int e = threadIdx.x; e < ncol * CQ_TRSM_ROWS; e += CQ_TRSM_NT) {
      const int r = e & 15, c = e >> 4;
      const int64_t gr = r0 + r;
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(tsm + c * CQ_QLD + r)),
                   "l"(p.XR + cq_tile((int)(gr >> 5), p.to + (c >> 5)) * 1024 + (c & 31) * 32 + (gr & 31))
                   : "memory");
    }
  } else {
    for (int e = threadIdx.x; e < ncol * CQ_TRSM_ROWS; e += CQ_TRSM_NT) {
      const int r = e & 15, c = e >> 4;
      const int64_t gr = r0 + r;
      const bool ok = c < p.N && gr < d;
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(
                       smem_u32(tsm + c * CQ_QLD + r)),
                   "l"(ok ? cq_col(p.X, c) + gr : p.X.A), "r"(ok ? 8 : 0)
                   : "memory");
    }
  }
  asm volatile("cp.async.commit_group;\n\tcp.async.wait_all;" ::: "memory");
  __syncthreads();
  if (warp == Js % CQ_TRSM_WARPS) {
    double bi[8][4];
    cq_trsm_fetch_rf(p.Rfi + (int64_t)(p.to + Js) * 1024, bi);
    cq_df_form_q<GT>(p, tsm, Js, Jt, rb, r0, bi, &qbar[Js]);
  }
  for (int J = Js; J + 1 < nb; ++J) {
    const int L0 = J + 1 + ((warp - (J + 1)) % 8 + 8) % 8;  // my first block column > J
    if (L0 >= nb) break;
    double bf[8][4];
    cq_trsm_fetch_rf(p.Rf + cq_tile(p.to + J, p.to + L0) * 1024, bf);
    double qf0[8], qf1[8];
    int L = L0;
    if (L0 == J + 1) {  // T_{J+1} becomes final here: the next link of the chain first
      double bi[8][4];
      cq_trsm_fetch_rf(p.Rfi + (int64_t)(p.to + L0) * 1024, bi);
      mbar_wait(&qbar[J], 0);
#pragma unroll
      for (int ks = 0; ks < 8; ++ks) {
        const int k = J * 32 + ks * 4 + tq;
        qf0[ks] = tsm[k * CQ_QLD + g];
        qf1[ks] = tsm[k * CQ_QLD + g + 8];
      }
      cq_df_update<true>(p, tsm, J, L, qf0, qf1, bf, bf);
      cq_df_form_q<GT>(p, tsm, L, Jt, rb, r0, bi, &qbar[L]);
      L += CQ_TRSM_WARPS;
      if (L < nb) cq_trsm_fetch_rf(p.Rf + cq_tile(p.to + J, p.to + L) * 1024, bf);
    } else {
      mbar_wait(&qbar[J], 0);
#pragma unroll
      for (int ks = 0; ks < 8; ++ks) {
        const int k = J * 32 + ks * 4 + tq;
        qf0[ks] = tsm[k * CQ_QLD + g];
        qf1[ks] = tsm[k * CQ_QLD + g + 8];
      }
    }
    for (; L < nb; L += CQ_TRSM_WARPS) {
      double bn[8][4];
      cq_df_update<false>(p, tsm, J, L, qf0, qf1, bf, bn);
      cq_copy_frags(bf, bn);
    }
  }
}

template <bool GT>
__global__ void __launch_bounds__(CQ_TRSM_NT, 1) cqr_trsm_df_kernel(const TrsmParams p) {
  cq_df_body<GT>(p, (int)blockIdx.x);
}

// Up to three independent TRSMs in one launch (CTA ranges [cta0[k],
// cta0[k+1])): the 2 x 2 split of R^{-1} -- A^{-1} and C^{-1} of the two
// diagonal blocks, and W = B C^{-1} for the off-diagonal block B -- whose
// chains then run side by side, each at most half as long as R^{-1}'s.
struct TrsmBatch {
  TrsmParams p[3];
  int cta0[4];
};

__global__ void __launch_bounds__(CQ_TRSM_NT, 1) cqr_trsm_df_batch_kernel(const TrsmBatch b) {
  const int x = (int)blockIdx.x;
  const int k = x < b.cta0[1] ? 0 : (x < b.cta0[2] ? 1 : 2);
  cq_df_body<false>(b.p[k], x - b.cta0[k]);
}

// The off-diagonal block of R^{-1} = [[A^{-1}, -A^{-1} B C^{-1}], [0, C^{-1}]]:
// out = -Ai W with Ai = A^{-1} (h x h tiles, upper; dense column-major at
// ld) and W = B C^{-1} (ld ldw).  One CTA per 32 x 32 output tile, the K
// tiles I..h-1 split over the 8 warps and folded in fixed order.
__device__ __forceinline__ void cq_dtile_mma(double (&acc)[2][4][4], const double* X, int64_t ldx,
                                             const double* Y, int64_t ldy) {
  const int lane = threadIdx.x & 31, g = lane >> 2, tq = lane & 3;
#pragma unroll
  for (int ks = 0; ks < 8; ++ks) {
    double af[2][2], bf[4];
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
      for (int h2 = 0; h2 < 2; ++h2) af[mt][h2] = __ldcg(X + (int64_t)(ks * 4 + tq) * ldx + mt * 16 + h2 * 8 + g);
#pragma unroll
    for (int nt = 0; nt < 4; ++nt) bf[nt] = __ldcg(Y + (int64_t)(nt * 8 + g) * ldy + ks * 4 + tq);
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) cq_dmma(acc[mt][nt], af[mt][0], af[mt][1], bf[nt]);
  }
}

__global__ void __launch_bounds__(256) cqr_rinv_offdiag_kernel(double* Ri, int64_t ld, int h, int nc,
                                                               int64_t ncols, const double* W,
                                                               int64_t ldw, const int* need) {
  __shared__ double red[4][1024];
  pdl_enter();
  if (*need == 0) return;
  const int I = (int)blockIdx.x % h, J = (int)blockIdx.x / h;  // output tile (I, h + J)
  const int warp = threadIdx.x >> 5;
  double acc[2][4][4];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b2 = 0; b2 < 4; ++b2)
#pragma unroll
      for (int c = 0; c < 4; ++c) acc[a][b2][c] = 0.0;
  for (int K = I + warp; K < h; K += 8)
    cq_dtile_mma(acc, Ri + (int64_t)K * 32 * ld + I * 32, ld, W + (int64_t)J * 32 * ldw + K * 32, ldw);
  cq_fold8(acc, red);
  for (int e = threadIdx.x; e < 1024; e += 256) {
    const int r = e & 31, c = e >> 5;
    const int64_t gc = (int64_t)(h + J) * 32 + c;
    if (gc < ncols)
      Ri[gc * ld + I * 32 + r] = -(((red[0][e] + red[1][e]) + red[2][e]) + red[3][e]);
  }
  (void)nc;
}

// ----------------------------------------------------------------- solves
// R = R2 R1 (upper, tile layout) and the inverses of its diagonal tiles
// (R_II^{-1} = R1_II^{-1} R2_II^{-1}).  One CTA per upper tile, the K terms
// of the tile product split over the 8 warps and folded in fixed order.
struct ProdParams {
  const double* R1t;
  const double* R2t;
  const double* R1inv;
  const double* R2inv;
  double* Rt;
  double* Rinv;
  const int* sel;        // R1 of the unshifted variant (+ vs_r, + vs_i) when *sel
  int64_t vs_r, vs_i;
};

// acc += A B for 32 x 32 global tiles (column-major, ld 32), one warp.
__device__ __forceinline__ void cq_gtile_mma(double (&acc)[2][4][4], const double* A,
                                             const double* B) {
  const int lane = threadIdx.x & 31, g = lane >> 2, tq = lane & 3;
  double af[8][2][2], bf[8][4];
#pragma unroll
  for (int ks = 0; ks < 8; ++ks) {
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
      for (int h = 0; h < 2; ++h) af[ks][mt][h] = __ldg(A + (ks * 4 + tq) * 32 + mt * 16 + h * 8 + g);
#pragma unroll
    for (int nt = 0; nt < 4; ++nt) bf[ks][nt] = __ldg(B + (nt * 8 + g) * 32 + ks * 4 + tq);
  }
#pragma unroll
  for (int ks = 0; ks < 8; ++ks)
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) cq_dmma(acc[mt][nt], af[ks][mt][0], af[ks][mt][1], bf[ks][nt]);
}

__global__ void __launch_bounds__(256) cqr_rprod_kernel(const ProdParams p0) {
  __shared__ double red[4][1024];
  pdl_enter();
  const ProdParams& p = p0;
  const int t = blockIdx.x;
  int J = (int)((sqrtf(8.0f * t + 1.0f) - 1.0f) * 0.5f);
  while ((J + 1) * (J + 2) / 2 <= t) ++J;
  while (J * (J + 1) / 2 > t) --J;
  const int I = t - J * (J + 1) / 2;
  if (p.sel != nullptr && *p.sel) {  // semi-normal solve: R = R1 of the unshifted variant
    for (int e = threadIdx.x; e < 1024; e += 256) {
      p.Rt[(int64_t)t * 1024 + e] = p.R1t[p.vs_r + (int64_t)t * 1024 + e];
      if (I == J) p.Rinv[(int64_t)I * 1024 + e] = p.R1inv[p.vs_i + (int64_t)I * 1024 + e];
    }
    return;
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, tq = lane & 3;
  double acc[2][4][4];
  auto zero = [&]() {
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int b2 = 0; b2 < 4; ++b2)
#pragma unroll
        for (int c = 0; c < 4; ++c) acc[a][b2][c] = 0.0;
  };
  auto spill = [&](int w, bool add) {
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
      for (int nt = 0; nt < 4; ++nt)
#pragma unroll
        for (int h = 0; h < 4; ++h) {
          double& r = red[w][(nt * 8 + 2 * tq + (h & 1)) * 32 + mt * 16 + g + (h >= 2 ? 8 : 0)];
          r = add ? r + acc[mt][nt][h] : acc[mt][nt][h];
        }
  };
  zero();
  for (int K = I + warp; K <= J; K += 8)
    cq_gtile_mma(acc, p.R2t + cq_tile(I, K) * 1024, p.R1t + cq_tile(K, J) * 1024);
  // fixed-order fold of the 8 warps' partial tiles: (w + 4) into w, then 0..3
  if (warp >= 4) spill(warp - 4, false);
  __syncthreads();
  if (warp < 4) spill(warp, true);
  __syncthreads();
  for (int e = threadIdx.x; e < 1024; e += 256)
    p.Rt[(int64_t)t * 1024 + e] = ((red[0][e] + red[1][e]) + red[2][e]) + red[3][e];
  if (I == J) {
    __syncthreads();
    if (warp == 0) {
      zero();
      cq_gtile_mma(acc, p.R1inv + (int64_t)I * 1024, p.R2inv + (int64_t)I * 1024);
      spill(0, false);
    }
    __syncthreads();
    for (int e = threadIdx.x; e < 1024; e += 256) p.Rinv[(int64_t)I * 1024 + e] = red[0][e];
  }
}

struct SolveParams {
  int* refine;         // set by solve_a: run the refinement step
  const double* fro2;  // ||SA||_F^2 when the shift kernel ran (G1 shifted in place), else null
  const double* G1t;   // Gram of M (unshifted): ||SA||_F from its diagonal
  const double* Rt;    // R = R2 R1, upper tiles (order N = n + 1)
  const double* Rinv;  // inverses of its diagonal tiles
  int64_t n;           // R[:n,:n]; column n = Q^T Sb
  const int* flag;
  double* x;
  double* g;           // SA^T r (solve_b input); r12 on the semi-normal path
  int64_t* bad_col;
  double* bad_val;
  const int* sel;      // semi-normal solve on R1 (cqr_pick_kernel): always refined
};

constexpr int CQ_RS_GROUPS = 16;               // column groups of the GEMV kernels
constexpr int CQ_SOLVE_ROWS = 512;             // one thread per row (n <= 511)
constexpr int CQ_SOLVE_NT = CQ_SOLVE_ROWS + 32;  // + the diagonal-block warp

__device__ __forceinline__ double cq_rt(const double* Rt, int64_t i, int64_t j) {
  return Rt[cq_tile((int)(i >> 5), (int)(j >> 5)) * 1024 + (j & 31) * 32 + (i & 31)];
}

// y <- R[:n,:n]^{-1} y, one CTA, y in shared memory.  Diagonal blocks from
// the bottom: x_b = Rinv_bb y_b (the extra warp), then every row above
// subtracts R[i, block b] x_b.  The block's R values (thread = row) and
// Rinv_bb (extra warp) are loaded one block ahead, so only the products and
// two barriers per block stay on the dependent chain.
__device__ __forceinline__ void cq_bs_fetch(const double* Rt, const double* Rinv, int b,
                                            double (&c)[32]) {
  const int tid = threadIdx.x;
  const int64_t lo = (int64_t)b * 32;
  if (tid < lo && tid < CQ_SOLVE_ROWS) {
    const double* rc = Rt + cq_tile(tid >> 5, b) * 1024 + (tid & 31);
#pragma unroll
    for (int j = 0; j < 32; ++j) c[j] = __ldg(rc + j * 32);
  } else if (tid >= CQ_SOLVE_ROWS) {  // Rinv_bb row `lane`
    const double* rb = Rinv + (int64_t)b * 1024 + (tid & 31);
#pragma unroll
    for (int j = 0; j < 32; ++j) c[j] = __ldg(rb + j * 32);
  }
}

__device__ void cq_backsolve(const double* Rt, const double* Rinv, int64_t n, double* ys,
                             double* xb) {
  const int tid = threadIdx.x, lane = tid & 31;
  const int nbn = (int)((n + 31) / 32);
  double c[32];
  cq_bs_fetch(Rt, Rinv, nbn - 1, c);
  for (int b = nbn - 1; b >= 0; --b) {
    const int64_t lo = (int64_t)b * 32;
    const int w = (int)min((int64_t)32, n - lo);
    if (tid >= CQ_SOLVE_ROWS) {
      double a0 = 0.0, a1 = 0.0;
#pragma unroll
      for (int j = 0; j < 32; j += 2) {
        a0 = fma(c[j], j < w ? ys[lo + j] : 0.0, a0);
        a1 = fma(c[j + 1], j + 1 < w ? ys[lo + j + 1] : 0.0, a1);
      }
      const double xv = lane < w ? a0 + a1 : 0.0;
      xb[lane] = xv;
      if (lane < w) ys[lo + lane] = xv;
    }
    __syncthreads();
    double t0 = 0.0, t1 = 0.0;
    const bool mine = tid < lo && tid < CQ_SOLVE_ROWS;
    if (mine) {
#pragma unroll
      for (int j = 0; j < 32; j += 2) {
        t0 = fma(c[j], xb[j], t0);
        t1 = fma(c[j + 1], xb[j + 1], t1);
      }
    }
    // rows 512 .. 1023 (n > 512): a second row per thread, loaded at use
    // (rows past 1023 lie in the last block only, so no update reaches them)
    const int64_t i2 = tid + CQ_SOLVE_ROWS;
    double s2 = 0.0;
    if (tid < CQ_SOLVE_ROWS && i2 < lo) {
      const double* rc = Rt + cq_tile((int)(i2 >> 5), b) * 1024 + (i2 & 31);
      double u0 = 0.0, u1 = 0.0;
#pragma unroll
      for (int j = 0; j < 32; j += 2) {
        u0 = fma(__ldg(rc + j * 32), xb[j], u0);
        u1 = fma(__ldg(rc + (j + 1) * 32), xb[j + 1], u1);
      }
      s2 = u0 + u1;
    }
    if (b > 0) cq_bs_fetch(Rt, Rinv, b - 1, c);
    if (mine) ys[tid] -= t0 + t1;
    if (tid < CQ_SOLVE_ROWS && i2 < lo) ys[i2] -= s2;
    __syncthreads();
  }
}

// y <- R[:n,:n]^{-T} y (forward substitution with R^T), same storage: row i
// below block b subtracts sum_j R[lo + j][i] z_j (its 32 contiguous values
// of tile (b, i>>5)); the extra warp applies (Rinv_bb)^T.
__device__ __forceinline__ void cq_fs_fetch(const double* Rt, const double* Rinv, int b,
                                            int64_t n, double (&c)[32]) {
  const int tid = threadIdx.x;
  const double2* src = nullptr;
  if (tid >= (int64_t)b * 32 + 32 && tid < n && tid < CQ_SOLVE_ROWS)
    src = reinterpret_cast<const double2*>(Rt + cq_tile(b, tid >> 5) * 1024 + (tid & 31) * 32);
  else if (tid >= CQ_SOLVE_ROWS)  // (Rinv^T)[lane][j] = Rinv[j][lane]
    src = reinterpret_cast<const double2*>(Rinv + (int64_t)b * 1024 + (tid & 31) * 32);
  if (src) {
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const double2 v = __ldg(src + j);
      c[2 * j] = v.x;
      c[2 * j + 1] = v.y;
    }
  }
}

__device__ void cq_fwdsolve_t(const double* Rt, const double* Rinv, int64_t n, double* ys,
                              double* zb) {
  const int tid = threadIdx.x, lane = tid & 31;
  const int nbn = (int)((n + 31) / 32);
  double c[32];
  cq_fs_fetch(Rt, Rinv, 0, n, c);
  for (int b = 0; b < nbn; ++b) {
    const int64_t lo = (int64_t)b * 32;
    const int w = (int)min((int64_t)32, n - lo);
    if (tid >= CQ_SOLVE_ROWS) {
      double a0 = 0.0, a1 = 0.0;
#pragma unroll
      for (int j = 0; j < 32; j += 2) {
        a0 = fma(c[j], j < w ? ys[lo + j] : 0.0, a0);
        a1 = fma(c[j + 1], j + 1 < w ? ys[lo + j + 1] : 0.0, a1);
      }
      const double zv = lane < w ? a0 + a1 : 0.0;
      zb[lane] = zv;
      if (lane < w) ys[lo + lane] = zv;
    }
    __syncthreads();
    const bool mine = tid >= lo + 32 && tid < n && tid < CQ_SOLVE_ROWS;
    double t0 = 0.0, t1 = 0.0;
    if (mine) {
#pragma unroll
      for (int j = 0; j < 32; j += 2) {
        t0 = fma(c[j], zb[j], t0);
        t1 = fma(c[j + 1], zb[j + 1], t1);
      }
    }
    // rows 512 .. 1023 and 1024 .. 1055 (n > 512, n > 1024): a second and a
    // third row per thread, loaded at use
    const int64_t i2 = tid + CQ_SOLVE_ROWS, i3 = tid + 2 * CQ_SOLVE_ROWS;
    const bool mine2 = tid < CQ_SOLVE_ROWS && i2 >= lo + 32 && i2 < n;
    const bool mine3 = tid < CQ_SOLVE_ROWS && i3 >= lo + 32 && i3 < n;
    auto row_dot = [&](int64_t i) {
      const double2* rc = reinterpret_cast<const double2*>(Rt + cq_tile(b, (int)(i >> 5)) * 1024 + (i & 31) * 32);
      double u0 = 0.0, u1 = 0.0;
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const double2 v = __ldg(rc + j);
        u0 = fma(v.x, zb[2 * j], u0);
        u1 = fma(v.y, zb[2 * j + 1], u1);
      }
      return u0 + u1;
    };
    const double s2 = mine2 ? row_dot(i2) : 0.0;
    const double s3 = mine3 ? row_dot(i3) : 0.0;
    if (b + 1 < nbn) cq_fs_fetch(Rt, Rinv, b + 1, n, c);
    if (mine) ys[tid] -= t0 + t1;
    if (mine2) ys[i2] -= s2;
    if (mine3) ys[i3] -= s3;
    __syncthreads();
  }
}

// Rank check (diag R vs 1e-14 ||SA||_F), y = R[:n, n], x = R[:n,:n]^{-1} y.
__global__ void __launch_bounds__(CQ_SOLVE_NT) cqr_solve_a_kernel(const SolveParams p) {
  __shared__ double ys[CQ_MAXNB_BIG * 32];
  __shared__ double xb[32];
  __shared__ double red[CQ_SOLVE_NT / 32];
  __shared__ unsigned long long first_bad;
  pdl_enter();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t n = p.n;
  double s = 0.0;
  double dmax = 0.0, dmin = INFINITY;
  if (tid == 0) first_bad = ~0ull;
  __syncthreads();
  for (int64_t i = tid; i < n; i += CQ_SOLVE_NT) {  // rows beyond 511 in a second pass
    if (p.fro2 == nullptr) s += cq_rt(p.G1t, i, i);
    const double dgi = cq_rt(p.Rt, i, i);
    ys[i] = cq_rt(p.Rt, i, n);
    dmax = fmax(dmax, dgi);
    dmin = fmin(dmin, dgi);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) red[warp] = s;
  __syncthreads();
  double fro2 = 0.0;
  if (p.fro2 != nullptr) {
    fro2 = *p.fro2;
  } else {
#pragma unroll
    for (int w = 0; w < CQ_SOLVE_NT / 32; ++w) fro2 += red[w];
  }
  const double fro = sqrt(fro2);
  for (int64_t i = tid; i < n; i += CQ_SOLVE_NT)
    if (!(fro > 0.0) || !(cq_rt(p.Rt, i, i) >= CQ_RANK_TOL * fro))
      atomicMin(&first_bad, (unsigned long long)i);
  // diagonal extremes (all entries positive by construction)
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    dmax = fmax(dmax, __shfl_xor_sync(0xffffffffu, dmax, o));
    dmin = fmin(dmin, __shfl_xor_sync(0xffffffffu, dmin, o));
  }
  __shared__ double ext[2][CQ_SOLVE_NT / 32];
  if (lane == 0) {
    ext[0][warp] = dmax;
    ext[1][warp] = dmin;
  }
  __syncthreads();
  if (tid == 0) {
    double mx = 0.0, mn = INFINITY;
    for (int w = 0; w < CQ_SOLVE_NT / 32; ++w) {
      mx = fmax(mx, ext[0][w]);
      mn = fmin(mn, ext[1][w]);
    }
    const bool broke = *p.flag != 0 || !(mx <= CQ_DIAG_RATIO_MAX * mn);
    *p.refine = (mx <= CQ_REFINE_RATIO * mn && !cq_stopped(p.sel)) ? 0 : 1;
    const long long fb = first_bad == ~0ull ? -1 : (long long)first_bad;
    *p.bad_col = broke ? -2 : fb;
    *p.bad_val = (!broke && fb >= 0) ? cq_rt(p.Rt, fb, fb) : 0.0;
  }
  if (cq_stopped(p.sel)) {  // semi-normal path: x = R^{-1} r12 by the explicit inverse
    for (int64_t i = tid; i < n; i += CQ_SOLVE_NT) p.g[i] = ys[i];
    return;
  }
  cq_backsolve(p.Rt, p.Rinv, n, ys, xb);
  for (int64_t i = tid; i < n; i += CQ_SOLVE_NT) p.x[i] = ys[i];
}

// x += R^{-1} R^{-T} g (CholeskyQR2 path; the semi-normal path applies the
// explicit inverse instead: cqr_trmv_t_kernel, cqr_trmv_kernel).
__global__ void __launch_bounds__(CQ_SOLVE_NT) cqr_solve_b_kernel(const SolveParams p) {
  pdl_enter();
  if (*p.refine == 0 || cq_stopped(p.sel)) return;
  __shared__ double ys[CQ_MAXNB_BIG * 32];
  __shared__ double xb[32];
  const int64_t n = p.n;
  const int tid = threadIdx.x;
  for (int64_t i = tid; i < n; i += CQ_SOLVE_NT) ys[i] = p.g[i];
  __syncthreads();
  cq_fwdsolve_t(p.Rt, p.Rinv, n, ys, xb);
  cq_backsolve(p.Rt, p.Rinv, n, ys, xb);
  for (int64_t i = tid; i < n; i += CQ_SOLVE_NT) p.x[i] += ys[i];
}

// Semi-normal path, with Ri = R^{-1} (upper, column-major, ld even, only
// j >= i ever read: the rest of the buffer is stale).
// out = Ri[:n, :n] y: 64 rows per CTA (a row pair per lane) x 16 column groups
// over the columns right of the block's first row, folded in fixed order.
// Finishing form (xacc != nullptr): x += out instead, and the correction
// must have contracted (||dx|| <= 1e-6 ||x||, kappa^2 u well below one) --
// per-CTA sums, the last CTA folds them in CTA order -- else the solve is
// handed to the Householder factorisation (bad_col = -2).
struct TrmvFinish {
  double* xacc;
  int64_t* bad_col;
  unsigned* ticket;  // zero on entry, left zero
  double* part;      // [2 * CTAs]
};

__global__ void __launch_bounds__(CQ_RS_GROUPS * 32) cqr_trmv_kernel(const double* Ri, int64_t ld,
                                                                   int64_t n, const double* y,
                                                                   double* out, const int* need,
                                                                   const TrmvFinish fin) {
  extern __shared__ double ysm[];  // n
  __shared__ double part[CQ_RS_GROUPS][64];
  __shared__ double ab[2][2];
  __shared__ int is_last;
  pdl_enter();
  if (*need == 0) return;
  for (int64_t c = threadIdx.x; c < n; c += CQ_RS_GROUPS * 32) ysm[c] = y[c];
  __syncthreads();
  const int lane = threadIdx.x & 31, grp = threadIdx.x >> 5;
  const int64_t cb = (int64_t)blockIdx.x * 64, i0 = cb + 2 * lane;
  const int64_t c0 = cb + (n - cb) * grp / CQ_RS_GROUPS, c1 = cb + (n - cb) * (grp + 1) / CQ_RS_GROUPS;
  double s0 = 0.0, s1 = 0.0, u0 = 0.0, u1 = 0.0;
  int64_t c = c0;
  for (; c + 8 <= c1; c += 8) {  // eight column loads in flight
    double2 v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = __ldcg(reinterpret_cast<const double2*>(Ri + (c + k) * ld + i0));
#pragma unroll
    for (int k = 0; k < 8; k += 2) {
      s0 = fma(c + k >= i0 ? v[k].x : 0.0, ysm[c + k], s0);
      s1 = fma(c + k >= i0 + 1 ? v[k].y : 0.0, ysm[c + k], s1);
      u0 = fma(c + k + 1 >= i0 ? v[k + 1].x : 0.0, ysm[c + k + 1], u0);
      u1 = fma(c + k + 1 >= i0 + 1 ? v[k + 1].y : 0.0, ysm[c + k + 1], u1);
    }
  }
  for (; c < c1; ++c) {
    const double2 v = __ldcg(reinterpret_cast<const double2*>(Ri + c * ld + i0));
    s0 = fma(c >= i0 ? v.x : 0.0, ysm[c], s0);
    s1 = fma(c >= i0 + 1 ? v.y : 0.0, ysm[c], s1);
  }
  part[grp][2 * lane] = s0 + u0;
  part[grp][2 * lane + 1] = s1 + u1;
  __syncthreads();
  if (threadIdx.x < 64) {
    const int64_t i = cb + threadIdx.x;
    double t = 0.0;
#pragma unroll
    for (int g2 = 0; g2 < CQ_RS_GROUPS; ++g2) t += part[g2][threadIdx.x];
    if (fin.xacc == nullptr) {
      if (i < n) out[i] = t;
    } else {
      double a = 0.0, b = 0.0;
      if (i < n) {
        const double xi = fin.xacc[i] + t;
        fin.xacc[i] = xi;
        a = t * t;
        b = xi * xi;
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        a += __shfl_xor_sync(0xffffffffu, a, o);
        b += __shfl_xor_sync(0xffffffffu, b, o);
      }
      if (lane == 0) {
        ab[threadIdx.x >> 5][0] = a;
        ab[threadIdx.x >> 5][1] = b;
      }
    }
  }
  if (fin.xacc == nullptr) return;
  __syncthreads();
  if (threadIdx.x == 0) {
    fin.part[2 * blockIdx.x] = ab[0][0] + ab[1][0];
    fin.part[2 * blockIdx.x + 1] = ab[0][1] + ab[1][1];
    __threadfence();
    is_last = atomicAdd(fin.ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (is_last && threadIdx.x == 0) {
    __threadfence();
    double a = 0.0, b = 0.0;
    for (unsigned q = 0; q < gridDim.x; ++q) {
      a += __ldcg(fin.part + 2 * q);
      b += __ldcg(fin.part + 2 * q + 1);
    }
    if (!(a <= 1e-12 * b) && *fin.bad_col == -1) *fin.bad_col = -2;
    *fin.ticket = 0u;
  }
}

// out = Ri[:n, :n]^T y: one warp per column j (rows 0..j, a row pair per lane;
// y 16-byte aligned with one readable entry past n - 1).
__global__ void __launch_bounds__(256) cqr_trmv_t_kernel(const double* Ri, int64_t ld, int64_t n,
                                                         const double* y, double* out,
                                                         const int* need) {
  pdl_enter();
  if (*need == 0) return;
  const int lane = threadIdx.x & 31;
  const int64_t j = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  if (j >= n) return;
  const double* col = Ri + j * ld;
  double t0 = 0.0, t1 = 0.0;
  int64_t i = 2 * lane;
  for (; i + 3 * 64 <= j; i += 4 * 64) {  // four row pairs in flight, all within rows <= j
    double2 v[4], w[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      v[k] = __ldcg(reinterpret_cast<const double2*>(col + i + k * 64));
      w[k] = __ldcg(reinterpret_cast<const double2*>(y + i + k * 64));
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      t0 = fma(v[k].x, w[k].x, t0);
      t1 = (i + k * 64 + 1 <= j) ? fma(v[k].y, w[k].y, t1) : t1;
    }
  }
  for (; i <= j; i += 64) {
    const double2 v = __ldcg(reinterpret_cast<const double2*>(col + i));
    const double2 w = __ldcg(reinterpret_cast<const double2*>(y + i));
    t0 = fma(v.x, w.x, t0);
    if (i + 1 <= j) t1 = fma(v.y, w.y, t1);
  }
  double t = t0 + t1;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
  if (lane == 0) out[j] = t;
}

// r = b - A x: 64 rows per CTA (16-byte loads, a row pair per lane) x 16
// column groups (one warp each, eight column loads in flight), the 16
// partials of a row folded in fixed order.
template <bool VEC>
__global__ void __launch_bounds__(CQ_RS_GROUPS * 32) cqr_resid_kernel(const double* A, int64_t lda,
                                                                    const double* b, int64_t d,
                                                                    int64_t n, const double* x,
                                                                    double* r, const int* refine) {
  extern __shared__ double xs[];  // n
  __shared__ double part[CQ_RS_GROUPS][64];
  pdl_enter();
  if (*refine == 0) return;
  for (int64_t c = threadIdx.x; c < n; c += CQ_RS_GROUPS * 32) xs[c] = x[c];
  __syncthreads();
  const int lane = threadIdx.x & 31, grp = threadIdx.x >> 5;
  const int64_t i0 = (int64_t)blockIdx.x * 64 + 2 * lane;
  const int64_t c0 = n * grp / CQ_RS_GROUPS, c1 = n * (grp + 1) / CQ_RS_GROUPS;
  double s0 = 0.0, s1 = 0.0, u0 = 0.0, u1 = 0.0;
  if (VEC && i0 + 1 < d) {
    int64_t c = c0;
    for (; c + 8 <= c1; c += 8) {
      double2 v[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) v[k] = __ldcs(reinterpret_cast<const double2*>(A + (c + k) * lda + i0));
#pragma unroll
      for (int k = 0; k < 8; k += 2) {
        s0 = fma(v[k].x, xs[c + k], s0);
        s1 = fma(v[k].y, xs[c + k], s1);
        u0 = fma(v[k + 1].x, xs[c + k + 1], u0);
        u1 = fma(v[k + 1].y, xs[c + k + 1], u1);
      }
    }
    for (; c < c1; ++c) {
      const double2 v = __ldcs(reinterpret_cast<const double2*>(A + c * lda + i0));
      s0 = fma(v.x, xs[c], s0);
      s1 = fma(v.y, xs[c], s1);
    }
  } else {
    for (int64_t c = c0; c < c1; ++c) {
      if (i0 < d) s0 = fma(A[c * lda + i0], xs[c], s0);
      if (i0 + 1 < d) s1 = fma(A[c * lda + i0 + 1], xs[c], s1);
    }
  }
  part[grp][2 * lane] = s0 + u0;
  part[grp][2 * lane + 1] = s1 + u1;
  __syncthreads();
  if (threadIdx.x < 64) {
    const int64_t i = (int64_t)blockIdx.x * 64 + threadIdx.x;
    double t = 0.0;
#pragma unroll
    for (int g2 = 0; g2 < CQ_RS_GROUPS; ++g2) t += part[g2][threadIdx.x];
    if (i < d) r[i] = b[i] - t;
  }
}

// g = A^T r: two warps per column (one per half of the rows: 16 warps per
// CTA for the loads in flight), 16-byte loads, eight in flight; fixed
// shuffle tree, halves added in order.
template <bool VEC>
__global__ void __launch_bounds__(512) cqr_gemv_t_kernel(const double* A, int64_t lda, int64_t d,
                                                         int64_t n, const double* r, double* g,
                                                         const int* refine) {
  __shared__ double half1[8];
  pdl_enter();
  if (*refine == 0) return;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, hf = w >> 3;
  const int64_t c = (int64_t)blockIdx.x * 8 + (w & 7);
  const int64_t dh = (d / 2 + 63) / 64 * 64;  // first half: rows [0, dh), a multiple of 64
  const int64_t lo = hf ? dh : 0, hi = hf ? d : min(dh, d);
  double t = 0.0;
  if (c < n) {
    const double* col = A + c * lda;
    double t0 = 0.0, t1 = 0.0, t2 = 0.0, t3 = 0.0;
    int64_t i = lo + 2 * lane;
    if (VEC) {
      for (; i + 7 * 64 + 1 < hi; i += 8 * 64) {
        double2 v[8], u[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          v[k] = __ldcs(reinterpret_cast<const double2*>(col + i + k * 64));
          u[k] = __ldcg(reinterpret_cast<const double2*>(r + i + k * 64));
        }
#pragma unroll
        for (int k = 0; k < 8; k += 2) {
          t0 = fma(v[k].x, u[k].x, t0);
          t1 = fma(v[k].y, u[k].y, t1);
          t2 = fma(v[k + 1].x, u[k + 1].x, t2);
          t3 = fma(v[k + 1].y, u[k + 1].y, t3);
        }
      }
    }
    for (; i < hi; i += 64) {
      t0 = fma(col[i], r[i], t0);
      if (i + 1 < hi) t1 = fma(col[i + 1], r[i + 1], t1);
    }
    t = (t0 + t1) + (t2 + t3);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
  }
  if (hf && lane == 0) half1[w & 7] = t;
  __syncthreads();
  if (!hf && lane == 0 && c < n) g[c] = t + half1[w & 7];
}

}  // namespace skl

using namespace skl;

namespace {

struct CqWork {
  size_t bytes = 0;
  size_t oG1, oG2, oPart, oCnt, oR1, oR2, oI1, oI2, oQ, oR, oG, oBad, oBadV, oRt, oRi, oFro, oRef, oRf, oRfi, oY;
};

CqWork cq_layout(int64_t d, int64_t N, int nb, int nslots) {
  CqWork w;
  size_t off = 0;
  auto take = [&](size_t b) {
    const size_t o = off;
    off += (b + 255) / 256 * 256;
    return o;
  };
  const size_t nt = (size_t)nb * (nb + 1) / 2;
  const int64_t ldq = (d + 1) / 2 * 2;
  // G1, R1, I1, Rf, Rfi: two variants (shifted, unshifted) back to back
  w.oG1 = take(2 * nt * 1024 * 8);
  w.oG2 = take(nt * 1024 * 8);
  w.oPart = take((size_t)nslots * 1024 * 8);
  w.oCnt = take(nt * 4 + 16);  // tile counters, then the flags (one memset)
  w.oR1 = take(2 * nt * 1024 * 8);
  w.oR2 = take(nt * 1024 * 8);
  w.oI1 = take(2 * (size_t)nb * 1024 * 8);
  w.oI2 = take((size_t)nb * 1024 * 8);
  // Q1; on the semi-normal path R^{-1} (ld nb * 32; GEMV row pairs read up to 64 past it)
  w.oQ = take(((size_t)std::max<int64_t>(ldq, (int64_t)nb * 32) * N + 64) * 8);
  w.oR = take((size_t)d * 8);
  w.oG = take((size_t)N * 8);
  w.oBad = take(8);
  w.oBadV = take(8);
  w.oRt = take(nt * 1024 * 8);
  w.oRi = take((size_t)nb * 1024 * 8);
  w.oFro = take(8);
  w.oRef = take(4);
  w.oRf = take(2 * nt * 1024 * 8);
  w.oRfi = take(2 * (size_t)nb * 1024 * 8);
  w.oY = take((size_t)N * 8);
  w.bytes = off;
  return w;
}

// Stream-K geometry of the Gram: P = min(2 x SMs, units) CTAs, partial
// slots for the most tiles any CTA's unit range touches.
struct CqGramGeom {
  uint32_t nchunk, U, P;
  int SEG;
};
CqGramGeom cq_gram_geom(int64_t d, int nt) {
  CqGramGeom g;
  g.nchunk = (uint32_t)((d + 15) / 16);
  g.U = (uint32_t)nt * g.nchunk;
  g.P = (uint32_t)std::min<int64_t>(2 * sm_count_cached(), g.U);
  int seg = 1;
  for (uint32_t c = 0; c < g.P; ++c) {
    const uint32_t lo = (uint32_t)((uint64_t)g.U * c / g.P), hi = (uint32_t)((uint64_t)g.U * (c + 1) / g.P);
    seg = std::max(seg, (int)((hi - 1) / g.nchunk - lo / g.nchunk + 1));
  }
  g.SEG = seg;
  return g;
}

struct GramOut {
  double* Gt2 = nullptr;
  const int* skip = nullptr;
};

int cq_gram(const CqCols& X, int64_t N, int nb, double* part, double* Gt, unsigned* cnt,
            bool pdl, cudaStream_t st, const GramOut& go = GramOut()) {
  const int nt = nb * (nb + 1) / 2;
  const CqGramGeom gg = cq_gram_geom(X.d, nt);
  SKL_REQUIRE((uint64_t)gg.U * (gg.P + 1) < (1ULL << 32), SKL_ERR_SPEC, "cqr_gram: %lld rows too many",
              (long long)X.d);
  const bool vec = ((uintptr_t)X.A % 16 == 0) && (X.lda % 2 == 0) &&
                   (X.b == nullptr || (uintptr_t)X.b % 16 == 0);
  GramParams gp{X, N, gg.nchunk, gg.U, gg.P, gg.SEG, part, Gt, cnt, go.Gt2, go.skip};
  if (vec)
    SKL_CUDA(launch_k(cqr_gram_kernel<true>, dim3(gg.P), dim3(128), 0, st, pdl, gp));
  else
    SKL_CUDA(launch_k(cqr_gram_kernel<false>, dim3(gg.P), dim3(128), 0, st, pdl, gp));
  return SKL_OK;
}

// One Cholesky chain: nv = 2 factors the unshifted variant beside the shifted
// one (its buffers at + vs_*, its flag at flag + 1); skip: the chain's
// kernels return at once when cq_stopped.
struct CqChain {
  double* Gt;
  double* Rt;
  double* Rinv;
  int* flag;
  double* Rf;
  double* Rfi;
  int nv = 1;
  int64_t vs_g = 0, vs_r = 0, vs_i = 0;
  const int* skip = nullptr;
};

int cq_chol(const CqChain& ch, int nb, int64_t N, double shift_coef, bool pdl, cudaStream_t st,
            int to = 0) {
  static std::once_flag attr_set[64];
  const size_t smem_max = ((size_t)CQ_MAXNB * CQ_TILE + 32) * sizeof(double);
  const int arc = once_per_device(attr_set, [&]() -> int {
    SKL_CUDA(cudaFuncSetAttribute(cqr_chol_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    SKL_CUDA(cudaFuncSetAttribute(cqr_chol_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)smem_max));
    return SKL_OK;
  });
  if (arc) return arc;
  CholParams cp{ch.Gt, nb, N, shift_coef, ch.Rt, ch.Rinv, ch.flag, to,
                ch.vs_g, ch.vs_r, ch.vs_i, ch.skip};
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)nb, (unsigned)ch.nv);
  cfg.blockDim = dim3(CQ_CHOL_NT);
  cfg.dynamicSmemBytes = ((size_t)nb * CQ_TILE + 32) * sizeof(double);
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = (unsigned)nb;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = (pdl && pdl_enabled()) ? 2 : 1;
  SKL_CUDA(cudaLaunchKernelEx(&cfg, cqr_chol_kernel, cp));
  return SKL_OK;
}

// Cholesky of the tile-layout Gram: one cluster factorisation for nb <= 16,
// else right-looking over 16-tile super-blocks (cluster kernel on the
// diagonal block, block-row solve, trailing SYRK).  `shift_coef` only on the
// single-cluster path (the blocked path shifts beforehand).
int cq_chol_any(const CqChain& ch, int nb, int64_t N, double shift_coef, bool pdl,
                cudaStream_t st) {
  if (nb <= CQ_MAXNB) return cq_chol(ch, nb, N, shift_coef, pdl, st);
  const dim3 v1(1, (unsigned)ch.nv);
  // equal super-blocks (33 tiles: 11 + 11 + 11, not 16 + 16 + 1): the
  // block-row solves' chains are one step per tile of their super-block
  static const int sb_env = env_int("SKL_CQR_SB", 0);  // A/B knob: fixed super-block size
  const int nsb = (nb + CQ_MAXNB - 1) / CQ_MAXNB;
  const int sb = sb_env > 0 ? std::min(sb_env, CQ_MAXNB) : (nb + nsb - 1) / nsb;
  for (int to = 0; to < nb; to += sb) {
    const int nbs = std::min(sb, nb - to);
    int rc = cq_chol(ch, nbs, N, 0.0, pdl, st, to);
    if (rc) return rc;
    const int rest = nb - to - nbs;
    if (rest == 0) break;
    // R(to.., J0..) = R11^{-T} G(to.., J0..): its transpose is the TRSM of
    // G(to.., J0..)^T by R11 (16 rows per CTA)
    const size_t tsm = (size_t)nbs * 32 * CQ_QLD * sizeof(double);
    SKL_CUDA(raise_smem_limit(cqr_trsm_df_kernel<true>, tsm));
    const FragParams fp{ch.Rt, ch.Rinv, ch.Rf, ch.Rfi, to, nbs, ch.vs_r, ch.vs_i, ch.skip, nullptr,
                        nullptr, 0};
    SKL_CUDA(launch_k(cqr_rfrag_kernel, dim3((unsigned)(nbs * (nbs + 1) / 2 + nbs), ch.nv),
                      dim3(256), 0, st, true, fp));
    const CqCols none{nullptr, 0, nullptr, 0, (int64_t)rest * 32};
    TrsmParams sp{none, (int64_t)nbs * 32, nbs, ch.Rt, ch.Rinv, nullptr, 0, ch.Rf, ch.Rfi,
                  ch.Gt, ch.Rt, to, to + nbs, ch.vs_g, ch.vs_r, ch.vs_i, ch.skip, 0, nullptr,
                  nullptr};
    SKL_CUDA(launch_k(cqr_trsm_df_kernel<true>, dim3((unsigned)(rest * 32 / CQ_TRSM_ROWS), ch.nv),
                      dim3(CQ_TRSM_NT), tsm, st, true, sp));
    TriParams tp{ch.Gt, ch.Rt, ch.Rinv, to, nbs, nb, ch.vs_g, ch.vs_r, ch.skip};
    SKL_CUDA(launch_k(cqr_syrk_kernel, dim3((unsigned)(rest * (rest + 1) / 2), ch.nv), dim3(256), 0,
                      st, true, tp));
  }
  (void)v1;
  return SKL_OK;
}

int cq_trsm(const CqCols& X, int64_t N, int nb, const CqChain& ch, int* pick, double* Q,
            int64_t ldq, bool pdl, cudaStream_t st) {
  const int* stop = pick != nullptr ? pick + 2 : nullptr;
  static std::once_flag attr_set[64];
  const size_t smem_max = (size_t)CQ_MAXNB_BIG * 32 * CQ_QLD * sizeof(double);
  const int arc = once_per_device(attr_set, [&]() -> int {
    SKL_CUDA(cudaFuncSetAttribute(cqr_trsm_df_kernel<false>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_max));
    return SKL_OK;
  });
  if (arc) return arc;
  // the pick, then R1 of the picked variant and its diagonal inverses in
  // fragment order (for this TRSM, or for R1u^{-1} on the semi-normal path)
  const FragParams fp{ch.Rt, ch.Rinv, ch.Rf, ch.Rfi, 0, nb, ch.vs_r, ch.vs_i, nullptr, nullptr,
                      pick, X.n};
  SKL_CUDA(launch_k(cqr_rfrag_kernel, dim3((unsigned)(nb * (nb + 1) / 2 + nb)), dim3(256), 0, st,
                    pdl, fp));
  TrsmParams tp{X, N, nb, ch.Rt, ch.Rinv, Q, ldq, ch.Rf, ch.Rfi, nullptr, nullptr, 0, 0,
                0, 0, 0, stop, 0, nullptr, nullptr};
  const unsigned grid = (unsigned)((X.d + CQ_TRSM_ROWS - 1) / CQ_TRSM_ROWS);
  SKL_CUDA(launch_k(cqr_trsm_df_kernel<false>, dim3(grid), dim3(CQ_TRSM_NT),
                    (size_t)nb * 32 * CQ_QLD * sizeof(double), st, pdl, tp));
  return SKL_OK;
}

}  // namespace

// Sizes the CholeskyQR path covers: N = n + 1 <= 1056 and at least one row
// more than N (a square augmented system is rank deficient by construction).
extern "C" int skl_cqr_supported(int64_t d, int64_t n) {
  const int64_t N = n + 1;
  return (n >= 1 && N <= 32 * CQ_MAXNB_BIG && d > N) ? 1 : 0;
}

// Enqueue the CholeskyQR2 solve; *bad_col (pinned host or device) receives
// -1, the first rank-deficient column, or -2 when a Cholesky pivot broke
// down (then the caller re-solves with skl_qr_solve).
extern "C" int skl_cqr_solve_async(const double* SA, int64_t ldsa, const double* Sb, int64_t d,
                                   int64_t n, double* x, int64_t* bad_col, double* bad_val,
                                   void* stream) {
  clear_error();
  cudaStream_t st = (cudaStream_t)stream;
  SKL_REQUIRE(SA && Sb && x && bad_col && bad_val && ldsa >= d, SKL_ERR_INVALID,
              "cqr_solve: bad arguments");
  SKL_REQUIRE(skl_cqr_supported(d, n), SKL_ERR_SPEC,
              "cqr_solve: %lld x %lld outside the CholeskyQR path (n + 1 <= 1056 < d)",
              (long long)d, (long long)n);
  const int64_t N = n + 1;
  const int nb = (int)((N + 31) / 32);
  const int nt = nb * (nb + 1) / 2;
  const CqGramGeom gg = cq_gram_geom(d, nt);
  const CqWork w = cq_layout(d, N, nb, gg.P * gg.SEG);
  const int64_t ldq = (d + 1) / 2 * 2;
  unsigned char* ws = nullptr;
  SKL_CUDA(malloc_async(&ws, w.bytes, st));
  auto P = [&](size_t o) { return (void*)(ws + o); };
  double* G1 = (double*)P(w.oG1);
  double* G2 = (double*)P(w.oG2);
  double* part = (double*)P(w.oPart);
  unsigned* cnt = (unsigned*)P(w.oCnt);
  double* R1 = (double*)P(w.oR1);
  double* R2 = (double*)P(w.oR2);
  double* I1 = (double*)P(w.oI1);
  double* I2 = (double*)P(w.oI2);
  double* Q = (double*)P(w.oQ);
  // flag of the chosen variant, flag of the unshifted variant, sel, ticket
  int* flag = (int*)P(w.oCnt) + nt;
  double* r = (double*)P(w.oR);
  double* g = (double*)P(w.oG);
  int rc = SKL_OK;
  do {
    cudaError_t e = cudaMemsetAsync(cnt, 0, (size_t)nt * 4 + 16, st);
    if (e != cudaSuccess) {
      set_error("cqr_solve: %s", cudaGetErrorString(e));
      rc = SKL_ERR_CUDA;
      break;
    }
    const CqCols M{SA, ldsa, Sb, n, d};
    const CqCols Q1{Q, ldq, nullptr, N, d};
    const double u = 0.5 * 2.220446049250313e-16;
    const double shift = 11.0 * ((double)d * N + (double)N * (N + 1)) * u;
    const bool big = nb > CQ_MAXNB;
    double* fro2 = (double*)P(w.oFro);
    // the unshifted variant is factored beside the shifted one (SKL_CQR_SINGLE=1:
    // shifted only, A/B knob); when it is picked (well-conditioned SA) the
    // CholeskyQR2 kernels after the pick return at once and the solve is the
    // corrected semi-normal one on R1
    static const bool single = env_flag("SKL_CQR_SINGLE");
    const bool dual = !single;
    const int64_t vsT = (int64_t)nt * 1024, vsI = (int64_t)nb * 1024;
    GramOut g1;
    if (big && dual) g1.Gt2 = G1 + vsT;
    if ((rc = cq_gram(M, N, nb, part, G1, cnt, false, st, g1))) break;
    if (big) {  // shift once, before the super-block updates change the diagonal
      if ((e = launch_k(cqr_shift_kernel, dim3(1), dim3(1024), 0, st, true, G1, N, n, shift,
                        fro2)) != cudaSuccess) {
        set_error("cqr_solve: %s", cudaGetErrorString(e));
        rc = SKL_ERR_CUDA;
        break;
      }
    }
    double* Rf = (double*)P(w.oRf);
    double* Rfi = (double*)P(w.oRfi);
    CqChain c1{G1, R1, I1, flag, Rf, Rfi};
    c1.nv = dual ? 2 : 1;
    c1.vs_g = big ? vsT : 0;
    c1.vs_r = vsT;
    c1.vs_i = vsI;
    if ((rc = cq_chol_any(c1, nb, N, big ? 0.0 : shift, true, st))) break;
    int* sel = dual ? flag + 2 : nullptr;
    if ((rc = cq_trsm(M, N, nb, c1, dual ? flag : nullptr, Q, ldq, true, st))) break;
    GramOut g2;
    g2.skip = sel;
    if ((rc = cq_gram(Q1, N, nb, part, G2, cnt, true, st, g2))) break;
    CqChain c2{G2, R2, I2, flag, Rf, Rfi};
    c2.skip = sel;
    if ((rc = cq_chol_any(c2, nb, N, 0.0, true, st))) break;
    double* Rt = (double*)P(w.oRt);
    double* Ri = (double*)P(w.oRi);
    ProdParams pp{R1, R2, I1, I2, Rt, Ri, sel, vsT, vsI};
    int* refine = (int*)P(w.oRef);
    SolveParams sp{refine, big ? fro2 : nullptr, G1, Rt, Ri, n, flag, x, g, (int64_t*)P(w.oBad),
                   (double*)P(w.oBadV), sel};
    const size_t ysm = (size_t)N * sizeof(double);
#define CQ_LAUNCH(call)                                                          \
  if ((e = (call)) != cudaSuccess) {                                             \
    set_error("cqr_solve: kernel launch failed: %s", cudaGetErrorString(e));     \
    rc = SKL_ERR_CUDA;                                                           \
    break;                                                                       \
  }
    CQ_LAUNCH(launch_k(cqr_rprod_kernel, dim3((unsigned)nt), dim3(256), 0, st, true, pp));
    CQ_LAUNCH(launch_k(cqr_solve_a_kernel, dim3(1), dim3(CQ_SOLVE_NT), 0, st, true, sp));
    // semi-normal path: R^{-1} explicitly (the dataflow TRSM on the identity,
    // into the unused Q buffer), then x = R^{-1} r12 (r12 left in g by solve_a)
    const int64_t ldi = (int64_t)nb * 32;
    if (dual) {
      if (nb < 8) {
        const CqCols idc{nullptr, 0, nullptr, 0, N};
        TrsmParams ip{idc, N, nb, Rt, Ri, Q, ldi, Rf, Rfi, nullptr, nullptr, 0, 0, 0, 0, 0,
                      nullptr, 1, sel, nullptr};
        CQ_LAUNCH(launch_k(cqr_trsm_df_kernel<false>, dim3((unsigned)(2 * nb)), dim3(CQ_TRSM_NT),
                           (size_t)nb * 32 * CQ_QLD * sizeof(double), st, true, ip));
      } else {
        // 2 x 2 split R = [[A, B], [0, C]] at tile h: A^{-1}, C^{-1} and
        // W = B C^{-1} side by side in one launch, then -A^{-1} W
        const int h = nb / 2, hc = nb - h;
        const int64_t hr = (int64_t)h * 32;
        double* Wb = G2;  // free on this path
        TrsmBatch tb{};
        tb.p[0] = TrsmParams{CqCols{nullptr, 0, nullptr, 0, hr}, hr, h, Rt, Ri, Q, ldi, Rf, Rfi,
                             nullptr, nullptr, 0, 0, 0, 0, 0, nullptr, 1, sel, nullptr};
        tb.p[1] = TrsmParams{CqCols{nullptr, 0, nullptr, 0, N - hr}, N - hr, hc, Rt, Ri,
                             Q + hr * ldi + hr, ldi, Rf, Rfi, nullptr, nullptr, h, 0, 0, 0, 0,
                             nullptr, 1, sel, nullptr};
        tb.p[2] = TrsmParams{CqCols{nullptr, 0, nullptr, 0, hr}, N - hr, hc, Rt, Ri, Wb, hr, Rf,
                             Rfi, nullptr, nullptr, h, 0, 0, 0, 0, nullptr, 0, sel, Rt};
        tb.cta0[0] = 0;
        tb.cta0[1] = 2 * h;
        tb.cta0[2] = 2 * h + 2 * hc;
        tb.cta0[3] = 4 * h + 2 * hc;
        const size_t bsm = (size_t)hc * 32 * CQ_QLD * sizeof(double);
        if ((e = raise_smem_limit(cqr_trsm_df_batch_kernel, bsm)) != cudaSuccess) {
          set_error("cqr_solve: %s", cudaGetErrorString(e));
          rc = SKL_ERR_CUDA;
          break;
        }
        CQ_LAUNCH(launch_k(cqr_trsm_df_batch_kernel, dim3((unsigned)tb.cta0[3]), dim3(CQ_TRSM_NT),
                           bsm, st, true, tb));
        CQ_LAUNCH(launch_k(cqr_rinv_offdiag_kernel, dim3((unsigned)(h * hc)), dim3(256), 0, st, true,
                           Q, ldi, h, hc, N, (const double*)Wb, hr, (const int*)sel));
      }
      CQ_LAUNCH(launch_k(cqr_trmv_kernel, dim3((unsigned)((n + 63) / 64)), dim3(CQ_RS_GROUPS * 32),
                         (size_t)n * sizeof(double), st, true, (const double*)Q, ldi, n,
                         (const double*)g, x, (const int*)sel, TrmvFinish{}));
    }
    // corrected semi-normal step: r = Sb - SA x, g = SA^T r, x += R^{-1} R^{-T} g
    const bool vec = ((uintptr_t)SA % 16 == 0) && (ldsa % 2 == 0);
    CQ_LAUNCH(launch_k(vec ? cqr_resid_kernel<true> : cqr_resid_kernel<false>,
                       dim3((unsigned)((d + 63) / 64)), dim3(CQ_RS_GROUPS * 32), ysm, st, true, SA,
                       ldsa, Sb, d, n, (const double*)x, r, (const int*)refine));
    CQ_LAUNCH(launch_k(vec ? cqr_gemv_t_kernel<true> : cqr_gemv_t_kernel<false>,
                       dim3((unsigned)((n + 7) / 8)), dim3(512), 0, st, true, SA, ldsa, d, n,
                       (const double*)r, g, (const int*)refine));
    CQ_LAUNCH(launch_k(cqr_solve_b_kernel, dim3(1), dim3(CQ_SOLVE_NT), 0, st, true, sp));
    if (dual) {  // x += R^{-1} R^{-T} g, with the contraction check
      CQ_LAUNCH(launch_k(cqr_trmv_t_kernel, dim3((unsigned)((n + 7) / 8)), dim3(256), 0, st, true,
                         (const double*)Q, ldi, n, (const double*)g, r, (const int*)sel));
      const TrmvFinish fin{x, (int64_t*)P(w.oBad), (unsigned*)(flag + 3), (double*)P(w.oY)};
      CQ_LAUNCH(launch_k(cqr_trmv_kernel, dim3((unsigned)((n + 63) / 64)), dim3(CQ_RS_GROUPS * 32),
                         (size_t)n * sizeof(double), st, true, (const double*)Q, ldi, n,
                         (const double*)r, (double*)nullptr, (const int*)sel, fin));
    }
#undef CQ_LAUNCH
    e = cudaMemcpyAsync(bad_col, P(w.oBad), 8, cudaMemcpyDefault, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(bad_val, P(w.oBadV), 8, cudaMemcpyDefault, st);
    if (e != cudaSuccess) {
      set_error("cqr_solve: %s", cudaGetErrorString(e));
      rc = SKL_ERR_CUDA;
    }
  } while (0);
  cudaFreeAsync(ws, st);
  return rc;
}

#ifdef SKL_CQR_PROBE
// Copy the Cholesky probe timestamps ([2][16][72] ns) to host memory.
extern "C" int skl_cqr_probe_dump(long long* out) {
  cudaDeviceSynchronize();
  return cudaMemcpyFromSymbol(out, g_cqr_probe, sizeof(g_cqr_probe)) == cudaSuccess ? 0 : 7;
}
#endif
