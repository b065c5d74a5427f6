// Reduced solve on device: Householder QR of M = [SA | Sb] (d x (n+1)) and
// back substitution, with the reference's conventions
// (/root/reference/pkg/src/sketchls/linalg.py:166-192, 214-218;
// solvers.py:309):
//   * reflectors follow LAPACK dlarfg/dgeqr2 (beta = -sign(alpha)*||x||,
//     tau = (beta-alpha)/beta, v = x/(alpha-beta));
//   * diag(R) is normalised to be >= 0 (row sign flips of R and Q^T Sb,
//     which leave x unchanged);
//   * rank check |R[c,c]| < RANK_TOL * ||M||_F (RANK_TOL = 1e-14) reports
//     the first offending column;
//   * x = R^{-1} (Q^T Sb), the triangular solve in the column order of
//     LAPACK dtrsv ('U','N').
// Q^T Sb is obtained by applying the reflectors to the Sb column as the
// (n+1)-th trailing column; Q itself is only formed when requested
// (economy_qr), by backward accumulation of the reflectors into I.
//
// Execution: the blocked factorisation in skl_qr_blocked.cu (cluster panel
// + GEMM-shaped trailing updates) for n >= 64 when a panel fits a
// thread-block cluster (d <= 10880); otherwise this file's unblocked fallback: one
// persistent cooperative kernel, step k split across all CTAs (each owns
// trailing columns round-robin) with one grid barrier per step, the CTA that
// updates column k+1 publishing its norm for the next step.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>

#include "skl_common.h"
#include "skl_ptx.cuh"

namespace cg = cooperative_groups;

namespace skl {

constexpr int QR_NT = 256;
constexpr double RANK_TOL = 1e-14;

__device__ __forceinline__ double block_sum(double v, double* red) {
  // deterministic: fixed shuffle tree, then warp 0 folds the warp sums
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x < 32) {
    s = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (threadIdx.x == 0) red[32] = s;
  }
  __syncthreads();
  return red[32];
}

struct QrParams {
  double* M;        // d x (n+1), ld = d (working copy, destroyed)
  int64_t d, n;
  double* tau;      // n
  double* beta;     // n   (diag of R before sign normalisation)
  double* colinfo;  // 2*(n+1): alpha, xnorm of the current pivot column
};

// Norm of column j below row k (rows k+1..d-1) and alpha = M[k, j].
__device__ void publish_column(const QrParams& p, int64_t k, int64_t j, double* red) {
  const double* col = p.M + j * p.d;
  double s = 0.0;
  for (int64_t i = k + 1 + threadIdx.x; i < p.d; i += QR_NT) s += col[i] * col[i];
  s = block_sum(s, red);
  if (threadIdx.x == 0) {
    p.colinfo[2 * k] = col[k];
    p.colinfo[2 * k + 1] = sqrt(s);
  }
}

__global__ void __launch_bounds__(QR_NT) qr_householder_kernel(QrParams p) {
  cg::grid_group grid = cg::this_grid();
  __shared__ double red[33];
  const int64_t d = p.d, n = p.n;
  if (blockIdx.x == 0) publish_column(p, 0, 0, red);
  grid.sync();
  for (int64_t k = 0; k < n; ++k) {
    const double alpha = p.colinfo[2 * k];
    const double xnorm = p.colinfo[2 * k + 1];
    double tau, beta, scale;
    if (xnorm == 0.0) {
      tau = 0.0;
      beta = alpha;
      scale = 0.0;
    } else {
      beta = -copysign(hypot(alpha, xnorm), alpha);
      tau = (beta - alpha) / beta;
      scale = 1.0 / (alpha - beta);
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      p.tau[k] = tau;
      p.beta[k] = beta;
    }
    const double* vk = p.M + k * d;
    // trailing columns j = k+1 .. n (n is the Sb column)
    for (int64_t j = k + 1 + blockIdx.x; j <= n; j += gridDim.x) {
      double* cj = p.M + j * d;
      if (tau != 0.0) {
        double s = 0.0;
        for (int64_t i = k + 1 + threadIdx.x; i < d; i += QR_NT) s += (vk[i] * scale) * cj[i];
        s = block_sum(s, red);
        const double w = tau * (cj[k] + s);
        for (int64_t i = k + 1 + threadIdx.x; i < d; i += QR_NT) cj[i] -= (vk[i] * scale) * w;
        __syncthreads();
        if (threadIdx.x == 0) cj[k] -= w;
      }
      __syncthreads();
      if (j == k + 1 && k + 1 < n) publish_column(p, k + 1, j, red);
    }
    grid.sync();
  }
}

// Store v (scaled reflector, implicit unit head) below the diagonal so Q can
// be formed: v_i = M[i,k] / (alpha_k - beta_k).  alpha_k is lost after the
// step, recover it from beta and tau: alpha - beta = -beta*tau... (tau =
// (beta-alpha)/beta  =>  alpha - beta = -tau*beta).
__global__ void qr_scale_reflectors(double* M, int64_t d, int64_t n, const double* tau,
                                    const double* beta) {
  for (int64_t k = blockIdx.x; k < n; k += gridDim.x) {
    const double t = tau[k];
    const double scale = t != 0.0 ? 1.0 / (-t * beta[k]) : 0.0;
    for (int64_t i = k + 1 + threadIdx.x; i < d; i += blockDim.x) M[k * d + i] *= scale;
  }
}

// Rank check + R output with nonnegative diagonal, y = sign-fixed Q^T Sb.
// One CTA.  fro2 = ||SA||_F^2 computed beforehand.
__global__ void qr_finish_kernel(const double* M, int64_t d, int64_t n, const double* beta,
                                 const double* fro2, double* R, int64_t ldr, double* y,
                                 int64_t* bad_col, double* bad_val) {
  pdl_enter();
  __shared__ int64_t first_bad;
  if (threadIdx.x == 0) first_bad = -1;
  __syncthreads();
  const double fro = sqrt(*fro2);
  for (int64_t c = threadIdx.x; c < n; c += blockDim.x) {
    const double dg = fabs(beta[c]);
    const bool bad = fro > 0.0 ? (dg < RANK_TOL * fro) : true;
    if (bad) atomicMin((unsigned long long*)&first_bad, (unsigned long long)c);
  }
  // atomicMin on -1 (all ones) works as "no bad column yet"
  __syncthreads();
  if (threadIdx.x == 0) {
    *bad_col = first_bad == (int64_t)-1 ? -1 : first_bad;
    *bad_val = (first_bad >= 0 && fro > 0.0) ? fabs(beta[first_bad]) : 0.0;
  }
  for (int64_t r = threadIdx.x; r < n; r += blockDim.x) {
    const double sg = beta[r] < 0.0 ? -1.0 : 1.0;
    y[r] = sg * M[n * d + r];
    if (R) {
      for (int64_t c = 0; c < n; ++c) {
        double v = 0.0;
        if (c > r) v = sg * M[c * d + r];
        else if (c == r) v = sg * beta[r];
        R[c * ldr + r] = v;
      }
    }
  }
}

// Column-oriented back substitution (dtrsv 'U','N' order):
// for j = n-1..0: x_j = y_j / R_jj; y_i -= x_j * R_ij (i < j).
// R is read from the factored M (upper part) with the sign-normalised
// diagonal; one CTA, y in shared memory when it fits.
__global__ void __launch_bounds__(1024) qr_backsolve_kernel(const double* M, int64_t d, int64_t n,
                                                            const double* beta, const double* y_in,
                                                            double* x) {
  extern __shared__ double ys[];
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) ys[i] = y_in[i];
  __syncthreads();
  for (int64_t j = n - 1; j >= 0; --j) {
    const double sgj = beta[j] < 0.0 ? -1.0 : 1.0;
    const double xj = ys[j] / fabs(beta[j]);
    __syncthreads();
    if (threadIdx.x == 0) x[j] = xj;
    for (int64_t i = threadIdx.x; i < j; i += blockDim.x) {
      const double sgi = beta[i] < 0.0 ? -1.0 : 1.0;
      ys[i] -= xj * (sgi * M[j * d + i]);
    }
    (void)sgj;
    __syncthreads();
  }
}

// Blocked back substitution: 32 x 32 diagonal blocks from the bottom.  Warp
// 0 preloads the block (lane r holds row r of R in registers) and solves it
// with shuffles (x_j = y_j * (1 / R_jj) in dtrsv's column order); then every
// thread updates one row above the block with a 32-term dot product whose
// loads are all in flight together.  R = sign-normalised upper triangle of
// the factored M (ld ldm): R_ij = sign(beta_i) M_ij, R_ii = |beta_i|.
__global__ void __launch_bounds__(512) qr_backsolve_blocked_kernel(const double* M, int64_t ldm,
                                                                    int64_t n, const double* beta,
                                                                    const double* y_in, double* x) {
  pdl_enter();
  extern __shared__ double ys[];
  __shared__ double xb[32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
#ifdef SKL_QR_PROBE
  long long pb0 = 0, pb1 = 0, pb2 = 0, tq = clock64();
#endif
  for (int64_t i = tid; i < n; i += blockDim.x) ys[i] = y_in[i];
  __syncthreads();
  for (int64_t hi = n; hi > 0; hi -= 32) {
    const int64_t lo = hi > 32 ? hi - 32 : 0;
    const int w = (int)(hi - lo);
    if (warp == 0) {
      const int64_t row = lo + lane;
      const bool live = lane < w;
      const double sgr = (live && beta[row] < 0.0) ? -1.0 : 1.0;
      double Rr[32];
#pragma unroll
      for (int j = 0; j < 32; ++j)
        Rr[j] = (live && j > lane && j < w) ? sgr * M[(lo + j) * ldm + row] : 0.0;
      // reciprocals of the diagonal in parallel; the solve chain is then a
      // multiply, a shuffle and an FMA per column
      const double rinv = live ? 1.0 / fabs(beta[row]) : 1.0;
      double yr = live ? ys[row] : 0.0;
      double xr = 0.0;
#pragma unroll
      for (int j = 31; j >= 0; --j) {
        if (j < w) {
          if (lane == j) xr = yr * rinv;
          const double xj = __shfl_sync(0xffffffffu, xr, j);
          yr = fma(-xj, Rr[j], yr);  // Rr[j] = 0 unless lane < j
        }
      }
      if (live) {
        x[row] = xr;
        xb[lane] = xr;
      }
    }
#ifdef SKL_QR_PROBE
    if (tid == 0) { long long t = clock64(); pb0 += t - tq; tq = t; }
#endif
    __syncthreads();
#ifdef SKL_QR_PROBE
    if (tid == 0) { long long t = clock64(); pb1 += t - tq; tq = t; }
#endif
    for (int64_t i = tid; i < lo; i += blockDim.x) {
      const double sgi = beta[i] < 0.0 ? -1.0 : 1.0;
      // 16 loads in flight per group (one column stride apart)
      const double* mp = M + lo * ldm + i;
      double t0 = 0.0, t1 = 0.0;
#pragma unroll 1
      for (int g = 0; g < 32; g += 16) {
        double mv[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) mv[j] = (g + j) < w ? mp[(g + j) * ldm] : 0.0;
#pragma unroll
        for (int j = 0; j < 16; j += 2) {
          t0 = fma(mv[j], xb[g + j], t0);
          t1 = fma(mv[j + 1], xb[g + j + 1], t1);
        }
      }
      ys[i] -= sgi * (t0 + t1);
    }
    __syncthreads();
#ifdef SKL_QR_PROBE
    if (tid == 0) { long long t = clock64(); pb2 += t - tq; tq = t; }
#endif
  }
#ifdef SKL_QR_PROBE
  if (tid == 0) printf("backsolve n=%lld cycles: diag %lld sync %lld update %lld\n", (long long)n, pb0, pb1, pb2);
#endif
}

// Inverses of the 32 x 32 diagonal blocks of R, all blocks at once (one
// warp per block), so the back substitution's serial chain becomes one
// 32 x 32 product per block.  Block bi covers rows/columns [lo, hi) with
// hi = n - 32 bi, lo = max(0, hi - 32), counted from the bottom; a partial
// block is padded with the identity.  Lane j builds column j of the inverse
// (X[j][j] = 1 / R_jj, X[i][j] = -(sum_{k>i} R_ik X_kj) / R_ii upward) with
// the block's rows broadcast from shared memory; Rinv[bi] is stored
// row-major (32 x 32).
constexpr int TRI_WPB = 4;  // blocks (warps) per CTA
__global__ void __launch_bounds__(TRI_WPB * 32) qr_trinv_kernel(const double* M, int64_t ldm,
                                                                 int64_t n, const double* beta,
                                                                 double* Rinv) {
  pdl_enter();
  __shared__ double Rs[TRI_WPB][32][33];
  const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
  const int64_t bi = (int64_t)blockIdx.x * TRI_WPB + wl;
  const int64_t nb = (n + 31) / 32;
  if (bi >= nb) return;
  const int64_t hi = n - 32 * bi, lo = hi > 32 ? hi - 32 : 0;
  const int w = (int)(hi - lo);
  double (*R)[33] = Rs[wl];
  // lane = row i (coalesced along the column): R[i][j] for i < j (sign of
  // row i), diagonal |beta_i|, identity padding past w
  {
    const bool live = lane < w;
    const double bt = live ? beta[lo + lane] : 1.0;
    const double sg = bt < 0.0 ? -1.0 : 1.0;
    double v[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] = (live && j > lane && j < w) ? M[(lo + j) * ldm + lo + lane] : 0.0;
#pragma unroll
    for (int j = 0; j < 32; ++j) R[lane][j] = j == lane ? (live ? fabs(bt) : 1.0) : sg * v[j];
  }
  __syncwarp();
  // Upward over k; acc[i] collects sum_{k' > i, done} R[i][k'] X[k'] as soon
  // as each X[k'] is known, so a step's critical path is one multiply.
  const double rd = 1.0 / R[lane][lane];
  double acc[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) acc[i] = 0.0;
  double* out = Rinv + bi * 1024;
#pragma unroll
  for (int k = 31; k >= 0; --k) {
    const double rk = __shfl_sync(0xffffffffu, rd, k);
    const double xk = k == lane ? rk : (k < lane ? -acc[k] * rk : 0.0);
    out[k * 32 + lane] = xk;
#pragma unroll
    for (int i = 0; i < k; ++i) acc[i] = fma(R[i][k], xk, acc[i]);
  }
}

// Back substitution with the inverted diagonal blocks: per block (from the
// bottom) warp 0 forms x_b = Rinv_b y_b (lane i: row i of Rinv_b from shared
// memory, y_b broadcast), then every thread subtracts R[i, lo:hi] x_b from
// its rows above the block.  Nothing of R depends on x: the loads of the
// column block are issued before the product and the next Rinv block is
// staged by the other warps meanwhile, so per block the critical path is
// one 32-term product, two barriers and one 32-term dot product per row.
constexpr int BS_NT = 512;
__global__ void __launch_bounds__(BS_NT) qr_backsolve_inv_kernel(const double* M, int64_t ldm,
                                                                 int64_t n, const double* beta,
                                                                 const double* Rinv,
                                                                 const double* y_in, double* x) {
  pdl_enter();
  extern __shared__ double ys[];
  __shared__ double rv[2][32][33];
  __shared__ double xb[32];
  const int tid = threadIdx.x, lane = tid & 31;
  for (int64_t i = tid; i < n; i += BS_NT) ys[i] = y_in[i];
  const int64_t nb = (n + 31) / 32;
  for (int e = tid; e < 1024; e += BS_NT) rv[0][e >> 5][e & 31] = Rinv[e];
  __syncthreads();
  for (int64_t bi = 0; bi < nb; ++bi) {
    const int64_t hi = n - 32 * bi, lo = hi > 32 ? hi - 32 : 0;
    const int w = (int)(hi - lo);
    const int buf = (int)(bi & 1);
    // row tid's part of the column block (independent of x): in flight now
    double c[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) c[j] = (tid < lo && j < w) ? M[(lo + j) * ldm + tid] : 0.0;
    if (tid < 32) {
      double a0 = 0.0, a1 = 0.0;
#pragma unroll
      for (int j = 0; j < 32; j += 2) {
        const double y0 = j < w ? ys[lo + j] : 0.0, y1 = j + 1 < w ? ys[lo + j + 1] : 0.0;
        a0 = fma(rv[buf][lane][j], y0, a0);
        a1 = fma(rv[buf][lane][j + 1], y1, a1);
      }
      const double xr = a0 + a1;
      xb[lane] = xr;
      if (lane < w) x[lo + lane] = xr;
    } else if (bi + 1 < nb) {  // next block's inverse: async copies, waited at the block end
      for (int e = tid - 32; e < 1024; e += BS_NT - 32) {
        const uint32_t dst = (uint32_t)__cvta_generic_to_shared(&rv[buf ^ 1][e >> 5][e & 31]);
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst),
                     "l"(Rinv + (bi + 1) * 1024 + e)
                     : "memory");
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
    }
    __syncthreads();
    if (tid < lo) {
      double t0 = 0.0, t1 = 0.0;
#pragma unroll
      for (int j = 0; j < 32; j += 2) {
        t0 = fma(c[j], xb[j], t0);
        t1 = fma(c[j + 1], xb[j + 1], t1);
      }
      ys[tid] -= (beta[tid] < 0.0 ? -1.0 : 1.0) * (t0 + t1);
    }
    for (int64_t i = tid + BS_NT; i < lo; i += BS_NT) {  // n > BS_NT + 32: more rows
      double t0 = 0.0, t1 = 0.0;
#pragma unroll
      for (int j = 0; j < 32; j += 2) {
        const double m0 = j < w ? M[(lo + j) * ldm + i] : 0.0;
        const double m1 = j + 1 < w ? M[(lo + j + 1) * ldm + i] : 0.0;
        t0 = fma(m0, xb[j], t0);
        t1 = fma(m1, xb[j + 1], t1);
      }
      ys[i] -= (beta[i] < 0.0 ? -1.0 : 1.0) * (t0 + t1);
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncthreads();
  }
}

// Q = H_0 H_1 ... H_{n-1} [I; 0] by backward accumulation (dorg2r), one
// cooperative kernel, then column sign normalisation.
__global__ void __launch_bounds__(QR_NT) qr_form_q_kernel(const double* V, int64_t d, int64_t n,
                                                          const double* tau, const double* beta,
                                                          double* Q, int64_t ldq) {
  cg::grid_group grid = cg::this_grid();
  __shared__ double red[33];
  // Q = [I; 0]
  for (int64_t c = blockIdx.x; c < n; c += gridDim.x)
    for (int64_t i = threadIdx.x; i < d; i += QR_NT) Q[c * ldq + i] = (i == c) ? 1.0 : 0.0;
  grid.sync();
  for (int64_t k = n - 1; k >= 0; --k) {
    const double t = tau[k];
    if (t != 0.0) {
      const double* v = V + k * d;  // v_k = 1, v_i (i>k) stored
      for (int64_t j = k + blockIdx.x; j < n; j += gridDim.x) {
        double* qj = Q + j * ldq;
        double s = 0.0;
        for (int64_t i = k + 1 + threadIdx.x; i < d; i += QR_NT) s += v[i] * qj[i];
        s = block_sum(s, red);
        const double w = t * (qj[k] + s);
        for (int64_t i = k + 1 + threadIdx.x; i < d; i += QR_NT) qj[i] -= v[i] * w;
        __syncthreads();
        if (threadIdx.x == 0) qj[k] -= w;
        __syncthreads();
      }
    }
    grid.sync();
  }
  for (int64_t c = blockIdx.x; c < n; c += gridDim.x) {
    if (beta[c] < 0.0)
      for (int64_t i = threadIdx.x; i < d; i += QR_NT) Q[c * ldq + i] = -Q[c * ldq + i];
  }
}

__global__ void copy_aug_kernel(const double* SA, int64_t ldsa, const double* Sb, int64_t d,
                                int64_t n, double* M, int64_t ldm, double* fro_part) {
  // M[:, :n] = SA, M[:, n] = Sb; per-block partial of ||SA||_F^2
  __shared__ double red[33];
  double s = 0.0;
  const int64_t total = d * (n + 1);
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = idx / d, i = idx % d;
    double v;
    if (c < n) {
      v = SA[c * ldsa + i];
      s += v * v;
    } else {
      v = Sb ? Sb[i] : 0.0;
    }
    M[c * ldm + i] = v;
  }
  s = block_sum(s, red);
  if (threadIdx.x == 0) fro_part[blockIdx.x] = s;
}

__global__ void sum_parts_kernel(const double* part, int nparts, double* out) {
  pdl_enter();
  __shared__ double red[33];
  double s = 0.0;
  for (int i = threadIdx.x; i < nparts; i += blockDim.x) s += part[i];
  s = block_sum(s, red);
  if (threadIdx.x == 0) *out = s;
}

// Q workspace = [I; 0]
__global__ void eye_kernel(double* Q, int64_t ldq, int64_t d, int64_t n) {
  const int64_t total = d * n;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = idx / d, i = idx % d;
    Q[c * ldq + i] = (i == c) ? 1.0 : 0.0;
  }
}

// Q_out = Qw with columns of negative beta negated (diag(R) >= 0 convention)
__global__ void q_signfix_copy_kernel(const double* Qw, int64_t ldw, const double* beta, int64_t d,
                                      int64_t n, double* Q, int64_t ldq) {
  const int64_t total = d * n;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = idx / d, i = idx % d;
    const double v = Qw[c * ldw + i];
    Q[c * ldq + i] = beta[c] < 0.0 ? -v : v;
  }
}

bool qr_blocked_supported(int64_t d);
int qr_blocked_factor(double* M, int64_t ldm, int64_t d, int64_t n, double* tau, double* beta,
                      double* V, double* Tall, double* W, double* W2, double* part,
                      int64_t part_cap, double* W2b, double* partb, cudaStream_t st);
int qr_blocked_form_q(double* Q, int64_t ldq, int64_t d, int64_t n, const double* V, int64_t ldv,
                      const double* Tall, double* W, double* W2, double* part, int64_t part_cap,
                      cudaStream_t st);

}  // namespace skl

using namespace skl;

static int qr_solve_impl(const double* SA, int64_t ldsa, const double* Sb, int64_t d, int64_t n,
                         double* x, double* R, int64_t ldr, double* Q, int64_t ldq,
                         int64_t* bad_col, double* bad_val, void* stream, bool sync);

extern "C" int skl_qr_solve(const double* SA, int64_t ldsa, const double* Sb, int64_t d,
                            int64_t n, double* x, double* R, int64_t ldr, double* Q, int64_t ldq,
                            int64_t* bad_col, double* bad_val, void* stream) {
  clear_error();
  return qr_solve_impl(SA, ldsa, Sb, d, n, x, R, ldr, Q, ldq, bad_col, bad_val, stream, true);
}

extern "C" int skl_qr_solve_async(const double* SA, int64_t ldsa, const double* Sb, int64_t d,
                                  int64_t n, double* x, double* R, int64_t ldr, double* Q,
                                  int64_t ldq, int64_t* bad_col, double* bad_val, void* stream) {
  clear_error();
  return qr_solve_impl(SA, ldsa, Sb, d, n, x, R, ldr, Q, ldq, bad_col, bad_val, stream, false);
}

static int qr_solve_impl(const double* SA, int64_t ldsa, const double* Sb, int64_t d, int64_t n,
                         double* x, double* R, int64_t ldr, double* Q, int64_t ldq,
                         int64_t* bad_col, double* bad_val, void* stream, bool sync) {
  cudaStream_t st = (cudaStream_t)stream;
  SKL_REQUIRE(d >= n && n >= 1, SKL_ERR_SHAPE,
              "economy_qr requires rows >= cols, got %lldx%lld", (long long)d, (long long)n);
  SKL_REQUIRE(SA && ldsa >= d && bad_col && bad_val, SKL_ERR_INVALID, "qr_solve: bad arguments");
  SKL_REQUIRE(!R || ldr >= n, SKL_ERR_INVALID, "qr_solve: ldr < n");
  SKL_REQUIRE(!Q || ldq >= d, SKL_ERR_INVALID, "qr_solve: ldq < d");
  // the back-solves keep y (n doubles) in shared memory
  SKL_REQUIRE(n <= (200 * 1024) / 8, SKL_ERR_SPEC, "qr_solve: n=%lld too large", (long long)n);
  if (n * 8 > 48 * 1024) {
    const int bytes = (int)(n * 8);
    SKL_CUDA(raise_smem_limit(qr_backsolve_inv_kernel, (size_t)bytes));
    SKL_CUDA(raise_smem_limit(qr_backsolve_blocked_kernel, (size_t)bytes));
    SKL_CUDA(raise_smem_limit(qr_backsolve_kernel, (size_t)bytes));
  }

  const int fro_blocks = 256;
  // the blocked factorisation (register cluster panels + GEMM-shaped
  // trailing updates) wins from a few panels on; very narrow systems use the
  // unblocked kernel (SKL_QR_BLOCKED_MIN_N overrides the cut-over)
  static const int64_t min_n = env_int("SKL_QR_BLOCKED_MIN_N", 64);
  const bool blocked = n >= min_n && qr_blocked_supported(d);
  const int64_t ldm = blocked ? (d + 1) / 2 * 2 : d;
  const int64_t npan = (n + 31) / 32;
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off += (bytes + 255) / 256 * 256;
    return o;
  };
  const size_t oM = take((size_t)ldm * (n + 1) * 8), oTau = take(n * 8), oBeta = take(n * 8),
               oInfo = take(2 * (n + 1) * 8), oY = take(n * 8), oPart = take(fro_blocks * 8),
               oFro = take(8), oBad = take(8), oBadV = take(8), oX = take(n * 8),
               oV = blocked ? take((size_t)ldm * n * 8) : 0,
               oT = blocked ? take((size_t)npan * 32 * 32 * 8) : 0,
               oW = blocked ? take((size_t)32 * (n + 1) * 8) : 0,
               oW2 = blocked ? take((size_t)32 * (n + 1) * 8) : 0,
               oW2b = blocked ? take((size_t)32 * (n + 1) * 8) : 0,
               oRinv = blocked ? take((size_t)((n + 31) / 32) * 1024 * 8) : 0,
               oQ = (blocked && Q) ? take((size_t)ldm * n * 8) : 0;
  const int64_t part_cap = blocked ? 32 * (n + 1) * ((d + 63) / 64) : 0;  // 64-row splits
  const size_t oP = blocked ? take((size_t)part_cap * 8) : 0;
  const size_t oPb = blocked ? take((size_t)part_cap * 8) : 0;  // second stream's scratch
  unsigned char* ws = nullptr;
  SKL_CUDA(malloc_async(&ws, off, st));
  double* M = (double*)(ws + oM);
  double* tau = (double*)(ws + oTau);
  double* beta = (double*)(ws + oBeta);
  double* info = (double*)(ws + oInfo);
  double* y = (double*)(ws + oY);
  double* part = (double*)(ws + oPart);
  double* fro2 = (double*)(ws + oFro);
  int64_t* badc = (int64_t*)(ws + oBad);
  double* badv = (double*)(ws + oBadV);
  double* xd = x ? x : (double*)(ws + oX);

  int rc = SKL_OK;
  do {
    copy_aug_kernel<<<fro_blocks, 256, 0, st>>>(SA, ldsa, Sb, d, n, M, ldm, part);
    // a launch error leaves the loop with rc set, so the workspace is freed
#define QR_LAUNCH(call)                                                     \
  if ((e = (call)) != cudaSuccess) {                                        \
    set_error("qr_solve: kernel launch failed: %s", cudaGetErrorString(e)); \
    rc = SKL_ERR_CUDA;                                                      \
    break;                                                                  \
  }
    cudaError_t e = cudaSuccess;
    QR_LAUNCH(launch_k(sum_parts_kernel, dim3(1), dim3(256), 0, st, true, (const double*)part,
                       fro_blocks, fro2));
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (blocked) {
      double* V = (double*)(ws + oV);
      double* T = (double*)(ws + oT);
      double* W = (double*)(ws + oW);
      double* W2 = (double*)(ws + oW2);
      double* Pw = (double*)(ws + oP);
      rc = qr_blocked_factor(M, ldm, d, n, tau, beta, V, T, W, W2, Pw, part_cap,
                             (double*)(ws + oW2b), (double*)(ws + oPb), st);
      if (rc) break;
      qr_finish_kernel<<<1, 256, 0, st>>>(M, ldm, n, beta, fro2, R, ldr, y, badc, badv);
      static const bool subst = env_flag("SKL_QR_SUBST_BACKSOLVE");  // A/B knob
      if (!subst) {
        double* Rinv = (double*)(ws + oRinv);
        const int64_t nb = (n + 31) / 32;
        QR_LAUNCH(launch_k(qr_trinv_kernel, dim3((unsigned)((nb + TRI_WPB - 1) / TRI_WPB)),
                           dim3(TRI_WPB * 32), 0, st, true, (const double*)M, ldm, n,
                           (const double*)beta, Rinv));
        QR_LAUNCH(launch_k(qr_backsolve_inv_kernel, dim3(1), dim3(BS_NT), n * sizeof(double), st,
                           true, (const double*)M, ldm, n, (const double*)beta,
                           (const double*)Rinv, (const double*)y, xd));
      } else {
        qr_backsolve_blocked_kernel<<<1, 512, n * sizeof(double), st>>>(M, ldm, n, beta, y, xd);
      }
      if (Q) {
        double* Qw = (double*)(ws + oQ);
        const int64_t tot = d * n;
        const int blocks = (int)std::min<int64_t>((tot + 255) / 256, 8LL * sms);
        eye_kernel<<<blocks, 256, 0, st>>>(Qw, ldm, d, n);
        rc = qr_blocked_form_q(Qw, ldm, d, n, V, ldm, T, W, W2, Pw, part_cap, st);
        if (rc) break;
        q_signfix_copy_kernel<<<blocks, 256, 0, st>>>(Qw, ldm, beta, d, n, Q, ldq);
      }
    } else {
      int per_sm = 1;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, qr_householder_kernel, QR_NT, 0);
      int grid = (int)std::min<int64_t>((int64_t)sms * std::max(1, per_sm), n + 1);
      QrParams p{M, d, n, tau, beta, info};
      void* args[] = {&p};
      e = cudaLaunchCooperativeKernel((void*)qr_householder_kernel, grid, QR_NT, args, 0, st);
      if (e != cudaSuccess) {
        set_error("qr kernel launch failed: %s", cudaGetErrorString(e));
        rc = SKL_ERR_CUDA;
        break;
      }
      qr_finish_kernel<<<1, 256, 0, st>>>(M, d, n, beta, fro2, R, ldr, y, badc, badv);
      qr_backsolve_kernel<<<1, 1024, n * sizeof(double), st>>>(M, d, n, beta, y, xd);
      if (Q) {
        qr_scale_reflectors<<<(int)std::min<int64_t>(n, 1024), 256, 0, st>>>(M, d, n, tau, beta);
        int gq = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&gq, qr_form_q_kernel, QR_NT, 0);
        int gridq = (int)std::min<int64_t>((int64_t)sms * std::max(1, gq), n);
        void* qargs[] = {&M, &d, &n, &tau, &beta, &Q, &ldq};
        e = cudaLaunchCooperativeKernel((void*)qr_form_q_kernel, gridq, QR_NT, qargs, 0, st);
        if (e != cudaSuccess) {
          set_error("form-Q kernel launch failed: %s", cudaGetErrorString(e));
          rc = SKL_ERR_CUDA;
          break;
        }
      }
    }
    e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaMemcpyAsync(bad_col, badc, 8, cudaMemcpyDefault, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(bad_val, badv, 8, cudaMemcpyDefault, st);
    if (e == cudaSuccess && sync) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) {
      set_error("qr_solve: %s", cudaGetErrorString(e));
      rc = SKL_ERR_CUDA;
    }
  } while (0);
#undef QR_LAUNCH
  cudaFreeAsync(ws, st);
  if (rc == SKL_OK && sync && *bad_col >= 0) {
    set_error("input is numerically rank deficient at column %lld (|R[%lld,%lld]| = %.3e)",
              (long long)*bad_col, (long long)*bad_col, (long long)*bad_col, *bad_val);
    return SKL_ERR_SINGULAR;
  }
  return rc;
}
