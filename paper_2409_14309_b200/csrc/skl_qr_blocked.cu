// Blocked Householder QR of the sketched system on device (the path
// skl_qr_solve takes when the panel fits a thread-block cluster).
//
// Reference semantics: LAPACK dgeqrf as called through numpy.linalg.qr
// (/root/reference/pkg/src/sketchls/linalg.py:175); reflectors follow dlarfg
// and the block reflector I - V T V^T follows dlarft (forward, columnwise).
//
// Per panel of NB = 32 columns:
//  1. qr_panel_cluster_kernel: ONE thread-block cluster (up to 16 CTAs)
//     holds the panel's rows j0..d-1 in distributed shared memory, split in
//     row blocks.  Each of the NB reflector steps computes per-CTA partial
//     dot products (lane = column), publishes them in shared memory, and
//     after one cluster barrier every CTA sums all CTAs' partials (DSMEM
//     reads, fixed CTA order -> deterministic) and updates its rows.  At the
//     end the CTAs reduce V^T V the same way and CTA 0 forms T.
//  2. W = V^T C (row-split partials, fixed-order reduction), W <- T^T W,
//     and C <- C - V W (register-tiled DFMA kernel) for the trailing columns,
//     which include the Sb column, so Q^T Sb falls out of the factorisation.
// One cluster barrier per column replaces the grid-wide synchronisation an
// unblocked right-looking factorisation needs, and the O(d n^2) trailing
// work becomes GEMM-shaped.
#include <cuda_runtime.h>

#include <vector>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>

#include "skl_common.h"
#include "skl_ptx.cuh"

namespace skl {

constexpr int QB_NB = 32;        // panel width
constexpr int QB_PLD = 33;       // panel row stride in shared memory (conflict-free)
constexpr int QB_NT = 1024;      // threads per CTA (32 warps)
constexpr int QB_NW = QB_NT / 32;
constexpr int QB_MAXCL = 16;     // max cluster size (non-portable)
constexpr int QB_MAXROWS = 680;  // rows per CTA that fit in shared memory
// pub[2][64] + red[32][32] + G[32][32] + sc[2][64] + Ts[32][32]
constexpr int QB_SMEM_EXTRA = 128 + 1024 + 1024 + 128 + 1024;

__device__ __forceinline__ uint32_t cta_rank_in_cluster() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;"
               ::: "memory");
}
// Remote shared-memory load.  Ordering w.r.t. the remote writes comes from
// the cluster barrier that precedes every use, so the asm is not volatile and
// independent loads can be in flight together.
__device__ __forceinline__ double ld_dsmem(const double* local, uint32_t cta) {
  const uint32_t a = static_cast<uint32_t>(__cvta_generic_to_shared(local));
  uint32_t ra;
  asm("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(a), "r"(cta));
  double v;
  asm("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(ra));
  return v;
}

// Instrumented builds (SKL_NVCC_DEFINES=-DSKL_QR_PROBE): CTA 0 thread 0 of
// the panel kernel accumulates clock64 cycles per phase; the host prints the
// totals after each factorisation.
#ifdef SKL_QR_PROBE
__device__ unsigned long long g_qr_probe[12];
#define QR_PROBE_INIT long long pr_[12] = {}; long long t0_ = clock64();
#define QR_PROBE(i) do { if (rank == 0 && tid == 0) { long long t_ = clock64(); pr_[i] += t_ - t0_; t0_ = t_; } } while (0)
#define QR_PROBE_FLUSH do { if (rank == 0 && tid == 0) for (int q_ = 0; q_ < 12; ++q_) atomicAdd(&g_qr_probe[q_], (unsigned long long)pr_[q_]); } while (0)
#else
#define QR_PROBE_INIT
#define QR_PROBE(i) do {} while (0)
#define QR_PROBE_FLUSH do {} while (0)
#endif

struct PanelParams {
  double* M;        // ld ldm, the whole augmented matrix
  int64_t ldm, d;
  int64_t j0;       // first panel column (and row)
  int jb;           // panel width (<= 32)
  int rows_per;     // rows per CTA
  double* V;        // explicit reflectors, ld ldm (rows j0.. of columns j0..j0+jb)
  double* T;        // jb x jb (ld 32) block reflector factor
  double* tau;
  double* beta;
};

__global__ void __launch_bounds__(QB_NT) qr_panel_cluster_kernel(const PanelParams p) {
  pdl_enter();
  extern __shared__ __align__(16) double qsm[];
  const uint32_t rank = cta_rank_in_cluster();
  const uint32_t ncta = gridDim.x;  // one cluster spans the grid
  double* P = qsm;                                  // [rows_per][QB_PLD]
  double* pub = P + (size_t)p.rows_per * QB_PLD;    // [2][64]: column sums, pivot row
  double* red = pub + 128;                          // [32 warps][32]
  double* G = red + 1024;                           // [32][32]: column k = V^T v_k
  double* sc = G + 1024;                            // [2][64]: w_j, scale, beta
  double* Ts = sc + 128;                            // [32][32]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t rbeg = p.j0 + (int64_t)rank * p.rows_per;
  const int nloc = (int)std::max<int64_t>(0, std::min<int64_t>(p.rows_per, p.d - rbeg));
  const int jb = p.jb;
  QR_PROBE_INIT

  // load the panel slice (column-major source -> row-major smem)
  #pragma unroll 8
  for (int idx = tid; idx < nloc * QB_NB; idx += QB_NT) {
    const int j = idx / nloc, i = idx % nloc;  // coalesced along rows
    P[i * QB_PLD + j] = j < jb ? p.M[(p.j0 + j) * p.ldm + rbeg + i] : 0.0;
  }
  __syncthreads();
  QR_PROBE(0);

  // Per column k (pivot row g): warps own local rows i = warp (mod 32) in
  // both the dot-product and the update loop, so P needs no barrier between
  // steps; two CTA barriers and one cluster barrier per column.  Warp 0 does
  // the scalar work (sums over warps and CTAs, dlarfg) once and publishes
  // w_j and the reflector scale.
  for (int k = 0; k < jb; ++k) {
    const int64_t g = p.j0 + k;
    double* pb = pub + (k & 1) * 64;
    double* sk = sc + (k & 1) * 64;
    const int gl = (int)std::max<int64_t>(-1, std::min<int64_t>(g - rbeg, nloc));
    // first local row > gl owned by this warp
    const int i0 = gl + 1 + ((warp - (gl + 1)) % 32 + 32) % 32;
    // s_j = sum_{i > g} P[i][k] P[i][j]  (j > k: trailing dots; j < k: V^T v)
    double s0 = 0.0, s1 = 0.0;
    int i = i0;
    for (; i + 32 < nloc; i += 64) {
      s0 = fma(P[i * QB_PLD + k], P[i * QB_PLD + lane], s0);
      s1 = fma(P[(i + 32) * QB_PLD + k], P[(i + 32) * QB_PLD + lane], s1);
    }
    if (i < nloc) s0 = fma(P[i * QB_PLD + k], P[i * QB_PLD + lane], s0);
    QR_PROBE(1);
    red[warp * 32 + lane] = s0 + s1;
    __syncthreads();
    QR_PROBE(2);
    if (warp == 0) {
      double t0 = 0.0, t1 = 0.0, t2 = 0.0, t3 = 0.0;
#pragma unroll
      for (int w = 0; w < QB_NW; w += 4) {
        t0 += red[w * 32 + lane];
        t1 += red[(w + 1) * 32 + lane];
        t2 += red[(w + 2) * 32 + lane];
        t3 += red[(w + 3) * 32 + lane];
      }
      pb[lane] = (t0 + t1) + (t2 + t3);
      if (gl >= 0 && gl < nloc) pb[32 + lane] = P[gl * QB_PLD + lane];
    }
    QR_PROBE(3);
    cluster_sync_all();
    QR_PROBE(4);
    if (warp == 0) {
      // sum the CTAs' partials in fixed CTA order (remote loads issued together)
      const uint32_t owner = (uint32_t)((g - p.j0) / p.rows_per);
      double part[QB_MAXCL];
#pragma unroll
      for (int q = 0; q < QB_MAXCL; ++q) part[q] = q < (int)ncta ? ld_dsmem(pb + lane, q) : 0.0;
      const double pj = ld_dsmem(pb + 32 + lane, owner);
      double Sj = 0.0;
#pragma unroll
      for (int q = 0; q < QB_MAXCL; ++q) Sj += part[q];
      const double Sk = __shfl_sync(0xffffffffu, Sj, k);
      const double alpha = __shfl_sync(0xffffffffu, pj, k);
      const double xnorm = sqrt(Sk);
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
      sk[lane] = (lane > k && lane < jb) ? tau * (pj + scale * Sj) : 0.0;
      // V_j^T v_k = V_j[g] + scale * sum_{i>g} V_j[i] x_i  (j < k)
      G[k * 32 + lane] = lane < k ? pj + scale * Sj : 0.0;
      if (lane == 0) {
        sk[32] = scale;
        sk[33] = beta;
        if (rank == 0) {
          p.tau[g] = tau;
          p.beta[g] = beta;
        }
        Ts[k * 32 + k] = tau;
      }
    }
    QR_PROBE(5);
    __syncthreads();
    QR_PROBE(6);
    const double wj = sk[lane], scale = sk[32];
    // update local rows below the pivot; column k becomes v
    for (int r = i0; r < nloc; r += 32) {
      const double v = scale * P[r * QB_PLD + k];
      const double o = P[r * QB_PLD + lane];
      P[r * QB_PLD + lane] = lane == k ? v : fma(-wj, v, o);
    }
    if (gl >= 0 && gl < nloc && warp == (gl & 31)) {
      const double o = P[gl * QB_PLD + lane];
      P[gl * QB_PLD + lane] = lane == k ? sk[33] : o - wj;
    }
    QR_PROBE(7);
  }
  __syncthreads();

  // T (dlarft, forward columnwise): T[k][k] = tau_k,
  // T[0:k, k] = -tau_k T[0:k, 0:k] G[0:k, k]; one warp, T in shared memory.
  if (warp == 0) {
    for (int k = 0; k < jb; ++k) {
      const double tk = Ts[k * 32 + k];
      double a0 = 0.0, a1 = 0.0;
      if (lane < k) {
        int l = lane;
        for (; l + 1 < k; l += 2) {
          a0 = fma(Ts[l * 32 + lane], G[k * 32 + l], a0);
          a1 = fma(Ts[(l + 1) * 32 + lane], G[k * 32 + l + 1], a1);
        }
        if (l < k) a0 = fma(Ts[l * 32 + lane], G[k * 32 + l], a0);
      }
      __syncwarp();
      if (lane != k) Ts[k * 32 + lane] = lane < k ? -tk * (a0 + a1) : 0.0;
      __syncwarp();
    }
  }
  __syncthreads();
  if (rank == 0)
    #pragma unroll 8
    for (int e = tid; e < QB_NB * QB_NB; e += QB_NT) p.T[e] = (e / 32) < jb ? Ts[e] : 0.0;
  // write back the panel and the explicit V
  #pragma unroll 8
  for (int idx = tid; idx < nloc * QB_NB; idx += QB_NT) {
    const int j = idx / nloc, i = idx % nloc;
    if (j >= jb) continue;
    const int64_t gi = rbeg + i, gj = p.j0 + j;
    const double val = P[i * QB_PLD + j];
    p.M[gj * p.ldm + gi] = val;
    p.V[gj * p.ldm + gi] = gi < gj ? 0.0 : (gi == gj ? 1.0 : val);
  }
  QR_PROBE(8);
  cluster_sync_all();  // keep shared memory alive for remote readers
  QR_PROBE(9);
  QR_PROBE_FLUSH;
}

// Register-resident panel factorisation: the production panel kernel.
//
// Rows of the panel [j0, d) x [j0, j0 + jb) are split into the HEAD (rows
// j0 .. j0+jb-1, which hold every pivot of the panel; CTA 0, two rows per
// warp) and the TAIL (rows below, spread over the cluster's CTAs, RPW rows
// per warp).  Thread (warp w, lane j) keeps column j of its rows in
// registers for the whole panel, so the per-column dot products and updates
// never touch shared memory; the pivot-column value of a row comes from lane
// k by a shuffle.  Tail rows lie below every pivot, so their updates carry
// no row predicates: P <- P - w_j (scale * x).  Column k itself is left
// unscaled (w_j = 0 for j <= k) and scaled by scale_k at write-back; the
// V^T v products the T factor needs come from the same dot products
// (lanes j < k), corrected by scale_j.
//
// Per column the only cross-CTA exchange is a push: each CTA reduces its 16
// warp partials and bulk-copies the 32 column sums into every CTA's inbox
// (cp.async.bulk shared::cta -> shared::cluster, completing on the
// receiver's mbarrier); CTA 0 also pushes the pivot row.  No cluster-wide
// barrier per column.  Double-buffered by column parity (see the ordering
// argument at the buffers).
constexpr int QR_NT2 = 512;
constexpr int QR_NW2 = QR_NT2 / 32;
#ifndef QR_PUSHW
#define QR_PUSHW 2  // warps that push the column sums to the cluster
#endif
// extra shared memory of the register panel (doubles): inbox[2][16][32],
// inrow[2][32], red[16][33], G[32][32], Ts[32][32], colscale[32],
// sc[2][128], mbarriers
constexpr int QR2_SMEM_EXTRA = 2 * QB_MAXCL * 32 + 64 + 16 * 33 + 1024 + 1024 + 32 + 256 + 8;

// staging doubles, even so the buffers after it stay 16-byte aligned
__host__ __device__ inline size_t qr2_staging(int rows_per) {
  return ((size_t)(rows_per > 32 ? rows_per : 32) * QB_PLD + 1) & ~(size_t)1;
}

// The block-reflector factor T of a panel (dlarft, forward columnwise):
// T[k][k] = tau_k (already in Ts), T[0:k, k] = -tau_k T[0:k, 0:k] G[0:k, k]
// with G[l][k] = V_l^T v_k stored at G[k * 32 + l].  One warp, lane = row
// i of T.  Instead of one dot product per column (a dependent chain of
// loads and FMAs), each finished T[i][k] is immediately folded into the
// running sums of every later column, acc[k'] += T[i][k] G[k][k'], so a
// column step is one multiply on the critical path plus independent FMAs.
// Runs after the panel's rows are written back, when their registers are
// free.
__device__ __forceinline__ void panel_t_build(double* Ts, const double* G, int jb, int lane) {
  double acc[32];
#pragma unroll
  for (int k = 0; k < 32; ++k) acc[k] = 0.0;
#pragma unroll
  for (int k = 0; k < 32; ++k) {
    if (k < jb) {
      const double tk = Ts[k * 32 + k];
      const double t = lane < k ? -tk * acc[k] : (lane == k ? tk : 0.0);
#pragma unroll
      for (int kk = k + 1; kk < 32; ++kk) acc[kk] = fma(t, G[kk * 32 + k], acc[kk]);
      __syncwarp();
      Ts[k * 32 + lane] = t;
    }
  }
  __syncwarp();
}

// dlarfg's scalars for a column with sum of squares below the pivot Sk > 0
// and pivot alpha: beta = -sign(alpha) N with N = sqrt(alpha^2 + Sk),
// tau = (beta - alpha) / beta = 1 + |alpha| / N and scale = 1 / (alpha -
// beta) = sign(alpha) / (|alpha| + N).  They sit on the panel's per-column
// critical path: N comes from the IEEE square root (~80 cycles on the B200;
// rsqrt.approx.f64 alone takes ~75), the two reciprocals from
// rcp.approx.ftz.f64 (~18 cycles) refined by two independent Newton steps
// each, side by side, instead of two IEEE divisions in sequence (~60 cycles
// each plus their slow-path branches).  A few ulp, not correctly rounded; R
// is compared with LAPACK within 1e-12.
__device__ __forceinline__ double rcp_nr(double t) {
  double q;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(q) : "d"(t));
#pragma unroll
  for (int it = 0; it < 2; ++it) q = fma(q, fma(-t, q, 1.0), q);
  return q;
}
__device__ __forceinline__ void house_scalars(double alpha, double Sk, double& beta, double& tau,
                                              double& scale) {
  const double N = sqrt(fma(alpha, alpha, Sk));
  const double aa = fabs(alpha);
  const double rN = rcp_nr(N), rs = rcp_nr(aa + N);
  beta = alpha < 0.0 ? N : -N;
  tau = fma(aa, rN, 1.0);
  scale = alpha < 0.0 ? -rs : rs;
}

template <int RPW>
__global__ void __launch_bounds__(QR_NT2) qr_panel_reg_kernel(const PanelParams p) {
  pdl_enter();
  constexpr bool KEEPX = RPW <= 16;
  extern __shared__ __align__(16) double qsm[];
  const uint32_t rank = cta_rank_in_cluster();
  const uint32_t ncta = gridDim.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int jb = p.jb;
  const int64_t tail0 = p.j0 + jb;                         // first tail row
  const int64_t tbeg = tail0 + (int64_t)rank * p.rows_per;
  const int nt = (int)std::max<int64_t>(0, std::min<int64_t>(p.rows_per, p.d - tbeg));
  const bool head = rank == 0;

  double* S = qsm;                                         // staging [max(rows_per, 32)][QB_PLD]
  double* inbox = S + qr2_staging(p.rows_per);             // [2][16][32]
  double* inrow = inbox + 2 * QB_MAXCL * 32;               // [2][32]
  double* red = inrow + 64;                                // [16][33]
  double* G = red + 16 * 33;                               // [32][32]: column k = V^T v_k
  double* Ts = G + 1024;                                   // [32][32]
  double* colscale = Ts + 1024;                            // [32]
  double* sc = colscale + 32;                              // [2][128]: w_j scale, w_j, beta
  uint64_t* mb = reinterpret_cast<uint64_t*>(sc + 256);    // [2]
  QR_PROBE_INIT

  if (tid == 0) {
    mbar_init(&mb[0], 1);
    mbar_init(&mb[1], 1);
    fence_mbar_init();
  }
  // stage tail rows (coalesced along rows), then the head rows
  #pragma unroll 8
  for (int idx = tid; idx < nt * QB_NB; idx += QR_NT2) {
    const int j = idx / nt, i = idx % nt;
    S[i * QB_PLD + j] = j < jb ? p.M[(p.j0 + j) * p.ldm + tbeg + i] : 0.0;
  }
  __syncthreads();
  // Layout A (RPW <= 16): lane = column, RPW rows per thread.  Layout B
  // (RPW == 32, d > 4096): lane = (column pair cp = lane & 15, row half
  // hh = lane >> 4), 16 rows x 2 columns per thread -- a column step then
  // needs 16 pivot values per thread (32 shuffles) instead of 32 (64), and
  // they fit in registers for the update, which needs none (layout A at
  // RPW = 32 spent two shuffle-bound phases of ~1.2 K cycles per column).
  // (the 2-column layout for RPW <= 16 too measured 1-5 % slower)
  constexpr bool LB = RPW == 32;
  constexpr int NP = LB ? RPW / 2 : RPW;  // row slots per thread
  const int cp = lane & 15, hh = lane >> 4;
  double P[NP];
  double P1[LB ? NP : 1];  // layout B: the pair's second column
#pragma unroll
  for (int r = 0; r < NP; ++r) {
    if constexpr (LB) {
      const int li = (2 * r + hh) * QR_NW2 + warp;
      P[r] = li < nt ? S[li * QB_PLD + 2 * cp] : 0.0;
      P1[r] = li < nt ? S[li * QB_PLD + 2 * cp + 1] : 0.0;
    } else {
      const int li = r * QR_NW2 + warp;
      P[r] = li < nt ? S[li * QB_PLD + lane] : 0.0;
    }
  }
  (void)P1;
  (void)cp;
  (void)hh;
  __syncthreads();
  double H0 = 0.0, H1 = 0.0;  // head rows warp and warp + 16 (CTA 0)
  if (head) {
    #pragma unroll 8
    for (int idx = tid; idx < 32 * QB_NB; idx += QR_NT2) {
      const int j = idx / 32, i = idx % 32;
      S[i * QB_PLD + j] = (j < jb && i < jb) ? p.M[(p.j0 + j) * p.ldm + p.j0 + i] : 0.0;
    }
    __syncthreads();
    H0 = S[warp * QB_PLD + lane];
    H1 = S[(warp + 16) * QB_PLD + lane];
  }
  cluster_sync_all();  // barriers initialised everywhere before any push
  // pivot row of column 0 -> every CTA's inrow[0]
  if (head && warp == 0)
    for (uint32_t q = 0; q < ncta; ++q)
      st_async_f64(mapa_u32(smem_u32(inrow + lane), q), H0, mapa_u32(smem_u32(&mb[0]), q));
  QR_PROBE(0);
  double myscale = 0.0;  // warp 0: scale of column `lane`

  for (int k = 0; k < jb; ++k) {
    const int b = k & 1;
    // ---- dot products s_j = sum_{i > pivot} x_i P_i[j]
    double xs[KEEPX ? NP : 1];
    double s0 = 0.0, s1 = 0.0;
    if constexpr (LB) {
      // pivot values of this thread's rows: column k lives in lane
      // (k >> 1) of the same row half, in P (k even) or P1 (k odd)
      const int src = (k >> 1) | (hh << 4);
      const bool odd = k & 1;
      double ev = 0.0, ov = 0.0;
#pragma unroll
      for (int r = 0; r < NP; ++r) {
        const double x = __shfl_sync(0xffffffffu, odd ? P1[r] : P[r], src);
        if constexpr (KEEPX) xs[r] = x;
        ev = fma(x, P[r], ev);
        ov = fma(x, P1[r], ov);
      }
      // lane (cp, hh) keeps column 2 cp + hh: its half plus the other half's
      const double other = __shfl_xor_sync(0xffffffffu, hh ? ev : ov, 16);
      s0 = (hh ? ov : ev) + other;
    } else {
#pragma unroll
      for (int r = 0; r < RPW; ++r) {
        const double x = __shfl_sync(0xffffffffu, P[r], k);
        if (KEEPX) xs[r & (KEEPX ? RPW - 1 : 0)] = x;
        if (r & 1)
          s1 = fma(x, P[r], s1);
        else
          s0 = fma(x, P[r], s0);
      }
    }
    double xh0 = 0.0, xh1 = 0.0;
    if (head) {
      xh0 = __shfl_sync(0xffffffffu, H0, k);
      xh1 = __shfl_sync(0xffffffffu, H1, k);
      if constexpr (LB) {
        // head rows stay in layout A (lane = column): move their column
        // sums to the lane that holds the tail sum of the same column
        double hs = 0.0;
        if (warp > k) hs = fma(xh0, H0, hs);
        if (warp + 16 > k) hs = fma(xh1, H1, hs);
        s1 = __shfl_sync(0xffffffffu, hs, 2 * cp + hh);
      } else {
        if (warp > k) s0 = fma(xh0, H0, s0);
        if (warp + 16 > k) s1 = fma(xh1, H1, s1);
      }
    }
    QR_PROBE(1);
    red[warp * 33 + (LB ? 2 * cp + hh : lane)] = s0 + s1;
    __syncthreads();
    QR_PROBE(2);
    // Buffers of parity b are rewritten only at column k + 2: by then this
    // CTA has received every CTA's column-(k+1) push, each sent after that
    // CTA's column-(k+1) __syncthreads, i.e. after it read its column-k
    // inbox, and after our column-k copies into it landed.
    // Warps 0 .. QR_PUSHW-1 each fold the 16 warp partials (fixed order, so
    // bitwise the same sums everywhere) and push them, one coalesced
    // 256-byte store per destination, into the inboxes of CTAs
    // w, w + QR_PUSHW, ...
    if (warp < QR_PUSHW) {
      double tot;
      if (RPW == 32) {
        double t[QR_NW2];
#pragma unroll
        for (int w = 0; w < QR_NW2; ++w) t[w] = red[w * 33 + lane];
#pragma unroll
        for (int w = QR_NW2 / 2; w >= 1; w >>= 1)
#pragma unroll
          for (int q = 0; q < w; ++q) t[q] += t[q + w];
        tot = t[0];
      } else {
        double t0 = 0.0, t1 = 0.0, t2 = 0.0, t3 = 0.0;
#pragma unroll
        for (int w = 0; w < QR_NW2; w += 4) {
          t0 += red[w * 33 + lane];
          t1 += red[(w + 1) * 33 + lane];
          t2 += red[(w + 2) * 33 + lane];
          t3 += red[(w + 3) * 33 + lane];
        }
        tot = (t0 + t1) + (t2 + t3);
      }
      if (warp == 0 && lane == 0) mbar_arrive_expect_tx(&mb[b], (ncta + 1) * 256);
      const uint32_t dst = smem_u32(inbox + (b * QB_MAXCL + rank) * 32 + lane);
      const uint32_t mbl = smem_u32(&mb[b]);
      for (uint32_t q = warp; q < ncta; q += QR_PUSHW)
        st_async_f64(mapa_u32(dst, q), tot, mapa_u32(mbl, q));
    }
    if (warp == 0) {
      QR_PROBE(3);
      mbar_wait_cluster(&mb[b], (uint32_t)((k >> 1) & 1));
      QR_PROBE(4);
      double Sj;
      const double* ib = inbox + b * QB_MAXCL * 32 + lane;
      if (RPW == 32) {
        double u[QB_MAXCL];
#pragma unroll
        for (int q = 0; q < QB_MAXCL; ++q)  // all loads in flight at once
          u[q] = q < (int)ncta ? ib[q * 32] : 0.0;
#pragma unroll
        for (int w = QB_MAXCL / 2; w >= 1; w >>= 1)  // fixed-order tree
#pragma unroll
          for (int q = 0; q < w; ++q) u[q] += u[q + w];
        Sj = u[0];
      } else {
        double u[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
        for (int q = 0; q < QB_MAXCL; ++q)  // all loads in flight at once
          if (q < (int)ncta) u[q & 3] += ib[q * 32];
        Sj = (u[0] + u[1]) + (u[2] + u[3]);
      }
      const double pj = inrow[b * 32 + lane];
      const double Sk = __shfl_sync(0xffffffffu, Sj, k);
      const double alpha = __shfl_sync(0xffffffffu, pj, k);
      double tau, beta, scale;
      if (Sk == 0.0) {
        tau = 0.0;
        beta = alpha;
        scale = 0.0;
      } else {
        if (RPW == 32) {
          house_scalars(alpha, Sk, beta, tau, scale);
        } else {  // measured faster here (timing, not accuracy)
          beta = -copysign(sqrt(fma(alpha, alpha, Sk)), alpha);
          tau = (beta - alpha) / beta;
          scale = 1.0 / (alpha - beta);
        }
      }
      if (lane == k) myscale = scale;
      // rows below the pivot: P_i[j] -= (w_j scale) x_i; the pivot row: -= w_j
      const double wv = (lane > k && lane < jb) ? tau * (pj + scale * Sj) : 0.0;
      sc[b * 128 + lane] = wv * scale;
      sc[b * 128 + 32 + lane] = wv;
      // V_j^T v_k = scale_j (U_j[g] + scale_k sum_{i>g} U_j[i] x_i), U unscaled
      G[k * 32 + lane] = lane < k ? myscale * (pj + scale * Sj) : 0.0;
      if (lane == 0) {
        sc[b * 128 + 64] = beta;
        colscale[k] = scale;
        Ts[k * 32 + k] = tau;
        if (head) {
          p.tau[p.j0 + k] = tau;
          p.beta[p.j0 + k] = beta;
        }
      }
    }
    QR_PROBE(5);
    __syncthreads();
    QR_PROBE(6);
    const double ws = sc[b * 128 + lane];
    if constexpr (LB) {
      // the pivot values again (no registers left to keep them: 16 rows x 2
      // columns of the panel, and the dlarfg path of warp 0)
      const double w0 = sc[b * 128 + 2 * cp], w1 = sc[b * 128 + 2 * cp + 1];
      const int src = (k >> 1) | (hh << 4);
      const bool odd = k & 1;
#pragma unroll
      for (int r = 0; r < NP; ++r) {
        double x;
        if constexpr (KEEPX)
          x = xs[r];
        else
          x = __shfl_sync(0xffffffffu, odd ? P1[r] : P[r], src);
        P[r] = fma(-w0, x, P[r]);
        P1[r] = fma(-w1, x, P1[r]);
      }
    } else {
#pragma unroll
      for (int r = 0; r < RPW; ++r) {
        const double x = KEEPX ? xs[r & (KEEPX ? RPW - 1 : 0)] : __shfl_sync(0xffffffffu, P[r], k);
        P[r] = fma(-ws, x, P[r]);
      }
    }
    if (head) {
      const double wj = sc[b * 128 + 32 + lane], beta = sc[b * 128 + 64];
      if (warp > k) H0 = fma(-ws, xh0, H0);
      else if (warp == k) H0 = lane == k ? beta : H0 - wj;
      if (warp + 16 > k) H1 = fma(-ws, xh1, H1);
      else if (warp + 16 == k) H1 = lane == k ? beta : H1 - wj;
      // push the next pivot row into every CTA's inrow (its mbarrier for
      // column k + 1 is in that phase: its column k - 1 wait completed before
      // it sent the column-k sums this CTA has received)
      if (k + 1 < jb && warp == ((k + 1) & 15)) {
        const int bn = (k + 1) & 1;
        const double rv = (k + 1) < 16 ? H0 : H1;
        const uint32_t dst = smem_u32(inrow + bn * 32 + lane), mbl = smem_u32(&mb[bn]);
        for (uint32_t q = 0; q < ncta; ++q) st_async_f64(mapa_u32(dst, q), rv, mapa_u32(mbl, q));
      }
    }
    QR_PROBE(7);
  }

  // ---- write back: column j rows below its pivot are scale_j * stored
  __syncthreads();
#pragma unroll
  for (int r = 0; r < NP; ++r) {
    if constexpr (LB) {
      const int li = (2 * r + hh) * QR_NW2 + warp;
      if (li < nt) {
        S[li * QB_PLD + 2 * cp] = P[r];
        S[li * QB_PLD + 2 * cp + 1] = P1[r];
      }
    } else {
      const int li = r * QR_NW2 + warp;
      if (li < nt) S[li * QB_PLD + lane] = P[r];
    }
  }
  __syncthreads();
  #pragma unroll 8
  for (int idx = tid; idx < nt * QB_NB; idx += QR_NT2) {
    const int j = idx / nt, i = idx % nt;
    if (j >= jb) continue;
    const int64_t gi = tbeg + i, gj = p.j0 + j;
    const double val = colscale[j] * S[i * QB_PLD + j];
    p.M[gj * p.ldm + gi] = val;
    p.V[gj * p.ldm + gi] = val;
  }
  QR_PROBE(10);
  if (head) {
    __syncthreads();
    S[warp * QB_PLD + lane] = H0;
    S[(warp + 16) * QB_PLD + lane] = H1;
    __syncthreads();
    #pragma unroll 8
    for (int idx = tid; idx < jb * QB_NB; idx += QR_NT2) {
      const int j = idx / jb, i = idx % jb;
      if (j >= jb) continue;
      const int64_t gi = p.j0 + i, gj = p.j0 + j;
      const double raw = S[i * QB_PLD + j];
      const double val = i > j ? colscale[j] * raw : raw;
      p.M[gj * p.ldm + gi] = val;
      p.V[gj * p.ldm + gi] = i < j ? 0.0 : (i == j ? 1.0 : val);
    }
    if (warp == 0) panel_t_build(Ts, G, jb, lane);
    QR_PROBE(11);
    __syncthreads();
    #pragma unroll 8
    for (int e = tid; e < QB_NB * QB_NB; e += QR_NT2) p.T[e] = (e / 32) < jb ? Ts[e] : 0.0;
  }
  QR_PROBE(8);
  cluster_sync_all();  // every push into this CTA has landed and been read
  QR_PROBE(9);
  QR_PROBE_FLUSH;
}

// C[rows x nc] -= V[rows x jb] * W2[jb x nc]; 64 x 64 tiles, 4 x 4 per thread.
__global__ void __launch_bounds__(256) qr_update_kernel(double* __restrict__ C, int64_t ldc,
                                                        const double* __restrict__ V, int64_t ldv,
                                                        const double* __restrict__ W2, int jb,
                                                        int64_t rows, int64_t nc) {
  __shared__ double Vs[32][64 + 1];
  pdl_enter();
  __shared__ double Ws[32][64 + 1];
  const int64_t i0 = (int64_t)blockIdx.x * 64, c0 = (int64_t)blockIdx.y * 64;
  const int tid = threadIdx.x;
  const int tr = tid % 16, tc = tid / 16;  // rows tr + 16a, cols tc + 16b
  // the 16 outputs are fetched first: their latency overlaps the staging
  double cv[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int64_t i = i0 + tr + 16 * a, c = c0 + tc + 16 * b;
      cv[a][b] = (i < rows && c < nc) ? C[c * ldc + i] : 0.0;
    }
#pragma unroll
  for (int e = tid; e < 32 * 64; e += 256) {
    const int k = e / 64, r = e % 64;
    Vs[k][r] = (k < jb && i0 + r < rows) ? V[(int64_t)k * ldv + i0 + r] : 0.0;
    Ws[k][r] = (k < jb && c0 + r < nc) ? W2[(c0 + r) * 32 + k] : 0.0;
  }
  __syncthreads();
  double acc[4][4] = {};
#pragma unroll 8
  for (int k = 0; k < 32; ++k) {
    double v[4], w[4];
#pragma unroll
    for (int a = 0; a < 4; ++a) v[a] = Vs[k][tr + 16 * a];
#pragma unroll
    for (int b = 0; b < 4; ++b) w[b] = Ws[k][tc + 16 * b];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) acc[a][b] = fma(v[a], w[b], acc[a][b]);
  }
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int64_t i = i0 + tr + 16 * a, c = c0 + tc + 16 * b;
      if (i < rows && c < nc) C[c * ldc + i] = cv[a][b] - acc[a][b];
    }
}

// Trailing update, pass 1: partial W = V^T C over 64-row splits.  Each CTA
// loads its whole 64 x 32 slice of V and of C (one 32-column tile) at once,
// so a split costs one memory latency; grid (column tiles, splits).
constexpr int QV_ROWS = 64;
__global__ void __launch_bounds__(256) qr_vtc64_kernel(const double* __restrict__ V, int64_t ldv,
                                                       const double* __restrict__ C, int64_t ldc,
                                                       int jb, int64_t rows, int64_t nc,
                                                       double* __restrict__ part) {
  __shared__ double Vs[QV_ROWS][33];
  pdl_enter();
  __shared__ double Cs[QV_ROWS][33];
  const int64_t c0 = (int64_t)blockIdx.x * 32;
  const int s = blockIdx.y;
  const int64_t ib = (int64_t)s * QV_ROWS;
  const int nr = (int)std::min<int64_t>(QV_ROWS, rows - ib);
  const int tid = threadIdx.x;
  #pragma unroll
  for (int e = tid; e < QV_ROWS * 32; e += 256) {
    const int col = e / QV_ROWS, r = e % QV_ROWS;
    Vs[r][col] = (r < nr && col < jb) ? V[col * ldv + ib + r] : 0.0;
    Cs[r][col] = (r < nr && c0 + col < nc) ? C[(c0 + col) * ldc + ib + r] : 0.0;
  }
  __syncthreads();
  const int k = tid & 31, cq = (tid >> 5) * 4;
  double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
#pragma unroll 16
  for (int r = 0; r < QV_ROWS; ++r) {
    const double v = Vs[r][k];
    a0 = fma(v, Cs[r][cq], a0);
    a1 = fma(v, Cs[r][cq + 1], a1);
    a2 = fma(v, Cs[r][cq + 2], a2);
    a3 = fma(v, Cs[r][cq + 3], a3);
  }
  double* out = part + ((int64_t)s * nc + c0) * 32;
  if (c0 + cq < nc) out[(cq + 0) * 32 + k] = a0;
  if (c0 + cq + 1 < nc) out[(cq + 1) * 32 + k] = a1;
  if (c0 + cq + 2 < nc) out[(cq + 2) * 32 + k] = a2;
  if (c0 + cq + 3 < nc) out[(cq + 3) * 32 + k] = a3;
}

// Pass 2: W = sum of the S partials (fixed split order), W2 = T' W
// (T' = T^T when factoring, T when forming Q).  8 columns per CTA.
__global__ void __launch_bounds__(256) qr_reduce_tt_kernel(const double* __restrict__ part, int S,
                                                           int64_t nc, const double* __restrict__ T,
                                                           int jb, int transpose,
                                                           double* __restrict__ W2) {
  pdl_enter();
  // 2 columns per CTA; 4 groups of 32 threads split each column's S partials
  __shared__ double Tsm[32][33];
  __shared__ double Wg[2][4][32];
  __shared__ double Wsm[2][33];
  const int tid = threadIdx.x, k = tid & 31, g = (tid >> 5) & 3, cl = tid >> 7;
  const int64_t c = (int64_t)blockIdx.x * 2 + cl;
#pragma unroll
  for (int e = tid; e < 1024; e += 256) Tsm[e & 31][e >> 5] = T[e];  // Tsm[row][col]
  double w0 = 0.0, w1 = 0.0;
  if (c < nc) {
    int q = g;
#pragma unroll 4
    for (; q + 4 < S; q += 8) {
      w0 += part[((int64_t)q * nc + c) * 32 + k];
      w1 += part[((int64_t)(q + 4) * nc + c) * 32 + k];
    }
    if (q < S) w0 += part[((int64_t)q * nc + c) * 32 + k];
  }
  Wg[cl][g][k] = w0 + w1;
  __syncthreads();
  if (g == 0) Wsm[cl][k] = (Wg[cl][0][k] + Wg[cl][1][k]) + (Wg[cl][2][k] + Wg[cl][3][k]);
  __syncthreads();
  if (c >= nc || g != 0) return;
  double u0 = 0.0, u1 = 0.0;
  if (k < jb) {
    if (transpose) {
      int l = 0;
      for (; l + 1 <= k; l += 2) {
        u0 = fma(Tsm[l][k], Wsm[cl][l], u0);
        u1 = fma(Tsm[l + 1][k], Wsm[cl][l + 1], u1);
      }
      if (l <= k) u0 = fma(Tsm[l][k], Wsm[cl][l], u0);
    } else {
      int l = k;
      for (; l + 1 < jb; l += 2) {
        u0 = fma(Tsm[k][l], Wsm[cl][l], u0);
        u1 = fma(Tsm[k][l + 1], Wsm[cl][l + 1], u1);
      }
      if (l < jb) u0 = fma(Tsm[k][l], Wsm[cl][l], u0);
    }
  }
  W2[c * 32 + k] = u0 + u1;
}

// W2 = T' V^T C for the block reflector (rows x jb, rows x nc)
static int qr_wt(const double* V, int64_t ldv, const double* C, int64_t ldc, int jb, int64_t rows,
                 int64_t nc, const double* T, int transpose, double* W2, double* part,
                 int64_t part_cap, cudaStream_t st) {
  const int64_t S = (rows + QV_ROWS - 1) / QV_ROWS;
  SKL_REQUIRE(S * nc * 32 <= part_cap, SKL_ERR_INVALID, "qr: partial buffer too small");
  SKL_CUDA(launch_k(qr_vtc64_kernel, dim3((unsigned)((nc + 31) / 32), (unsigned)S), dim3(256), 0,
                    st, false, V, ldv, C, ldc, jb, rows, nc, part));
  SKL_CUDA(launch_k(qr_reduce_tt_kernel, dim3((unsigned)((nc + 1) / 2)), dim3(256), 0, st, true,
                    (const double*)part, (int)S, nc, T, jb, transpose, W2));
  return SKL_OK;
}

// cluster size for the panel factorisation of rows [j0, d)
static int panel_cluster(int64_t rows, int* rows_per) {
  int cl = 1;
  while (cl < QB_MAXCL && (rows + cl - 1) / cl > 256) cl *= 2;
  *rows_per = (int)((rows + cl - 1) / cl);
  return *rows_per <= QB_MAXROWS ? cl : 0;
}

// True when every panel of a d-row problem fits the cluster panel kernel.
bool qr_blocked_supported(int64_t d) {
  int rp = 0;
  return panel_cluster(d, &rp) > 0;
}

// Per-thread, per-device helper streams of the look-ahead factorisation: a
// high-priority stream for the critical path (panels) and a low-priority one
// for the bulk trailing updates, plus a pool of events.  Thread-local, so
// concurrent callers never share them (the C-ABI is reentrant).
struct QrStreams {
  cudaStream_t hi = nullptr, lo = nullptr;
  std::vector<cudaEvent_t> ev;
};

static int qr_streams(QrStreams** out, size_t nev) {
  static thread_local QrStreams per_dev[16];
  int dev = 0;
  SKL_CUDA(cudaGetDevice(&dev));
  SKL_REQUIRE(dev >= 0 && dev < 16, SKL_ERR_CUDA, "qr: device index %d out of range", dev);
  QrStreams& q = per_dev[dev];
  if (!q.hi) {
    int least = 0, greatest = 0;
    SKL_CUDA(cudaDeviceGetStreamPriorityRange(&least, &greatest));
    SKL_CUDA(cudaStreamCreateWithPriority(&q.hi, cudaStreamNonBlocking, greatest));
    SKL_CUDA(cudaStreamCreateWithPriority(&q.lo, cudaStreamNonBlocking, least));
  }
  while (q.ev.size() < nev) {
    cudaEvent_t e;
    SKL_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    q.ev.push_back(e);
  }
  *out = &q;
  return SKL_OK;
}

static int qr_launch_panel(double* M, int64_t ldm, int64_t d, int64_t j0, int jb, double* V,
                           double* Tblk, double* tau, double* beta, bool pdl, cudaStream_t st) {
  static std::once_flag attr_set[64];
  const int smem_max = (int)(QB_SMEM_EXTRA + QB_MAXROWS * QB_PLD) * (int)sizeof(double);
  const int arc = once_per_device(attr_set, [&]() -> int {
    SKL_CUDA(cudaFuncSetAttribute(qr_panel_cluster_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    SKL_CUDA(cudaFuncSetAttribute(qr_panel_cluster_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_max));
    SKL_CUDA(cudaFuncSetAttribute(qr_panel_reg_kernel<8>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    SKL_CUDA(cudaFuncSetAttribute(qr_panel_reg_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_max));
    SKL_CUDA(cudaFuncSetAttribute(qr_panel_reg_kernel<16>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    SKL_CUDA(cudaFuncSetAttribute(qr_panel_reg_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_max));
    SKL_CUDA(cudaFuncSetAttribute(qr_panel_reg_kernel<32>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    SKL_CUDA(cudaFuncSetAttribute(qr_panel_reg_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_max));
    return SKL_OK;
  });
  if (arc) return arc;
  static const bool smem_panel = env_flag("SKL_QR_SMEM_PANEL");
  // register panel: tail rows over up to 16 CTAs, <= 32 rows per warp
  static const int tail_rows = (int)env_int("SKL_QR_PANEL_ROWS", 128);
  const int64_t tail = d - j0 - jb;
  int cl2 = (int)std::min<int64_t>(QB_MAXCL, std::max<int64_t>(1, (tail + tail_rows - 1) / tail_rows));
  const int rows2 = (int)((tail + cl2 - 1) / cl2);
  const int rpw = (rows2 + QR_NW2 - 1) / QR_NW2;
  cudaLaunchConfig_t cfg = {};
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = (pdl && pdl_enabled()) ? 2 : 1;
  if (!smem_panel && rpw <= 32) {
    PanelParams pp{M, ldm, d, j0, jb, rows2, V, Tblk, tau, beta};
    cfg.gridDim = dim3(cl2);
    cfg.blockDim = dim3(QR_NT2);
    cfg.dynamicSmemBytes = (qr2_staging(rows2) + QR2_SMEM_EXTRA) * sizeof(double);
    attr[0].val.clusterDim.x = cl2;
    if (rpw <= 8)
      SKL_CUDA(cudaLaunchKernelEx(&cfg, qr_panel_reg_kernel<8>, pp));
    else if (rpw <= 16)
      SKL_CUDA(cudaLaunchKernelEx(&cfg, qr_panel_reg_kernel<16>, pp));
    else
      SKL_CUDA(cudaLaunchKernelEx(&cfg, qr_panel_reg_kernel<32>, pp));
  } else {
    int rows_per = 0;
    const int cl = panel_cluster(d - j0, &rows_per);
    SKL_REQUIRE(cl > 0, SKL_ERR_INVALID, "qr panel does not fit the cluster");
    PanelParams pp{M, ldm, d, j0, jb, rows_per, V, Tblk, tau, beta};
    cfg.gridDim = dim3(cl);
    cfg.blockDim = dim3(QB_NT);
    cfg.dynamicSmemBytes = (size_t)(rows_per * QB_PLD + QB_SMEM_EXTRA) * sizeof(double);
    attr[0].val.clusterDim.x = cl;
    SKL_CUDA(cudaLaunchKernelEx(&cfg, qr_panel_cluster_kernel, pp));
  }
  return SKL_OK;
}

// C (rows x nc, ld ldm) <- (I - V T V^T)^T C for the block reflector of the
// panel at column j0 (rows j0 .. d-1).
static int qr_apply_panel(double* M, int64_t ldm, int64_t d, int64_t j0, int jb, int64_t c0,
                          int64_t nc, const double* V, const double* Tblk, double* W2,
                          double* part, int64_t part_cap, cudaStream_t st) {
  if (nc <= 0) return SKL_OK;
  const int64_t rows = d - j0;
  int rc = qr_wt(V + j0 * ldm + j0, ldm, M + c0 * ldm + j0, ldm, jb, rows, nc, Tblk, 1, W2, part,
                 part_cap, st);
  if (rc) return rc;
  dim3 g((unsigned)((rows + 63) / 64), (unsigned)((nc + 63) / 64));
  SKL_CUDA(launch_k(qr_update_kernel, g, dim3(256), 0, st, true, M + c0 * ldm + j0, ldm,
                    (const double*)(V + j0 * ldm + j0), ldm, (const double*)W2, jb, rows, nc));
  return SKL_OK;
}

// Blocked factorisation of M (d x (n+1), ld ldm); fills tau, beta, V
// (explicit reflectors, ld ldm), T (per panel 32 x 32 blocks, n/32+1 of
// them).  The last column of M (Sb) is transformed into Q^T Sb.
//
// Look-ahead: panel k + 1 only needs its own 32 columns updated by panel k's
// reflectors, so the critical path is panel, small update of the next
// panel's columns, panel, ... on a high-priority stream, while the bulk
// trailing update of panel k (every column after panel k + 1, including Sb)
// runs concurrently on a low-priority stream.  Event k orders: panel k done
// -> bulk update k; bulk update k - 2 done -> small update before panel k.
// Each stream has its own W2 / partial scratch.
int qr_blocked_factor(double* M, int64_t ldm, int64_t d, int64_t n, double* tau, double* beta,
                      double* V, double* Tall, double* W, double* W2, double* part,
                      int64_t part_cap, double* W2b, double* partb, cudaStream_t st) {
  (void)W;
  const int64_t npan = (n + QB_NB - 1) / QB_NB;
  QrStreams* qs = nullptr;
  int rc = qr_streams(&qs, (size_t)(2 * npan + 3));
  if (rc) return rc;
  cudaEvent_t* E = qs->ev.data();            // [0, npan): panel k done
  cudaEvent_t* F = qs->ev.data() + npan;     // [npan, 2 npan): bulk update k done
  cudaEvent_t* X = qs->ev.data() + 2 * npan; // fork / join
  SKL_CUDA(cudaEventRecord(X[0], st));
  SKL_CUDA(cudaStreamWaitEvent(qs->hi, X[0], 0));
  SKL_CUDA(cudaStreamWaitEvent(qs->lo, X[0], 0));
  // From here on work is forked onto hi / lo: every exit path -- success or
  // an error return from a launch below -- joins both back into the
  // caller's stream, so the caller's cudaFreeAsync of the workspace is
  // ordered after everything that still uses it.
  struct Join {
    QrStreams* q;
    cudaStream_t st;
    cudaEvent_t a, b;
    ~Join() {
      cudaEventRecord(a, q->hi);
      cudaEventRecord(b, q->lo);
      cudaStreamWaitEvent(st, a, 0);
      cudaStreamWaitEvent(st, b, 0);
    }
  } join{qs, st, X[1], X[2]};
#ifdef SKL_QR_TIMELINE
  // instrumented build: timing events on both streams, printed per panel;
  // SKL_QR_SKIP bit 1 drops the bulk updates, bit 2 the next-panel updates
  // (wrong results: timing experiments only)
  static const int skip = (int)env_int("SKL_QR_SKIP", 0);
  std::vector<cudaEvent_t> tl(4 * npan + 1);
  for (auto& e : tl) cudaEventCreate(&e);
  cudaEventRecord(tl[4 * npan], qs->hi);
#define QR_TL(i, s) cudaEventRecord(tl[i], s)
#define QR_SKIP(b) (skip & (b))
#else
#define QR_TL(i, s) do {} while (0)
#define QR_SKIP(b) 0
#endif
  for (int64_t k = 0; k < npan; ++k) {
    const int64_t j0 = k * QB_NB;
    const int jb = (int)std::min<int64_t>(QB_NB, n - j0);
    QR_TL(4 * k, qs->hi);
    if (k > 0 && !QR_SKIP(2)) {
      // panel k's columns: reflectors 0 .. k-2 came with bulk update k-2,
      // reflector k-1 is applied here
      if (k >= 2) SKL_CUDA(cudaStreamWaitEvent(qs->hi, F[k - 2], 0));
      const int64_t p0 = j0 - QB_NB;
      rc = qr_apply_panel(M, ldm, d, p0, QB_NB, j0, jb, V, Tall + (k - 1) * 32 * 32, W2, part,
                          part_cap, qs->hi);
      if (rc) return rc;
    }
    QR_TL(4 * k + 1, qs->hi);
    // PDL only right after the next-panel update kernels on this stream
    rc = qr_launch_panel(M, ldm, d, j0, jb, V, Tall + k * 32 * 32, tau, beta,
                         k > 0 && !QR_SKIP(2), qs->hi);
    if (rc) return rc;
    QR_TL(4 * k + 2, qs->hi);
    SKL_CUDA(cudaEventRecord(E[k], qs->hi));
    // bulk update: every column after panel k + 1 (and Sb)
    const int64_t c0 = j0 + jb;
    const int64_t jb_next = std::min<int64_t>(QB_NB, std::max<int64_t>(0, n - c0));
    const int64_t cs = c0 + jb_next;
    SKL_CUDA(cudaStreamWaitEvent(qs->lo, E[k], 0));
    if (!QR_SKIP(1)) {
      rc = qr_apply_panel(M, ldm, d, j0, jb, cs, (n + 1) - cs, V, Tall + k * 32 * 32, W2b, partb,
                          part_cap, qs->lo);
      if (rc) return rc;
    }
    QR_TL(4 * k + 3, qs->lo);
    SKL_CUDA(cudaEventRecord(F[k], qs->lo));
  }
#ifdef SKL_QR_TIMELINE
  {
    cudaStreamSynchronize(qs->hi);
    cudaStreamSynchronize(qs->lo);
    float t_small = 0, t_panel = 0, t_end = 0;
    fprintf(stderr, "qr timeline d=%lld n=%lld skip=%d (us from start: small-update start, panel start, panel end, bulk end)\n",
            (long long)d, (long long)n, skip);
    for (int64_t k = 0; k < npan; ++k) {
      float a, b, c, e;
      cudaEventElapsedTime(&a, tl[4 * npan], tl[4 * k]);
      cudaEventElapsedTime(&b, tl[4 * npan], tl[4 * k + 1]);
      cudaEventElapsedTime(&c, tl[4 * npan], tl[4 * k + 2]);
      cudaEventElapsedTime(&e, tl[4 * npan], tl[4 * k + 3]);
      t_small += b - a;
      t_panel += c - b;
      t_end = std::max(t_end, std::max(c, e));
      if (k < 4 || k + 2 >= npan)
        fprintf(stderr, "  %3lld %8.1f %8.1f %8.1f %8.1f\n", (long long)k, a * 1e3, b * 1e3, c * 1e3, e * 1e3);
    }
    fprintf(stderr, "  sum small-update+wait %.1f us, sum panels %.1f us, end %.1f us\n", t_small * 1e3,
            t_panel * 1e3, t_end * 1e3);
    for (auto& e : tl) cudaEventDestroy(e);
  }
#endif
#ifdef SKL_QR_PROBE
  {
    unsigned long long h[12] = {}, z[12] = {};
    cudaStreamSynchronize(qs->hi);
    cudaStreamSynchronize(qs->lo);
    cudaMemcpyFromSymbol(h, g_qr_probe, sizeof(h));
    cudaMemcpyToSymbol(g_qr_probe, z, sizeof(z));
    fprintf(stderr, "qr panel probe d=%lld n=%lld (cycles, CTA 0 thread 0, all panels):",
            (long long)d, (long long)n);
    for (int i = 0; i < 12; ++i) fprintf(stderr, " %llu", h[i]);
    fprintf(stderr, "\n");
  }
#endif
  return SKL_OK;
}

// Q = H_0 ... H_{n-1} [I; 0] by applying the block reflectors backwards.
int qr_blocked_form_q(double* Q, int64_t ldq, int64_t d, int64_t n, const double* V, int64_t ldv,
                      const double* Tall, double* W, double* W2, double* part, int64_t part_cap,
                      cudaStream_t st) {
  for (int64_t j0 = ((n - 1) / QB_NB) * QB_NB; j0 >= 0; j0 -= QB_NB) {
    const int jb = (int)std::min<int64_t>(QB_NB, n - j0);
    const int64_t rows = d - j0, nc = n - j0;
    int rc = qr_wt(V + j0 * ldv + j0, ldv, Q + j0 * ldq + j0, ldq, jb, rows, nc,
                   Tall + (j0 / QB_NB) * 32 * 32, 0, W2, part, part_cap, st);
    if (rc) return rc;
    SKL_CUDA_LAUNCH();
    dim3 g((unsigned)((rows + 63) / 64), (unsigned)((nc + 63) / 64));
    qr_update_kernel<<<g, 256, 0, st>>>(Q + j0 * ldq + j0, ldq, V + j0 * ldv + j0, ldv, W2, jb,
                                        rows, nc);
    SKL_CUDA_LAUNCH();
  }
  return SKL_OK;
}

}  // namespace skl
