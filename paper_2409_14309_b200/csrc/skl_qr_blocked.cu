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

#include <algorithm>
#include <cmath>

#include "skl_common.h"

namespace skl {

constexpr int QB_NB = 32;        // panel width
constexpr int QB_PLD = 33;       // panel row stride in shared memory (conflict-free)
constexpr int QB_NT = 1024;      // threads per CTA (32 warps)
constexpr int QB_NW = QB_NT / 32;
constexpr int QB_MAXCL = 16;     // max cluster size (non-portable)
constexpr int QB_MAXROWS = 680;  // rows per CTA that fit in shared memory
// pub[2][64] + red[32][32] + gram[32][32] + allp[17][32] + gsum[32][32]
constexpr int QB_SMEM_EXTRA = 128 + 1024 + 1024 + (QB_MAXCL + 1) * 32 + 1024;

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
  extern __shared__ __align__(16) double qsm[];
  const uint32_t rank = cta_rank_in_cluster();
  const uint32_t ncta = gridDim.x;  // one cluster spans the grid
  double* P = qsm;                                  // [rows_per][32]
  double* pub = P + (size_t)p.rows_per * QB_PLD;    // [2][64]
  double* red = pub + 128;                          // [32][32]
  double* gram = red + 1024;                        // [32][32]
  double* allp = gram + 1024;                       // [QB_MAXCL + 1][32]
  double* gsum = allp + (QB_MAXCL + 1) * 32;        // [32][32]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t rbeg = p.j0 + (int64_t)rank * p.rows_per;
  const int nloc = (int)std::max<int64_t>(0, std::min<int64_t>(p.rows_per, p.d - rbeg));
  const int jb = p.jb;

  // load the panel slice (column-major source -> row-major smem)
  for (int idx = tid; idx < nloc * QB_NB; idx += QB_NT) {
    const int j = idx / nloc, i = idx % nloc;  // coalesced along rows
    P[i * QB_PLD + j] = j < jb ? p.M[(p.j0 + j) * p.ldm + rbeg + i] : 0.0;
  }
  __syncthreads();

  for (int k = 0; k < jb; ++k) {
    const int64_t g = p.j0 + k;
    const double* pubr = pub + (k & 1) * 64;
    double* pubw = pub + (k & 1) * 64;
    // partial sums s_j = sum_{i > g, local} P[i][k] * P[i][j]
    double s0 = 0.0;
    for (int i = warp; i < nloc; i += QB_NW)
      if (rbeg + i > g) s0 = fma(P[i * QB_PLD + k], P[i * QB_PLD + lane], s0);
    red[warp * 32 + lane] = s0;
    __syncthreads();
    if (warp == 0) {
      double t = 0.0;
#pragma unroll
      for (int w = 0; w < QB_NW; ++w) t += red[w * 32 + lane];
      pubw[lane] = t;
      const int64_t gl = g - rbeg;
      if (gl >= 0 && gl < nloc) pubw[32 + lane] = P[gl * QB_PLD + lane];
    }
    cluster_sync_all();
    // gather every CTA's partials (one remote load per thread), then every
    // thread sums them in fixed CTA order from local shared memory
    const uint32_t owner = (uint32_t)((g - p.j0) / p.rows_per);
    for (int e = tid; e < (int)ncta * 32; e += QB_NT) {
      const uint32_t q = (uint32_t)(e >> 5);
      allp[e] = ld_dsmem(pubr + (e & 31), q);
    }
    if (tid < 32) allp[QB_MAXCL * 32 + tid] = ld_dsmem(pubr + 32 + tid, owner);
    __syncthreads();
    double Sj = 0.0, Sk = 0.0;
    for (uint32_t q = 0; q < ncta; ++q) {
      Sj += allp[q * 32 + lane];
      Sk += allp[q * 32 + k];
    }
    const double alpha = allp[QB_MAXCL * 32 + k];
    const double pj = allp[QB_MAXCL * 32 + lane];
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
    const double wj = (lane > k && lane < jb) ? tau * (pj + scale * Sj) : 0.0;
    // update local rows below the pivot; column k becomes v
    for (int i = warp; i < nloc; i += QB_NW) {
      const int64_t gi = rbeg + i;
      if (gi > g) {
        const double v = scale * P[i * QB_PLD + k];
        if (lane == k)
          P[i * QB_PLD + k] = v;
        else if (lane > k)
          P[i * QB_PLD + lane] -= wj * v;
      } else if (gi == g) {
        if (lane == k)
          P[i * QB_PLD + k] = beta;
        else if (lane > k)
          P[i * QB_PLD + lane] -= wj;
      }
    }
    if (rank == 0 && tid == 0) {
      p.tau[g] = tau;
      p.beta[g] = beta;
    }
    __syncthreads();
  }

  // V^T V partials (explicit V: 1 at its pivot, 0 above) for T: lane b,
  // 32 register accumulators over a; warps split the rows, then reduce.
  for (int half = 0; half < 2; ++half) {
    double ga[16];
#pragma unroll
    for (int a = 0; a < 16; ++a) ga[a] = 0.0;
    for (int i = warp; i < nloc; i += QB_NW) {
      const int64_t rel = rbeg + i - p.j0;  // row index inside the panel
      const double vb = rel < lane ? 0.0 : (rel == lane ? 1.0 : P[i * QB_PLD + lane]);
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        const int a = half * 16 + q;
        const double va = rel < a ? 0.0 : (rel == a ? 1.0 : P[i * QB_PLD + a]);
        ga[q] = fma(va, vb, ga[q]);
      }
    }
    // fixed-order reduction over warps through shared memory
    for (int q = 0; q < 16; ++q) {
      const int a = half * 16 + q;
      red[warp * 32 + lane] = ga[q];
      __syncthreads();
      if (warp == 0) {
        double t = 0.0;
        for (int w = 0; w < QB_NW; ++w) t += red[w * 32 + lane];
        gram[a * QB_NB + lane] = (a < jb && lane < jb) ? t : 0.0;
      }
      __syncthreads();
    }
  }
  cluster_sync_all();
  if (rank == 0) {
    // G = sum of all CTAs' V^T V partials (parallel remote loads, fixed
    // CTA order), then dlarft: T[k][k] = tau_k,
    // T[0:k, k] = -tau_k * T[0:k, 0:k] * G[0:k, k]   (one warp)
    for (int e = tid; e < QB_NB * QB_NB; e += QB_NT) {
      double v = 0.0;
      if ((e / QB_NB) < (e % QB_NB))
        for (uint32_t q = 0; q < ncta; ++q) v += ld_dsmem(gram + e, q);
      gsum[e] = v;
    }
    __syncthreads();
    if (warp == 0) {
      double* T = p.T;
      for (int k = 0; k < jb; ++k) {
        const double tk = p.tau[p.j0 + k];
        double t = 0.0;
        if (lane < k) {
          for (int pp = lane; pp < k; ++pp) t = fma(T[pp * 32 + lane], gsum[pp * QB_NB + k], t);
          t = -tk * t;
        }
        __syncwarp();
        if (lane < k) T[k * 32 + lane] = t;
        if (lane == k) T[k * 32 + k] = tk;
        if (lane > k) T[k * 32 + lane] = 0.0;
        __syncwarp();
      }
    }
  }
  // write back the panel and the explicit V
  for (int idx = tid; idx < nloc * QB_NB; idx += QB_NT) {
    const int j = idx / nloc, i = idx % nloc;
    if (j >= jb) continue;
    const int64_t gi = rbeg + i, gj = p.j0 + j;
    const double val = P[i * QB_PLD + j];
    p.M[gj * p.ldm + gi] = val;
    p.V[gj * p.ldm + gi] = gi < gj ? 0.0 : (gi == gj ? 1.0 : val);
  }
  cluster_sync_all();  // keep shared memory alive for remote readers
}

// Partial W = V^T C over a row range: part[s][c][k] = sum_i V[i][k] C[i][c]
// for the rows of split s.  Grid (ceil(nc/32), S); one CTA = 32 columns.
__global__ void __launch_bounds__(256) qr_vtc_kernel(const double* V, int64_t ldv, const double* C,
                                                     int64_t ldc, int jb, int64_t rows, int64_t nc,
                                                     int S, double* part) {
  __shared__ double Vs[32][33];
  __shared__ double Cs[32][33];
  const int64_t c0 = (int64_t)blockIdx.x * 32;
  const int s = blockIdx.y;
  const int64_t ib = rows * s / S, ie = rows * (s + 1) / S;
  const int tid = threadIdx.x, k = tid & 31, cq = (tid >> 5) * 4;
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  for (int64_t i0 = ib; i0 < ie; i0 += 32) {
    for (int e = tid; e < 1024; e += 256) {
      const int col = e >> 5, r = e & 31;
      const int64_t i = i0 + r;
      Vs[r][col] = (i < ie && col < jb) ? V[col * ldv + i] : 0.0;
      Cs[r][col] = (i < ie && c0 + col < nc) ? C[(c0 + col) * ldc + i] : 0.0;
    }
    __syncthreads();
#pragma unroll 8
    for (int r = 0; r < 32; ++r) {
      const double v = Vs[r][k];
#pragma unroll
      for (int q = 0; q < 4; ++q) acc[q] = fma(v, Cs[r][cq + q], acc[q]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int q = 0; q < 4; ++q)
    if (c0 + cq + q < nc) part[((int64_t)s * nc + c0 + cq + q) * 32 + k] = acc[q];
}

// W[c][k] = sum_s part[s][c][k] in fixed split order
__global__ void qr_vtc_reduce_kernel(const double* part, int S, int64_t nc, double* W) {
  const int64_t total = nc * 32;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    double v = 0.0;
    for (int q = 0; q < S; ++q) v += part[(int64_t)q * total + idx];
    W[idx] = v;
  }
}

// W = V^T C for the block reflector (rows x jb times rows x nc)
static int qr_vtc(const double* V, int64_t ldv, const double* C, int64_t ldc, int jb, int64_t rows,
                  int64_t nc, double* W, double* part, int64_t part_cap, cudaStream_t st) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t tiles = (nc + 31) / 32;
  int64_t S = std::max<int64_t>(1, std::min<int64_t>(rows / 256, (2 * sms + tiles - 1) / tiles));
  S = std::min<int64_t>(S, part_cap / (nc * 32));
  S = std::max<int64_t>(S, 1);
  qr_vtc_kernel<<<dim3((unsigned)tiles, (unsigned)S), 256, 0, st>>>(V, ldv, C, ldc, jb, rows, nc,
                                                                    (int)S, part);
  SKL_CUDA_LAUNCH();
  const int64_t tot = nc * 32;
  qr_vtc_reduce_kernel<<<(int)std::min<int64_t>((tot + 255) / 256, 4096), 256, 0, st>>>(
      part, (int)S, nc, W);
  SKL_CUDA_LAUNCH();
  return SKL_OK;
}

// W2 = T^T W  (T upper, jb x jb, ld 32; W jb x nc, ld 32)
__global__ void qr_apply_tt_kernel(const double* T, const double* W, double* W2, int jb, int64_t nc,
                                   int transpose) {
  const int64_t total = (int64_t)jb * nc;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = idx / jb;
    const int k = (int)(idx % jb);
    double s = 0.0;
    if (transpose) {  // (T^T W)[k] = sum_{l <= k} T[l][k] W[l]
      for (int l = 0; l <= k; ++l) s = fma(T[k * 32 + l], W[c * 32 + l], s);
    } else {          // (T W)[k] = sum_{l >= k} T[k][l] W[l]
      for (int l = k; l < jb; ++l) s = fma(T[l * 32 + k], W[c * 32 + l], s);
    }
    W2[c * 32 + k] = s;
  }
}

// C[rows x nc] -= V[rows x jb] * W2[jb x nc]; 64 x 64 tiles, 4 x 4 per thread.
__global__ void __launch_bounds__(256) qr_update_kernel(double* C, int64_t ldc, const double* V,
                                                        int64_t ldv, const double* W2, int jb,
                                                        int64_t rows, int64_t nc) {
  __shared__ double Vs[32][64 + 1];
  __shared__ double Ws[32][64 + 1];
  const int64_t i0 = (int64_t)blockIdx.x * 64, c0 = (int64_t)blockIdx.y * 64;
  const int tid = threadIdx.x;
  for (int e = tid; e < 32 * 64; e += 256) {
    const int k = e / 64, r = e % 64;
    Vs[k][r] = (k < jb && i0 + r < rows) ? V[(int64_t)k * ldv + i0 + r] : 0.0;
    Ws[k][r] = (k < jb && c0 + r < nc) ? W2[(c0 + r) * 32 + k] : 0.0;
  }
  __syncthreads();
  const int tr = tid % 16, tc = tid / 16;  // rows tr + 16a, cols tc + 16b
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
      if (i < rows && c < nc) C[c * ldc + i] -= acc[a][b];
    }
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

// Blocked factorisation of M (d x (n+1), ld ldm); fills tau, beta, V
// (explicit reflectors, ld ldm), T (per panel 32 x 32 blocks, n/32+1 of
// them).  The last column of M (Sb) is transformed into Q^T Sb.
int qr_blocked_factor(double* M, int64_t ldm, int64_t d, int64_t n, double* tau, double* beta,
                      double* V, double* Tall, double* W, double* W2, double* part,
                      int64_t part_cap, cudaStream_t st) {
  static bool attr_set = false;
  if (!attr_set) {
    SKL_CUDA(cudaFuncSetAttribute(qr_panel_cluster_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    SKL_CUDA(cudaFuncSetAttribute(qr_panel_cluster_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)(QB_SMEM_EXTRA + QB_MAXROWS * QB_PLD) * (int)sizeof(double)));
    attr_set = true;
  }
  for (int64_t j0 = 0; j0 < n; j0 += QB_NB) {
    const int jb = (int)std::min<int64_t>(QB_NB, n - j0);
    int rows_per = 0;
    const int cl = panel_cluster(d - j0, &rows_per);
    SKL_REQUIRE(cl > 0, SKL_ERR_INVALID, "qr panel does not fit the cluster");
    PanelParams pp{M, ldm, d, j0, jb, rows_per, V, Tall + (j0 / QB_NB) * 32 * 32, tau, beta};
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cl);
    cfg.blockDim = dim3(QB_NT);
    cfg.dynamicSmemBytes = (size_t)(rows_per * QB_PLD + QB_SMEM_EXTRA) * sizeof(double);
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = cl;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    SKL_CUDA(cudaLaunchKernelEx(&cfg, qr_panel_cluster_kernel, pp));
    const int64_t c0 = j0 + jb;
    const int64_t nc = (n + 1) - c0;  // trailing columns incl. Sb
    if (nc <= 0) continue;
    const int64_t rows = d - j0;
    int rc = qr_vtc(V + j0 * ldm + j0, ldm, M + c0 * ldm + j0, ldm, jb, rows, nc, W, part,
                    part_cap, st);
    if (rc) return rc;
    const int64_t tot = (int64_t)jb * nc;
    qr_apply_tt_kernel<<<(int)std::min<int64_t>((tot + 255) / 256, 4096), 256, 0, st>>>(
        Tall + (j0 / QB_NB) * 32 * 32, W, W2, jb, nc, 1);
    SKL_CUDA_LAUNCH();
    dim3 g((unsigned)((rows + 63) / 64), (unsigned)((nc + 63) / 64));
    qr_update_kernel<<<g, 256, 0, st>>>(M + c0 * ldm + j0, ldm, V + j0 * ldm + j0, ldm, W2, jb,
                                        rows, nc);
    SKL_CUDA_LAUNCH();
  }
  return SKL_OK;
}

// Q = H_0 ... H_{n-1} [I; 0] by applying the block reflectors backwards.
int qr_blocked_form_q(double* Q, int64_t ldq, int64_t d, int64_t n, const double* V, int64_t ldv,
                      const double* Tall, double* W, double* W2, double* part, int64_t part_cap,
                      cudaStream_t st) {
  for (int64_t j0 = ((n - 1) / QB_NB) * QB_NB; j0 >= 0; j0 -= QB_NB) {
    const int jb = (int)std::min<int64_t>(QB_NB, n - j0);
    const int64_t rows = d - j0, nc = n - j0;
    int rc = qr_vtc(V + j0 * ldv + j0, ldv, Q + j0 * ldq + j0, ldq, jb, rows, nc, W, part,
                    part_cap, st);
    if (rc) return rc;
    const int64_t tot = (int64_t)jb * nc;
    qr_apply_tt_kernel<<<(int)std::min<int64_t>((tot + 255) / 256, 4096), 256, 0, st>>>(
        Tall + (j0 / QB_NB) * 32 * 32, W, W2, jb, nc, 0);
    SKL_CUDA_LAUNCH();
    dim3 g((unsigned)((rows + 63) / 64), (unsigned)((nc + 63) / 64));
    qr_update_kernel<<<g, 256, 0, st>>>(Q + j0 * ldq + j0, ldq, V + j0 * ldv + j0, ldv, W2, jb,
                                        rows, nc);
    SKL_CUDA_LAUNCH();
  }
  return SKL_OK;
}

}  // namespace skl
