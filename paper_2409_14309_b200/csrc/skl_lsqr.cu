// Device kernels of the preconditioned LSQR iteration (reference:
// /root/reference/pkg/src/sketchls/solvers.py:110-255 `lsqr`, driven by
// `sketch_and_precondition` :323-361).  Per iteration the reference does
//   u = A (R^-1 v) - alfa u;  beta = ||u||;  u /= beta
//   v = R^-T (A^T u) - beta v;  alfa = ||v||;  v /= alfa
//   x += (phi/rho) w;  w = v - (theta/rho) w;  ||x||
// Two products with A (HBM-bound) and two n x n triangular solves.  For
// dense A with n <= 256 both products share one pass (skl_lsqr_fused, below);
// otherwise the kernels fuse each step's vector work into the pass that
// produces it:
//   skl_lsqr_gemv_n : u_out = s * (A y) - alpha * u_in, and ||u_out||^2
//   skl_lsqr_gemv_t : u_n = u_raw / beta (written back), z = A^T u_n
//   skl_lsqr_trsv_t : v_out = R^-T z - beta v, and ||v_out||^2
//   skl_lsqr_trsv_n : v_n = v_raw / alfa (written back), y = R^-1 v_n
//   skl_lsqr_xw     : x += c1 w;  w = v_n + c2 w;  ||x||^2
// Every reduction is two-level with a fixed order (the last CTA to finish
// folds the per-CTA partials in index order), so results are deterministic.
// The scalar recurrence (Givens rotations, stopping tests) stays on the host
// exactly as the reference writes it.
#include <cuda_runtime.h>

#include <algorithm>

#include "skl_common.h"
#include "skl_ptx.cuh"

namespace skl {

constexpr int LQ_NT = 256;

// Device-driven LSQR iteration (skl_lsqr_*_dev): the scalar state the host
// loop would otherwise read back three times per iteration, as doubles.
enum {
  LS_BETA2 = 0,   // ||r||^2 of the step's pass (written by the fused pass)
  LS_ALFA2 = 1,   // ||v||^2 (written by the transposed solve)
  LS_XNORM2 = 2,  // ||x||^2 (written by the x/w update)
  LS_ALFA = 3,    // alfa of the current step (the recurrence's input / output)
  LS_BETA = 4,
  LS_RHOBAR = 5,
  LS_PHIBAR = 6,
  LS_ANORM = 7,
  LS_C1 = 8,      // phi / rho
  LS_C2 = 9,      // -theta / rho
  LS_RNORM = 10,
  LS_ARNORM = 11,
  LS_BPREV = 12,  // beta the next pass divides r by (1 when beta == 0)
  LS_STATE = 16
};
constexpr int LQ_YMAX = 8192;  // y staged in shared memory up to this n
constexpr int LQ_TC = 16;      // columns per CTA in the transposed product

__device__ __forceinline__ double lq_block_sum(double v, double* red) {
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
  }
  return s;  // valid in thread 0
}

// The last CTA to arrive folds part[0..nparts) in index order into *out and
// resets the counter for the next launch.
__device__ __forceinline__ void lq_finish(const double* part, int nparts, double* out,
                                          unsigned int* counter) {
  __shared__ bool last;
  __threadfence();
  if (threadIdx.x == 0) last = atomicAdd(counter, 1u) == (unsigned)(nparts - 1);
  __syncthreads();
  if (!last) return;
  __threadfence();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int i = 0; i < nparts; ++i) s += ((volatile const double*)part)[i];
    *out = s;
    *counter = 0u;
  }
}

// u_out = s * (A y) - alpha * u_in (u_in may be null), ||u_out||^2.
// Column-major A; each thread owns two adjacent rows, the columns are folded
// in ascending order with FMA (dgemv 'N' axpy order).  A null: u_out =
// -alpha * u_in.
__global__ void __launch_bounds__(LQ_NT) lsqr_gemv_n_kernel(
    const double* __restrict__ A, int64_t m, int64_t n, int64_t lda, const double* __restrict__ y,
    double s, double alpha, const double* __restrict__ u_in, double* __restrict__ u_out,
    double* part, double* norm2, unsigned int* counter) {
  extern __shared__ double ys[];
  __shared__ double red[32];
  const bool stage = A && n <= LQ_YMAX;
  if (stage)
    for (int64_t c = threadIdx.x; c < n; c += LQ_NT) ys[c] = y[c];
  __syncthreads();
  const double* yv = stage ? ys : y;
  double ss = 0.0;
  const int64_t pairs = (m + 1) / 2;
  for (int64_t pr = blockIdx.x * (int64_t)LQ_NT + threadIdx.x; pr < pairs;
       pr += (int64_t)gridDim.x * LQ_NT) {
    const int64_t i = 2 * pr;
    double a0 = 0.0, a1 = 0.0;
    if (A) {
      if (i + 1 < m) {
        const double* row = A + i;
        int64_t c = 0;
        for (; c + 8 <= n; c += 8) {
          double2 v[8];
#pragma unroll
          for (int q = 0; q < 8; ++q)
            v[q] = __ldcs(reinterpret_cast<const double2*>(row + (c + q) * lda));
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            a0 = fma(v[q].x, yv[c + q], a0);
            a1 = fma(v[q].y, yv[c + q], a1);
          }
        }
        for (; c < n; ++c) {
          const double2 v = __ldcs(reinterpret_cast<const double2*>(row + c * lda));
          a0 = fma(v.x, yv[c], a0);
          a1 = fma(v.y, yv[c], a1);
        }
      } else {
        for (int64_t c = 0; c < n; ++c) a0 = fma(A[i + c * lda], yv[c], a0);
      }
    }
    const double r0 = s * a0 - (u_in ? alpha * u_in[i] : 0.0);
    u_out[i] = r0;
    ss = fma(r0, r0, ss);
    if (i + 1 < m) {
      const double r1 = s * a1 - (u_in ? alpha * u_in[i + 1] : 0.0);
      u_out[i + 1] = r1;
      ss = fma(r1, r1, ss);
    }
  }
  const double t = lq_block_sum(ss, red);
  if (threadIdx.x == 0) part[blockIdx.x] = t;
  lq_finish(part, gridDim.x, norm2, counter);
}

// u_n = u_raw / beta, once per element (the division is the reference's
// `u /= beta`; doing it here keeps it out of the per-column-group loop).
__global__ void lsqr_scale_kernel(const double* __restrict__ u_raw, double beta, int64_t m,
                                  double* __restrict__ u_n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x)
    u_n[i] = u_raw[i] / beta;
}

// z[c] = sum_i A[i, c] u_n[i].  Grid (column groups of LQ_TC, row chunks);
// per CTA the chunk's u_n is loaded once per row for the group's columns;
// partial dots are folded over the chunks in fixed order by the last CTA of
// each column group.
__global__ void __launch_bounds__(LQ_NT) lsqr_gemv_t_kernel(
    const double* __restrict__ A, int64_t m, int64_t n, int64_t lda, const double* u_n,
    int64_t rows_per, double* __restrict__ part, double* __restrict__ z,
    unsigned int* counters) {
  __shared__ double red[32];
  __shared__ double sums[LQ_TC];
  __shared__ bool last;
  const int64_t g = blockIdx.x, rc = blockIdx.y, nrc = gridDim.y;
  const int64_t c0 = g * LQ_TC;
  const int tc = (int)min((int64_t)LQ_TC, n - c0);
  const int64_t r0 = rc * rows_per, r1 = min(m, r0 + rows_per);
  // each thread takes row pairs (16-byte loads of A and u_n); rows_per is a
  // multiple of 2 * LQ_NT, so only the last chunk can end mid-pair
  double acc[LQ_TC];
#pragma unroll
  for (int q = 0; q < LQ_TC; ++q) acc[q] = 0.0;
#pragma unroll 2
  for (int64_t i = r0 + 2 * threadIdx.x; i < r1; i += 2 * LQ_NT) {
    if (i + 1 < r1) {
      const double2 un = *reinterpret_cast<const double2*>(u_n + i);
      if (A) {
        double2 av[LQ_TC];
#pragma unroll
        for (int q = 0; q < LQ_TC; ++q)
          av[q] = q < tc ? __ldcs(reinterpret_cast<const double2*>(A + (c0 + q) * lda + i))
                         : make_double2(0.0, 0.0);
#pragma unroll
        for (int q = 0; q < LQ_TC; ++q) acc[q] = fma(av[q].y, un.y, fma(av[q].x, un.x, acc[q]));
      }
    } else {
      const double un = u_n[i];
      if (A) {
#pragma unroll
        for (int q = 0; q < LQ_TC; ++q)
          if (q < tc) acc[q] = fma(A[(c0 + q) * lda + i], un, acc[q]);
      }
    }
  }
#pragma unroll
  for (int q = 0; q < LQ_TC; ++q) {
    const double t = lq_block_sum(acc[q], red);
    if (threadIdx.x == 0) sums[q] = t;
  }
  __syncthreads();
  if (threadIdx.x < LQ_TC) part[(g * nrc + rc) * LQ_TC + threadIdx.x] = sums[threadIdx.x];
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(&counters[g], 1u) == (unsigned)(nrc - 1);
  __syncthreads();
  if (!last) return;
  __threadfence();
  if (threadIdx.x < tc) {
    double s = 0.0;
    for (int64_t q = 0; q < nrc; ++q)
      s += ((volatile const double*)part)[(g * nrc + q) * LQ_TC + threadIdx.x];
    z[c0 + threadIdx.x] = s;
  }
  if (threadIdx.x == 0) counters[g] = 0u;
}

// ---- one pass over A per iteration (n <= 256) ----------------------------
// The reference's two products of one LSQR step share a pass over A:
//   u     = u_raw_prev / beta_prev                 (the previous `u /= beta`)
//   r     = s * (A y) - alpha * u ; ||r||^2         (the next u_raw)
//   z     = (A^T r) / sqrt(||r||^2)                 (= A^T (r / beta))
// A CTA takes 64-row blocks; warp g owns columns g, g+8, ... (NC of them)
// and lane l rows 2l, 2l+1 of the block.  Phase 1 folds each row's dot
// product over the warp's columns, the eight warp partials are added in
// warp order; phase 2 multiplies the same values, still in registers, by
// the block's r, and every lane keeps per-column partial sums of A^T r in
// registers across all of its CTA's blocks.  The per-CTA partials are folded
// in CTA order by the last CTA, so the result is deterministic; the
// rounding differs from the two-pass kernels only in the summation order of
// the products and in dividing A^T r (instead of r) by beta.
constexpr int LF_RB = 64;  // rows per block
template <int NC>
__global__ void __launch_bounds__(LQ_NT) lsqr_fused_kernel(
    const double* __restrict__ A, int64_t m, int64_t n, int64_t lda, const double* __restrict__ y,
    double s, double alpha, const double* __restrict__ r_prev, double beta_prev,
    double* __restrict__ r_out, double* __restrict__ zpart, double* __restrict__ npart,
    double* __restrict__ z, double* __restrict__ norm2, unsigned int* counter,
    const double* __restrict__ dscal) {
  pdl_enter();  // lets the step kernel after it launch early (launch_k)
  if (dscal) {  // device-driven iteration: alfa and beta_prev from the recurrence state
    alpha = dscal[LS_ALFA];
    beta_prev = dscal[LS_BPREV];
  }
  __shared__ double ys[8 * NC];
  __shared__ double pdot[2][8][LF_RB];  // by block parity: one barrier less per block
  __shared__ double rs[2][LF_RB];
  __shared__ double red[32];
  __shared__ bool last;
  const int tid = threadIdx.x, lane = tid & 31, g = tid >> 5;
  for (int c = tid; c < 8 * NC; c += LQ_NT) ys[c] = c < n ? y[c] : 0.0;
  double zacc[NC];
#pragma unroll
  for (int q = 0; q < NC; ++q) zacc[q] = 0.0;
  double ss = 0.0;
  __syncthreads();
  const int64_t nblk = (m + LF_RB - 1) / LF_RB;
  int par = 0;
  for (int64_t blk = blockIdx.x; blk < nblk; blk += gridDim.x, par ^= 1) {
    const int64_t i0 = blk * LF_RB + 2 * lane;
    const bool full = i0 + 1 < m;
    // the block's r_prev entries are loaded with A (not after the barrier:
    // that would put a second memory latency on every block)
    double rp = 0.0;
    if (tid < LF_RB && r_prev && blk * LF_RB + tid < m) rp = __ldcs(r_prev + blk * LF_RB + tid);
    // the block's A values stay in registers for both phases: all NC loads
    // are in flight at once and nothing is read twice
    double2 v[NC];
#pragma unroll
    for (int q = 0; q < NC; ++q) {
      const int c = g + 8 * q;
      v[q] = make_double2(0.0, 0.0);
      if (c < n) {
        if (full) {
          v[q] = __ldcs(reinterpret_cast<const double2*>(A + c * lda + i0));
        } else if (i0 < m) {
          v[q].x = A[c * lda + i0];
        }
      }
    }
    double a0 = 0.0, a1 = 0.0;
#pragma unroll
    for (int q = 0; q < NC; ++q) {
      const int c = g + 8 * q;
      if (c < n) {
        a0 = fma(v[q].x, ys[c], a0);
        a1 = fma(v[q].y, ys[c], a1);
      }
    }
    pdot[par][g][2 * lane] = a0;
    pdot[par][g][2 * lane + 1] = a1;
    __syncthreads();
    if (tid < LF_RB) {
      const int64_t i = blk * LF_RB + tid;
      double r = 0.0;
      if (i < m) {
        double dot = 0.0;
#pragma unroll
        for (int w = 0; w < 8; ++w) dot += pdot[par][w][tid];
        r = s * dot - (r_prev ? alpha * (rp / beta_prev) : 0.0);
        r_out[i] = r;
        ss = fma(r, r, ss);
      }
      rs[par][tid] = r;
    }
    __syncthreads();
    const double r0 = rs[par][2 * lane], r1 = rs[par][2 * lane + 1];
#pragma unroll
    for (int q = 0; q < NC; ++q) zacc[q] = fma(v[q].y, r1, fma(v[q].x, r0, zacc[q]));
  }
  // per-CTA partials: column sums over the lanes, the norm over the CTA
#pragma unroll
  for (int q = 0; q < NC; ++q) {
    double t = zacc[q];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    const int c = g + 8 * q;
    if (lane == 0 && c < n) zpart[(int64_t)blockIdx.x * n + c] = t;
  }
  const double tn = lq_block_sum(ss, red);
  if (tid == 0) npart[blockIdx.x] = tn;
  __threadfence();
  __syncthreads();
  if (tid == 0) last = atomicAdd(counter, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  __shared__ double nb;
  // fixed-order folds; loads are batched (L2, bypassing L1) so that their
  // latency is paid once per batch, not once per partial
  constexpr int FB = 16;
  if (tid == 0) {
    double sn = 0.0;
    for (unsigned b0 = 0; b0 < gridDim.x; b0 += FB) {
      double t[FB];
#pragma unroll
      for (int q = 0; q < FB; ++q) t[q] = b0 + q < gridDim.x ? __ldcg(npart + b0 + q) : 0.0;
#pragma unroll
      for (int q = 0; q < FB; ++q)
        if (b0 + q < gridDim.x) sn += t[q];
    }
    *norm2 = sn;
    nb = sqrt(sn);
    *counter = 0u;
  }
  __syncthreads();
  const double beta = nb;
  for (int c = tid; c < n; c += LQ_NT) {
    double sz = 0.0;
    for (unsigned b0 = 0; b0 < gridDim.x; b0 += FB) {
      double t[FB];
#pragma unroll
      for (int q = 0; q < FB; ++q)
        t[q] = b0 + q < gridDim.x ? __ldcg(zpart + (int64_t)(b0 + q) * n + c) : 0.0;
#pragma unroll
      for (int q = 0; q < FB; ++q)
        if (b0 + q < gridDim.x) sz += t[q];
    }
    z[c] = beta > 0.0 ? sz / beta : 0.0;
  }
}

// The same pass with the blocks of A streamed into shared memory by
// cp.async, two 32-row blocks in flight: the register version above keeps a
// 64-row block in registers (236 registers, one CTA per SM), so no load is
// in flight while a block is folded, and the pass ran at ~66 % of HBM.  Here
// block b+1 streams in while block b is folded from shared memory (lane l =
// row l, warp g = columns g, g+8, ...; the values stay in registers between
// the two products, as above).  Same operations in the same order per row
// and column as the register kernel with one row per lane.
constexpr int LF2_RB = 32;  // rows per block
__device__ __forceinline__ void lq_cp_async16(void* smem, const void* gmem, int src_bytes) {
  const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(gmem), "r"(src_bytes)
               : "memory");
}
template <int NC, int ST>
__global__ void __launch_bounds__(LQ_NT) lsqr_fused_async_kernel(
    const double* __restrict__ A, int64_t m, int64_t n, int64_t lda, const double* __restrict__ y,
    double s, double alpha, const double* __restrict__ r_prev, double beta_prev,
    double* __restrict__ r_out, double* __restrict__ zpart, double* __restrict__ npart,
    double* __restrict__ z, double* __restrict__ norm2, unsigned int* counter,
    const double* __restrict__ dscal) {
  pdl_enter();
  if (dscal) {
    alpha = dscal[LS_ALFA];
    beta_prev = dscal[LS_BPREV];
  }
  constexpr int NCOL = 8 * NC;              // columns held by the CTA (>= n)
  constexpr int BUF = NCOL * LF2_RB;        // doubles per block buffer, [col][row]
  constexpr int CH = BUF / 2;               // 16-byte chunks per block
  extern __shared__ __align__(16) double abuf[];  // [ST][NCOL][LF2_RB] ring
  __shared__ double ys[NCOL];
  __shared__ double pdot[8][LF2_RB];
  __shared__ double rs[LF2_RB];
  __shared__ double red[32];
  __shared__ bool last;
  const int tid = threadIdx.x, lane = tid & 31, g = tid >> 5;
  for (int c = tid; c < NCOL; c += LQ_NT) ys[c] = c < n ? y[c] : 0.0;
  const int64_t nblk = (m + LF2_RB - 1) / LF2_RB;
  auto issue = [&](int64_t blk, int slot) {
    if (blk < nblk) {
      const int64_t r0 = blk * LF2_RB;
      double* dst = abuf + slot * BUF;
#pragma unroll 4
      for (int ch = tid; ch < CH; ch += LQ_NT) {
        const int c = ch / (LF2_RB / 2), r = (ch % (LF2_RB / 2)) * 2;
        const int64_t i = r0 + r;
        const int bytes = (c < n && i < m) ? (int)(min((int64_t)2, m - i) * 8) : 0;
        lq_cp_async16(dst + c * LF2_RB + r, bytes ? A + c * lda + i : A, bytes);
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  double zacc[NC];
#pragma unroll
  for (int q = 0; q < NC; ++q) zacc[q] = 0.0;
  double ss = 0.0;
#pragma unroll
  for (int k = 0; k < ST - 1; ++k) issue(blockIdx.x + (int64_t)k * gridDim.x, k);
  int slot = 0;
  for (int64_t blk = blockIdx.x; blk < nblk; blk += gridDim.x) {
    double rp = 0.0;
    if (tid < LF2_RB && r_prev && blk * LF2_RB + tid < m) rp = __ldcs(r_prev + blk * LF2_RB + tid);
    asm volatile("cp.async.wait_group %0;" ::"n"(ST - 2) : "memory");
    __syncthreads();  // block blk has landed for every thread; the previous slot is free
    // ST - 1 blocks stay in flight while this one is folded
    issue(blk + (int64_t)(ST - 1) * gridDim.x, slot == 0 ? ST - 1 : slot - 1);
    const double* b = abuf + slot * BUF;
    double v[NC];
#pragma unroll
    for (int q = 0; q < NC; ++q) v[q] = b[(g + 8 * q) * LF2_RB + lane];
    double a = 0.0;
#pragma unroll
    for (int q = 0; q < NC; ++q) {
      const int c = g + 8 * q;
      if (c < n) a = fma(v[q], ys[c], a);
    }
    pdot[g][lane] = a;
    __syncthreads();
    if (tid < LF2_RB) {
      const int64_t i = blk * LF2_RB + tid;
      double r = 0.0;
      if (i < m) {
        double dot = 0.0;
#pragma unroll
        for (int w = 0; w < 8; ++w) dot += pdot[w][tid];
        r = s * dot - (r_prev ? alpha * (rp / beta_prev) : 0.0);
        r_out[i] = r;
        ss = fma(r, r, ss);
      }
      rs[tid] = r;
    }
    __syncthreads();  // rs ready
    const double r0 = rs[lane];
#pragma unroll
    for (int q = 0; q < NC; ++q) zacc[q] = fma(v[q], r0, zacc[q]);
    slot = slot == ST - 1 ? 0 : slot + 1;
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
#pragma unroll
  for (int q = 0; q < NC; ++q) {
    double t = zacc[q];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    const int c = g + 8 * q;
    if (lane == 0 && c < n) zpart[(int64_t)blockIdx.x * n + c] = t;
  }
  const double tn = lq_block_sum(ss, red);
  if (tid == 0) npart[blockIdx.x] = tn;
  __threadfence();
  __syncthreads();
  if (tid == 0) last = atomicAdd(counter, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  __shared__ double nb;
  constexpr int FB = 16;
  if (tid == 0) {
    double sn = 0.0;
    for (unsigned b0 = 0; b0 < gridDim.x; b0 += FB) {
      double t[FB];
#pragma unroll
      for (int q = 0; q < FB; ++q) t[q] = b0 + q < gridDim.x ? __ldcg(npart + b0 + q) : 0.0;
#pragma unroll
      for (int q = 0; q < FB; ++q)
        if (b0 + q < gridDim.x) sn += t[q];
    }
    *norm2 = sn;
    nb = sqrt(sn);
    *counter = 0u;
  }
  __syncthreads();
  const double beta = nb;
  for (int c = tid; c < n; c += LQ_NT) {
    double sz = 0.0;
    for (unsigned b0 = 0; b0 < gridDim.x; b0 += FB) {
      double t[FB];
#pragma unroll
      for (int q = 0; q < FB; ++q)
        t[q] = b0 + q < gridDim.x ? __ldcg(zpart + (int64_t)(b0 + q) * n + c) : 0.0;
#pragma unroll
      for (int q = 0; q < FB; ++q)
        if (b0 + q < gridDim.x) sz += t[q];
    }
    z[c] = beta > 0.0 ? sz / beta : 0.0;
  }
}

// ---- CSR operands -------------------------------------------------------
// u_out = s * (A y) - alpha * u_in, ||u_out||^2 for CSR A: one row per
// thread, the row's nonzeros folded in stored order from 0 (csr_matvec).
__global__ void __launch_bounds__(LQ_NT) lsqr_spmv_kernel(
    const int64_t* __restrict__ indptr, const int64_t* __restrict__ indices,
    const double* __restrict__ values, int64_t m, const double* __restrict__ y, double s,
    double alpha, const double* __restrict__ u_in, double* __restrict__ u_out, double* part,
    double* norm2, unsigned int* counter) {
  __shared__ double red[32];
  double ss = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)LQ_NT + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * LQ_NT) {
    double a = 0.0;
    const int64_t p1 = indptr[i + 1];
    for (int64_t p = indptr[i]; p < p1; ++p) a = fma(values[p], y[indices[p]], a);
    const double r = s * a - (u_in ? alpha * u_in[i] : 0.0);
    u_out[i] = r;
    ss = fma(r, r, ss);
  }
  const double t = lq_block_sum(ss, red);
  if (threadIdx.x == 0) part[blockIdx.x] = t;
  lq_finish(part, gridDim.x, norm2, counter);
}

// z[c] = sum over column c of A (CSC, rows ascending) of a_ic u_n[i]: one
// warp per column, lanes stride the column, fixed shuffle-tree reduction.
__global__ void __launch_bounds__(LQ_NT) lsqr_csc_t_kernel(const int64_t* __restrict__ colptr,
                                                           const int32_t* __restrict__ rowidx,
                                                           const double* __restrict__ cval,
                                                           int64_t n, const double* __restrict__ u_n,
                                                           double* __restrict__ z) {
  const int lane = threadIdx.x & 31;
  for (int64_t c = (blockIdx.x * (int64_t)LQ_NT + threadIdx.x) >> 5; c < n;
       c += ((int64_t)gridDim.x * LQ_NT) >> 5) {
    double t = 0.0;
    const int64_t p1 = colptr[c + 1];
    for (int64_t p = colptr[c] + lane; p < p1; p += 32) t = fma(cval[p], u_n[rowidx[p]], t);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    if (lane == 0) z[c] = t;
  }
}

// One-CTA triangular solves with the explicit n x n upper R (column-major,
// ld ldr), 32-row blocks.  The off-diagonal part of a block is 32 dot
// products (warp per row pair, lanes over the inner index, shuffle
// reduction); the 32 x 32 diagonal block is solved by warp 0 with the block
// in registers and x broadcast by shuffles, dividing by R_ii as dtrtrs does.
constexpr int LT_NT = 512;

// x <- R^-T x  (forward substitution with L = R^T)
// Rinv (optional): the inverted 32 x 32 diagonal blocks of R
// (lsqr_trinv_kernel; block b covers rows [n - 32(b+1), n - 32b), clipped at
// 0, row-major): the block step becomes one 32-term product instead of 32
// dependent divide-and-update steps.  Without it the substitution keeps
// dtrsv's division order.
__device__ void lq_solve_t(const double* __restrict__ R, int64_t ldr, int n, double* xs,
                           const double* __restrict__ Rinv = nullptr) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // with Rinv the blocks align with the inverses (from the bottom, the top
  // one partial); without, from the top as dtrsv's column sweep
  const int first = (Rinv && n % 32) ? n % 32 : 32;
  for (int lo = 0; lo < n; lo += (lo == 0 ? first : 32)) {
    const int w = min(lo == 0 ? first : 32, n - lo);
    // xs[lo + r] -= sum_{j < lo} R[j][lo + r] xs[j]
    for (int r = warp; r < w; r += LT_NT / 32) {
      const double* col = R + (int64_t)(lo + r) * ldr;
      double t = 0.0;
      for (int j = lane; j < lo; j += 32) t = fma(col[j], xs[j], t);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
      if (lane == 0) xs[lo + r] -= t;
    }
    __syncthreads();
    if (Rinv && warp == 0) {
      // x_b = Rinv_b^T y_b (lane r: column r of Rinv_b)
      // (a partial top block occupies the w x w top-left corner of its slot)
      const double* Ri = Rinv + (int64_t)((n - lo - w) / 32) * 1024;
      double a0 = 0.0, a1 = 0.0;
#pragma unroll
      for (int j = 0; j < 32; j += 2) {
        const double y0 = (j < w) ? xs[lo + j] : 0.0;
        const double y1 = (j + 1 < w) ? xs[lo + j + 1] : 0.0;
        a0 = fma((j < w && lane < w) ? Ri[j * 32 + lane] : 0.0, y0, a0);
        a1 = fma((j + 1 < w && lane < w) ? Ri[(j + 1) * 32 + lane] : 0.0, y1, a1);
      }
      __syncwarp();
      if (lane < w) xs[lo + lane] = a0 + a1;
    } else if (warp == 0) {
      // lane r holds column lo + r: Rc[j] = R[lo + j][lo + r] (j < r), diag
      double Rc[32];
#pragma unroll
      for (int j = 0; j < 32; ++j)
        Rc[j] = (lane < w && j < lane) ? R[(int64_t)(lo + lane) * ldr + lo + j] : 0.0;
      const double dg = lane < w ? R[(int64_t)(lo + lane) * ldr + lo + lane] : 1.0;
      double br = lane < w ? xs[lo + lane] : 0.0;
      double xr = 0.0;
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        if (j < w) {
          if (lane == j) xr = br / dg;
          const double xj = __shfl_sync(0xffffffffu, xr, j);
          br = fma(-Rc[j], xj, br);  // Rc[j] = 0 unless j < lane
        }
      }
      if (lane < w) xs[lo + lane] = xr;
    }
    __syncthreads();
  }
}

// x <- R^-1 x  (backward substitution, dtrsv 'U','N' column order per block)
__device__ void lq_solve_n(const double* __restrict__ R, int64_t ldr, int n, double* xs,
                           const double* __restrict__ Rinv = nullptr) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  __shared__ double xb[32];
  __shared__ double Rsm[32][33];  // Rinv_b staged by coalesced rows (padded: conflict-free)
  for (int hi = n; hi > 0; hi -= 32) {
    const int lo = max(0, hi - 32), w = hi - lo;
    if (Rinv && warp == 0) {
      // x_b = Rinv_b y_b (lane r: row r of Rinv_b).  Rinv_b is row-major, so
      // lane r reading its row directly would touch 32 sectors per load; the
      // block comes in by rows (32 coalesced loads in flight) instead.
      const double* Ri = Rinv + (int64_t)((n - hi) / 32) * 1024;
#pragma unroll
      for (int j = 0; j < 32; ++j) Rsm[j][lane] = Ri[j * 32 + lane];
      __syncwarp();
      double a0 = 0.0, a1 = 0.0;
#pragma unroll
      for (int j = 0; j < 32; j += 2) {
        const double y0 = (j < w) ? xs[lo + j] : 0.0;
        const double y1 = (j + 1 < w) ? xs[lo + j + 1] : 0.0;
        a0 = fma((j < w && lane < w) ? Rsm[lane][j] : 0.0, y0, a0);
        a1 = fma((j + 1 < w && lane < w) ? Rsm[lane][j + 1] : 0.0, y1, a1);
      }
      __syncwarp();
      if (lane < w) {
        xs[lo + lane] = a0 + a1;
        xb[lane] = a0 + a1;
      }
    } else if (warp == 0) {
      // lane r holds row lo + r: Rr[j] = R[lo + r][lo + j] (j > r)
      double Rr[32];
#pragma unroll
      for (int j = 0; j < 32; ++j)
        Rr[j] = (lane < w && j > lane && j < w) ? R[(int64_t)(lo + j) * ldr + lo + lane] : 0.0;
      const double dg = lane < w ? R[(int64_t)(lo + lane) * ldr + lo + lane] : 1.0;
      double yr = lane < w ? xs[lo + lane] : 0.0;
      double xr = 0.0;
#pragma unroll
      for (int j = 31; j >= 0; --j) {
        if (j < w) {
          if (lane == j) xr = yr / dg;
          const double xj = __shfl_sync(0xffffffffu, xr, j);
          yr = fma(-Rr[j], xj, yr);
        }
      }
      if (lane < w) {
        xs[lo + lane] = xr;
        xb[lane] = xr;
      }
    }
    __syncthreads();
    for (int i = tid; i < lo; i += LT_NT) {
      double t0 = 0.0, t1 = 0.0;
      int j = 0;
      for (; j + 1 < w; j += 2) {
        t0 = fma(R[(int64_t)(lo + j) * ldr + i], xb[j], t0);
        t1 = fma(R[(int64_t)(lo + j + 1) * ldr + i], xb[j + 1], t1);
      }
      if (j < w) t0 = fma(R[(int64_t)(lo + j) * ldr + i], xb[j], t0);
      xs[i] -= t0 + t1;
    }
    __syncthreads();
  }
}

// v_out = R^-T z - beta v_prev (R null: identity), ||v_out||^2.
// The inverted 32 x 32 diagonal blocks of an explicit upper-triangular R
// (column-major, ld ldr): block b = rows [max(0, n - 32(b+1)), n - 32b), a
// partial top block in the top-left w x w corner of its slot with identity
// padding; Rinv_b[i][k] at Rinv[b * 1024 + i * 32 + k].  One warp per block:
// lane l solves R_bb X = e_l upward (column l of the inverse), each finished
// X[k] folded into the running sums of the rows above at once.
__global__ void __launch_bounds__(128) lsqr_trinv_kernel(const double* __restrict__ R,
                                                         int64_t ldr, int n,
                                                         double* __restrict__ Rinv) {
  __shared__ double Rs[4][32][33];
  const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
  const int bi = blockIdx.x * 4 + wl;
  const int nb = (n + 31) / 32;
  if (bi >= nb) return;
  const int hi = n - 32 * bi, lo = hi > 32 ? hi - 32 : 0, w = hi - lo;
  double (*Rb)[33] = Rs[wl];
#pragma unroll
  for (int j = 0; j < 32; ++j)  // lane = row
    Rb[lane][j] = (lane < w && j < w) ? (j >= lane ? R[(int64_t)(lo + j) * ldr + lo + lane] : 0.0)
                                      : (j == lane ? 1.0 : 0.0);
  __syncwarp();
  const double rd = 1.0 / Rb[lane][lane];
  double acc[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) acc[i] = 0.0;
  double* out = Rinv + (int64_t)bi * 1024;
#pragma unroll
  for (int k = 31; k >= 0; --k) {
    const double rk = __shfl_sync(0xffffffffu, rd, k);
    const double xk = k == lane ? rk : (k < lane ? -acc[k] * rk : 0.0);
    out[k * 32 + lane] = xk;  // Rinv_b[k][lane]
#pragma unroll
    for (int i = 0; i < k; ++i) acc[i] = fma(Rb[i][k], xk, acc[i]);
  }
}

__global__ void __launch_bounds__(LT_NT) lsqr_trsv_t_kernel(const double* __restrict__ R,
                                                            int64_t ldr, int n,
                                                            const double* __restrict__ z,
                                                            double beta, const double* v_prev,
                                                            double* v_out, double* norm2,
                                                            const double* __restrict__ Rinv,
                                                            const double* __restrict__ dscal) {
  extern __shared__ double xs[];
  __shared__ double red[32];
  if (dscal) {  // beta = ||r|| of the step's pass; nothing to do when it is 0
    beta = sqrt(dscal[LS_BETA2]);
    if (beta == 0.0) return;
  }
  for (int i = threadIdx.x; i < n; i += LT_NT) xs[i] = z[i];
  __syncthreads();
  if (R) lq_solve_t(R, ldr, n, xs, Rinv);
  double ss = 0.0;
  for (int i = threadIdx.x; i < n; i += LT_NT) {
    const double v = xs[i] - beta * v_prev[i];
    v_out[i] = v;
    ss = fma(v, v, ss);
  }
  const double t = lq_block_sum(ss, red);
  if (threadIdx.x == 0) *norm2 = t;
}

// v_n = v_raw / alfa (alfa > 0; else unchanged), written back; y = R^-1 v_n.
__global__ void __launch_bounds__(LT_NT) lsqr_trsv_n_kernel(const double* __restrict__ R,
                                                            int64_t ldr, int n, double alfa,
                                                            double* v, double* y,
                                                            const double* __restrict__ Rinv,
                                                            const double* __restrict__ dscal,
                                                            double* __restrict__ vcopy) {
  extern __shared__ double xs[];
  if (dscal) {  // alfa = ||v|| from the transposed solve; skipped when beta == 0
    if (sqrt(dscal[LS_BETA2]) == 0.0) return;
    alfa = sqrt(dscal[LS_ALFA2]);
  }
  for (int i = threadIdx.x; i < n; i += LT_NT) {
    const double vn = alfa > 0.0 ? v[i] / alfa : v[i];
    v[i] = vn;
    if (vcopy) vcopy[i] = vn;
    xs[i] = vn;
  }
  __syncthreads();
  if (R) lq_solve_n(R, ldr, n, xs, Rinv);
  for (int i = threadIdx.x; i < n; i += LT_NT) y[i] = xs[i];
}

// x += c1 w; w = v + c2 w; ||x||^2
__global__ void __launch_bounds__(LT_NT) lsqr_xw_kernel(int n, double c1, double c2,
                                                        const double* v, double* w, double* x,
                                                        double* norm2,
                                                        const double* __restrict__ dscal) {
  __shared__ double red[32];
  if (dscal) {
    c1 = dscal[LS_C1];
    c2 = dscal[LS_C2];
  }
  double ss = 0.0;
  for (int i = threadIdx.x; i < n; i += LT_NT) {
    const double wi = w[i];
    const double xi = x[i] + c1 * wi;
    x[i] = xi;
    w[i] = v[i] + c2 * wi;
    ss = fma(xi, xi, ss);
  }
  const double t = lq_block_sum(ss, red);
  if (threadIdx.x == 0) *norm2 = t;
}

static int sm_count_lq() { return sm_count_cached(); }

}  // namespace skl

using namespace skl;

// Scratch for the reductions: doubles of `work` and unsigned ints of
// `counters` (zero-initialised once; the kernels reset what they use).
extern "C" int64_t skl_lsqr_work_size(int64_t m, int64_t n) {
  (void)m;
  const int64_t groups = (n + LQ_TC - 1) / LQ_TC;
  const int64_t sms = sm_count_lq();
  return std::max<int64_t>(4 * sms, (8 * sms + groups) * LQ_TC) + 64;
}

extern "C" int64_t skl_lsqr_counter_size(int64_t n) { return (n + LQ_TC - 1) / LQ_TC + 8; }

extern "C" int skl_lsqr_gemv_n(const double* A, int64_t m, int64_t n, int64_t lda, const double* y,
                               double s, double alpha, const double* u_in, double* u_out,
                               double* norm2, double* work, unsigned int* counters, void* stream) {
  clear_error();
  SKL_REQUIRE(m >= 1 && n >= 0 && u_out && norm2 && work && counters && (!A || (y && lda >= m)),
              SKL_ERR_INVALID, "lsqr_gemv_n: bad arguments");
  SKL_REQUIRE(!A || (((uintptr_t)A & 15) == 0 && (lda % 2 == 0 || m == 1)), SKL_ERR_INVALID,
              "lsqr_gemv_n: A must be 16-byte aligned with an even leading dimension");
  const int64_t pairs = (m + 1) / 2;
  const int blocks = (int)std::max<int64_t>(
      1, std::min<int64_t>((pairs + LQ_NT - 1) / LQ_NT, 4LL * sm_count_lq()));
  const size_t smem = (A && n <= LQ_YMAX) ? (size_t)n * sizeof(double) : 0;
  lsqr_gemv_n_kernel<<<blocks, LQ_NT, smem, (cudaStream_t)stream>>>(
      A, m, n, lda, y, s, alpha, u_in, u_out, work, norm2, counters);
  SKL_CUDA_LAUNCH();
  return SKL_OK;
}

extern "C" int skl_lsqr_gemv_t(const double* A, int64_t m, int64_t n, int64_t lda,
                               const double* u_raw, double beta, double* u_n, double* z,
                               double* work, unsigned int* counters, void* stream) {
  clear_error();
  SKL_REQUIRE(m >= 1 && n >= 1 && u_raw && u_n && z && work && counters && beta > 0.0 &&
                  (!A || lda >= m),
              SKL_ERR_INVALID, "lsqr_gemv_t: bad arguments");
  SKL_REQUIRE(!A || (((uintptr_t)A & 15) == 0 && lda % 2 == 0) || m == 1, SKL_ERR_INVALID,
              "lsqr_gemv_t: A must be 16-byte aligned with an even leading dimension");
  SKL_REQUIRE(((uintptr_t)u_n & 15) == 0, SKL_ERR_INVALID, "lsqr_gemv_t: u_n must be 16-byte aligned");
  const int64_t groups = (n + LQ_TC - 1) / LQ_TC;
  // one wave: row chunks so that groups x chunks fills the resident CTA slots
  // resident CTAs per SM, cached per device (atomic: concurrent callers)
  static std::atomic<int> occ_cache[64];
  int dev = 0;
  cudaGetDevice(&dev);
  int occ = (dev >= 0 && dev < 64) ? occ_cache[dev].load(std::memory_order_relaxed) : 0;
  if (!occ) {
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, lsqr_gemv_t_kernel, LQ_NT, 0);
    occ = std::max(occ, 1);
    if (dev >= 0 && dev < 64) occ_cache[dev].store(occ, std::memory_order_relaxed);
  }
  int64_t nrc = std::max<int64_t>(1, (int64_t)occ * sm_count_lq() / groups);
  nrc = std::min<int64_t>(nrc, 1024);
  int64_t rows_per = (m + nrc - 1) / nrc;
  rows_per = (rows_per + 2 * LQ_NT - 1) / (2 * LQ_NT) * (2 * LQ_NT);
  nrc = (m + rows_per - 1) / rows_per;
  const int sblocks = (int)std::min<int64_t>((m + 255) / 256, 8LL * sm_count_lq());
  lsqr_scale_kernel<<<sblocks, 256, 0, (cudaStream_t)stream>>>(u_raw, beta, m, u_n);
  SKL_CUDA_LAUNCH();
  lsqr_gemv_t_kernel<<<dim3((unsigned)groups, (unsigned)nrc), LQ_NT, 0, (cudaStream_t)stream>>>(
      A, m, n, lda, u_n, rows_per, work, z, counters);
  SKL_CUDA_LAUNCH();
  return SKL_OK;
}

// One pass: r_out = s A y - alpha (r_prev / beta_prev), ||r_out||^2 and
// z = A^T r_out / ||r_out|| (see lsqr_fused_kernel).  n <= 256; r_prev may
// be null (no alpha term).  `work` needs skl_lsqr_fused_work_size doubles.
extern "C" int64_t skl_lsqr_fused_work_size(int64_t n) {
  return (int64_t)sm_count_lq() * 2 * (n + 1) + 64;
}

static int fused_launch(const double* A, int64_t m, int64_t n, int64_t lda, const double* y,
                        double s, double alpha, const double* r_prev, double beta_prev,
                        double* r_out, double* z, double* norm2, double* work,
                        unsigned int* counters, const double* dscal, void* stream) {
  SKL_REQUIRE(A && y && r_out && z && norm2 && work && counters && m >= 1 && n >= 1 &&
                  n <= 256 && lda >= m && (dscal || !r_prev || beta_prev > 0.0),
              SKL_ERR_INVALID, "lsqr_fused: bad arguments");
  SKL_REQUIRE(((uintptr_t)A & 15) == 0 && lda % 2 == 0, SKL_ERR_INVALID,
              "lsqr_fused: A must be 16-byte aligned with an even leading dimension");
  const int64_t nblk = (m + LF_RB - 1) / LF_RB;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(nblk, 2LL * sm_count_lq()));
  double* zpart = work;
  double* npart = work + (int64_t)grid * n;
  unsigned int* counter = counters + (skl_lsqr_counter_size(n) - 1);
  cudaStream_t st = (cudaStream_t)stream;
  const int nc = (int)((n + 7) / 8);
#define SKL_LF_LAUNCH(NCV)                                                                    \
  do {                                                                                        \
    int occ = 1;                                                                              \
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, lsqr_fused_kernel<NCV>, LQ_NT, 0);    \
    const int gr = (int)std::max<int64_t>(                                                    \
        1, std::min<int64_t>({nblk, (int64_t)std::max(occ, 1) * sm_count_lq(), (int64_t)grid})); \
    lsqr_fused_kernel<NCV><<<gr, LQ_NT, 0, st>>>(A, m, n, lda, y, s, alpha, r_prev, beta_prev, \
                                                 r_out, zpart, npart, z, norm2, counter,      \
                                                 dscal);                                      \
  } while (0)
  static const bool reg_kernel = env_flag("SKL_LSQR_FUSED_REG");  // A/B knob
#define SKL_LF2_LAUNCH(NCV, STV)                                                              \
  do {                                                                                        \
    const size_t smem = (size_t)(STV) * 8 * (NCV) * LF2_RB * sizeof(double);                  \
    SKL_CUDA(raise_smem_limit(lsqr_fused_async_kernel<NCV, STV>, smem));                      \
    int occ = 1;                                                                              \
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, lsqr_fused_async_kernel<NCV, STV>,    \
                                                  LQ_NT, smem);                               \
    const int64_t nb2 = (m + LF2_RB - 1) / LF2_RB;                                            \
    const int gr = (int)std::max<int64_t>(                                                    \
        1, std::min<int64_t>({nb2, (int64_t)std::max(occ, 1) * sm_count_lq(), (int64_t)grid})); \
    lsqr_fused_async_kernel<NCV, STV><<<gr, LQ_NT, smem, st>>>(A, m, n, lda, y, s, alpha,     \
                                                               r_prev,                         \
                                                          beta_prev, r_out, zpart, npart, z,   \
                                                          norm2, counter, dscal);              \
  } while (0)
  if (reg_kernel) {
    if (nc <= 8)
      SKL_LF_LAUNCH(8);
    else if (nc <= 16)
      SKL_LF_LAUNCH(16);
    else
      SKL_LF_LAUNCH(32);
  } else {
    // stages: ~192 KB of ring per CTA (64 KB blocks at n = 256)
    if (nc <= 8)
      SKL_LF2_LAUNCH(8, 8);
    else if (nc <= 16)
      SKL_LF2_LAUNCH(16, 6);
    else
      SKL_LF2_LAUNCH(32, 3);
  }
#undef SKL_LF_LAUNCH
#undef SKL_LF2_LAUNCH
  SKL_CUDA_LAUNCH();
  return SKL_OK;
}

extern "C" int skl_lsqr_fused(const double* A, int64_t m, int64_t n, int64_t lda, const double* y,
                              double s, double alpha, const double* r_prev, double beta_prev,
                              double* r_out, double* z, double* norm2, double* work,
                              unsigned int* counters, void* stream) {
  clear_error();
  return fused_launch(A, m, n, lda, y, s, alpha, r_prev, beta_prev, r_out, z, norm2, work,
                      counters, nullptr, stream);
}

extern "C" int skl_lsqr_fused_dev(const double* A, int64_t m, int64_t n, int64_t lda,
                                  const double* y, const double* r_prev, double* r_out, double* z,
                                  double* norm2, double* work, unsigned int* counters,
                                  const double* state, void* stream) {
  clear_error();
  SKL_REQUIRE(state, SKL_ERR_INVALID, "lsqr_fused_dev: state is required");
  return fused_launch(A, m, n, lda, y, 1.0, 0.0, r_prev, 1.0, r_out, z, norm2, work, counters,
                      state, stream);
}

extern "C" int skl_lsqr_rinv_blocks(const double* R, int64_t ldr, int64_t n, double* Rinv,
                                    void* stream) {
  clear_error();
  SKL_REQUIRE(R && Rinv && n >= 1 && ldr >= n && n <= 24 * 1024, SKL_ERR_INVALID,
              "lsqr_rinv_blocks: bad arguments");
  const int nb = (int)((n + 31) / 32);
  lsqr_trinv_kernel<<<(nb + 3) / 4, 128, 0, (cudaStream_t)stream>>>(R, ldr, (int)n, Rinv);
  SKL_CUDA_LAUNCH();
  return SKL_OK;
}

static int trsv_t_launch(const double* R, int64_t ldr, int64_t n, const double* z, double beta,
                         const double* v_prev, double* v_out, double* norm2, const double* Rinv,
                         void* stream, const double* dscal = nullptr) {
  clear_error();
  SKL_REQUIRE(n >= 1 && n <= 24 * 1024 && z && v_prev && v_out && norm2 && (!R || ldr >= n),
              SKL_ERR_INVALID, "lsqr_trsv_t: bad arguments");
  const size_t smem = (size_t)n * sizeof(double);
  if (smem > 48 * 1024) SKL_CUDA(raise_smem_limit(lsqr_trsv_t_kernel, smem));
  lsqr_trsv_t_kernel<<<1, LT_NT, smem, (cudaStream_t)stream>>>(R, ldr, (int)n, z, beta, v_prev,
                                                               v_out, norm2, Rinv, dscal);
  SKL_CUDA_LAUNCH();
  return SKL_OK;
}

extern "C" int skl_lsqr_trsv_t(const double* R, int64_t ldr, int64_t n, const double* z,
                               double beta, const double* v_prev, double* v_out, double* norm2,
                               void* stream) {
  clear_error();
  return trsv_t_launch(R, ldr, n, z, beta, v_prev, v_out, norm2, nullptr, stream);
}

extern "C" int skl_lsqr_trsv_t_inv(const double* R, int64_t ldr, int64_t n, const double* Rinv,
                                   const double* z, double beta, const double* v_prev,
                                   double* v_out, double* norm2, void* stream) {
  clear_error();
  SKL_REQUIRE(R && Rinv, SKL_ERR_INVALID, "lsqr_trsv_t_inv: R and Rinv are required");
  return trsv_t_launch(R, ldr, n, z, beta, v_prev, v_out, norm2, Rinv, stream);
}

static int trsv_n_launch(const double* R, int64_t ldr, int64_t n, double alfa, double* v,
                         double* y, const double* Rinv, void* stream,
                         const double* dscal = nullptr, double* vcopy = nullptr) {
  clear_error();
  SKL_REQUIRE(n >= 1 && n <= 24 * 1024 && v && y && (!R || ldr >= n), SKL_ERR_INVALID,
              "lsqr_trsv_n: bad arguments");
  const size_t smem = (size_t)n * sizeof(double);
  if (smem > 48 * 1024) SKL_CUDA(raise_smem_limit(lsqr_trsv_n_kernel, smem));
  lsqr_trsv_n_kernel<<<1, LT_NT, smem, (cudaStream_t)stream>>>(R, ldr, (int)n, alfa, v, y, Rinv,
                                                               dscal, vcopy);
  SKL_CUDA_LAUNCH();
  return SKL_OK;
}

extern "C" int skl_lsqr_trsv_n(const double* R, int64_t ldr, int64_t n, double alfa, double* v,
                               double* y, void* stream) {
  clear_error();
  return trsv_n_launch(R, ldr, n, alfa, v, y, nullptr, stream);
}

extern "C" int skl_lsqr_trsv_n_inv(const double* R, int64_t ldr, int64_t n, const double* Rinv,
                                   double alfa, double* v, double* y, void* stream) {
  clear_error();
  SKL_REQUIRE(R && Rinv, SKL_ERR_INVALID, "lsqr_trsv_n_inv: R and Rinv are required");
  return trsv_n_launch(R, ldr, n, alfa, v, y, Rinv, stream);
}

extern "C" int skl_lsqr_xw(int64_t n, double c1, double c2, const double* v, double* w, double* x,
                           double* norm2, void* stream) {
  clear_error();
  SKL_REQUIRE(n >= 1 && v && w && x && norm2, SKL_ERR_INVALID, "lsqr_xw: bad arguments");
  lsqr_xw_kernel<<<1, LT_NT, 0, (cudaStream_t)stream>>>((int)n, c1, c2, v, w, x, norm2, nullptr);
  SKL_CUDA_LAUNCH();
  return SKL_OK;
}

// One step of LSQR's scalar recurrence on the device (solvers.py:193-222 as
// the host loop writes it, the same IEEE operations in the same order: no
// contraction, correctly rounded sqrt and division), so the host reads the
// state once per iteration instead of three times.
__device__ __forceinline__ void ls_sym_ortho(double a, double b, double* c, double* s,
                                             double* r) {
  if (b == 0.0) {
    *c = a != 0.0 ? copysign(1.0, a) : 1.0;
    *s = 0.0;
    *r = fabs(a);
    return;
  }
  if (a == 0.0) {
    *c = 0.0;
    *s = copysign(1.0, b);
    *r = fabs(b);
    return;
  }
  if (fabs(b) > fabs(a)) {
    const double tau = __ddiv_rn(a, b);
    const double sn = __ddiv_rn(copysign(1.0, b), __dsqrt_rn(__dadd_rn(1.0, __dmul_rn(tau, tau))));
    *c = __dmul_rn(sn, tau);
    *s = sn;
    *r = __ddiv_rn(b, sn);
    return;
  }
  const double tau = __ddiv_rn(b, a);
  const double cs = __ddiv_rn(copysign(1.0, a), __dsqrt_rn(__dadd_rn(1.0, __dmul_rn(tau, tau))));
  *c = cs;
  *s = __dmul_rn(cs, tau);
  *r = __ddiv_rn(a, cs);
}

__device__ __forceinline__ void ls_recur(double* st) {
  const double beta = __dsqrt_rn(st[LS_BETA2]);
  double alfa = st[LS_ALFA];
  double anorm = st[LS_ANORM];
  if (beta > 0.0) {
    anorm = __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(anorm, anorm), __dmul_rn(alfa, alfa)),
                                 __dmul_rn(beta, beta)));
    alfa = __dsqrt_rn(st[LS_ALFA2]);
  }
  double cs, sn, rho;
  ls_sym_ortho(st[LS_RHOBAR], beta, &cs, &sn, &rho);
  const double theta = __dmul_rn(sn, alfa);
  const double rhobar = __dmul_rn(-cs, alfa);
  const double phibar0 = st[LS_PHIBAR];
  const double phi = __dmul_rn(cs, phibar0);
  const double phibar = __dmul_rn(sn, phibar0);
  st[LS_C1] = __ddiv_rn(phi, rho);
  st[LS_C2] = __ddiv_rn(-theta, rho);
  st[LS_RNORM] = phibar;
  st[LS_ARNORM] = __dmul_rn(alfa, fabs(__dmul_rn(sn, phi)));
  st[LS_ALFA] = alfa;
  st[LS_BETA] = beta;
  st[LS_RHOBAR] = rhobar;
  st[LS_PHIBAR] = phibar;
  st[LS_ANORM] = anorm;
  st[LS_BPREV] = beta > 0.0 ? beta : 1.0;
}
__global__ void lsqr_recur_kernel(double* st) { ls_recur(st); }

// Full inverse of the n x n upper-triangular R (n <= 256), column-major with
// ld n, zeros below the diagonal: one warp per column j, back substitution
// right-looking over R's columns (z_i = t_i / R_ii, then t_l -= R_li z_i for
// l < i: a coalesced column read per step; lane holds t_l for l = lane +
// 32 q).  Once per preconditioned solve: R does not change across LSQR
// iterations, and the step's two triangular solves become products with
// R^{-1} (lq_gemv_full_*).
constexpr int LQ_FULL_MAX = 256;

__global__ void __launch_bounds__(256) lsqr_rinv_full_kernel(const double* __restrict__ R,
                                                             int64_t ldr, int n,
                                                             double* __restrict__ Ri) {
  const int lane = threadIdx.x & 31;
  const int j = (int)blockIdx.x * 8 + (threadIdx.x >> 5);
  if (j >= n) return;
  double t[LQ_FULL_MAX / 32];
#pragma unroll
  for (int q = 0; q < LQ_FULL_MAX / 32; ++q) t[q] = (lane + 32 * q == j) ? 1.0 : 0.0;
  double* col = Ri + (int64_t)j * n;
  for (int i = j + 1 + lane; i < n; i += 32) col[i] = 0.0;
  for (int i = j; i >= 0; --i) {
    double ti = 0.0;
#pragma unroll
    for (int q = 0; q < LQ_FULL_MAX / 32; ++q)
      if (q == (i >> 5)) ti = t[q];
    const double zi = __shfl_sync(0xffffffffu, ti, i & 31) / R[(int64_t)i * ldr + i];
    if (lane == (i & 31)) col[i] = zi;
    const double* ri = R + (int64_t)i * ldr;
#pragma unroll
    for (int q = 0; q < LQ_FULL_MAX / 32; ++q) {
      const int l = lane + 32 * q;
      if (l < i) t[q] = fma(-ri[l], zi, t[q]);
    }
  }
}

// xs <- R^{-T} xs with RF = R^{-1} (column-major, ld n): out_j = sum_{i <= j}
// RF[i + j n] xs_i, warp w the columns j = w (mod warps), lanes split i.
__device__ void lq_gemv_full_t(const double* __restrict__ RF, int n, double* xs, double* tmp) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int j = warp; j < n; j += nw) {
    const double* col = RF + (int64_t)j * n;
    double a = 0.0;
    for (int i = lane; i <= j; i += 32) a = fma(col[i], xs[i], a);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
    if (lane == 0) tmp[j] = a;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += blockDim.x) xs[i] = tmp[i];
  __syncthreads();
}

// xs <- R^{-1} xs: out_i = sum_{j >= i} RF[i + j n] xs_j, a thread per (row,
// half of the columns), halves added in order.
__device__ void lq_gemv_full_n(const double* __restrict__ RF, int n, double* xs, double* tmp) {
  const int nh = blockDim.x / 2;
  const int i = threadIdx.x % nh, hf = threadIdx.x / nh;
  const int jm = (n + 1) / 2;
  double a = 0.0;
  if (i < n) {
    const int j0 = hf ? max(jm, i) : i, j1 = hf ? n : jm;
    int j = j0;
    for (; j + 4 <= j1; j += 4) {
      const double r0 = RF[(int64_t)j * n + i], r1 = RF[(int64_t)(j + 1) * n + i];
      const double r2 = RF[(int64_t)(j + 2) * n + i], r3 = RF[(int64_t)(j + 3) * n + i];
      a = fma(r0, xs[j], a);
      a = fma(r1, xs[j + 1], a);
      a = fma(r2, xs[j + 2], a);
      a = fma(r3, xs[j + 3], a);
    }
    for (; j < j1; ++j) a = fma(RF[(int64_t)j * n + i], xs[j], a);
  }
  if (hf && i < n) tmp[i] = a;
  __syncthreads();
  if (!hf && i < n) a += tmp[i];
  __syncthreads();
  if (!hf && i < n) xs[i] = a;
  __syncthreads();
}

// The whole device step after a pass in one CTA (what lsqr_trsv_t_kernel,
// lsqr_trsv_n_kernel, lsqr_recur_kernel and lsqr_xw_kernel do in four
// launches, with the same operations in the same order: bitwise the same
// iterates), so an iteration is two kernels -- the pass and this -- and
// the step's three launch gaps are gone.  Launched with programmatic
// serialization right after the pass (pdl_enter).
__global__ void __launch_bounds__(LT_NT) lsqr_step_kernel(
    const double* __restrict__ R, int64_t ldr, int n, const double* __restrict__ Rinv,
    const double* __restrict__ z, double* v, double* v_raw, double* y, double* w, double* x,
    double* st, const double* __restrict__ RF) {
  pdl_enter();
  extern __shared__ double xs[];
  __shared__ double red[32];
  const int tid = threadIdx.x;
  const double beta = sqrt(st[LS_BETA2]);  // ||r|| of the step's pass
  if (beta != 0.0) {
    // v_raw = R^-T z - beta v, ||v_raw||^2 -> LS_ALFA2
    for (int i = tid; i < n; i += LT_NT) xs[i] = z[i];
    __syncthreads();
    if (RF)
      lq_gemv_full_t(RF, n, xs, xs + n);
    else if (R)
      lq_solve_t(R, ldr, n, xs, Rinv);
    double ss = 0.0;
    for (int i = tid; i < n; i += LT_NT) {
      const double vv = xs[i] - beta * v[i];
      v_raw[i] = vv;
      ss = fma(vv, vv, ss);
    }
    const double t = lq_block_sum(ss, red);
    if (tid == 0) st[LS_ALFA2] = t;
    __syncthreads();
    // v_n = v_raw / alfa into v_raw and v, y = R^-1 v_n
    const double alfa = sqrt(st[LS_ALFA2]);
    for (int i = tid; i < n; i += LT_NT) {
      const double vn = alfa > 0.0 ? v_raw[i] / alfa : v_raw[i];
      v_raw[i] = vn;
      v[i] = vn;
      xs[i] = vn;
    }
    __syncthreads();
    if (RF)
      lq_gemv_full_n(RF, n, xs, xs + n);
    else if (R)
      lq_solve_n(R, ldr, n, xs, Rinv);
    for (int i = tid; i < n; i += LT_NT) y[i] = xs[i];
  }
  __syncthreads();
  if (tid == 0) ls_recur(st);
  __syncthreads();
  // x += c1 w; w = v + c2 w; ||x||^2 -> LS_XNORM2
  const double c1 = st[LS_C1], c2 = st[LS_C2];
  double ss = 0.0;
  for (int i = tid; i < n; i += LT_NT) {
    const double wi = w[i];
    const double xi = x[i] + c1 * wi;
    x[i] = xi;
    w[i] = v[i] + c2 * wi;
    ss = fma(xi, xi, ss);
  }
  const double t = lq_block_sum(ss, red);
  if (tid == 0) st[LS_XNORM2] = t;
}

// One device-driven LSQR step after the fused pass (n <= 256 dense): the
// transposed solve (beta from the pass), the solve for y (alfa from it), the
// scalar recurrence and the x/w update, with no host scalar on the way;
// state (LS_STATE doubles, device) carries the recurrence.  v_prev holds v
// on entry and v_n on exit (v_raw is scratch).
extern "C" int skl_lsqr_step_dev(const double* R, int64_t ldr, int64_t n, const double* Rinv,
                                 const double* z, double* v, double* v_raw, double* y, double* w,
                                 double* x, double* state, void* stream) {
  clear_error();
  SKL_REQUIRE(z && v && v_raw && y && w && x && state && n >= 1, SKL_ERR_INVALID,
              "lsqr_step_dev: bad arguments");
  SKL_REQUIRE(n <= 24 * 1024 && (!R || ldr >= n), SKL_ERR_INVALID, "lsqr_step_dev: bad shape");
  const size_t smem = (size_t)n * sizeof(double);
  if (smem > 48 * 1024) SKL_CUDA(raise_smem_limit(lsqr_step_kernel, smem));
  // the pass is the kernel right before this one on the stream
  SKL_CUDA(launch_k(lsqr_step_kernel, dim3(1), dim3(LT_NT), smem, (cudaStream_t)stream, true, R,
                    ldr, (int)n, Rinv, z, v, v_raw, y, w, x, state, (const double*)nullptr));
  return SKL_OK;
}

// R^{-1} in full (n <= 256; Ri: n * n doubles, device), once per solve.
extern "C" int skl_lsqr_rinv_full(const double* R, int64_t ldr, int64_t n, double* Ri,
                                  void* stream) {
  clear_error();
  SKL_REQUIRE(R && Ri && n >= 1 && n <= LQ_FULL_MAX && ldr >= n, SKL_ERR_INVALID,
              "lsqr_rinv_full: bad arguments (n <= %d)", LQ_FULL_MAX);
  lsqr_rinv_full_kernel<<<(unsigned)((n + 7) / 8), 256, 0, (cudaStream_t)stream>>>(R, ldr, (int)n,
                                                                                   Ri);
  SKL_CUDA_LAUNCH();
  return SKL_OK;
}

// skl_lsqr_step_dev with both triangular solves as products with the full
// R^{-1} (skl_lsqr_rinv_full).
extern "C" int skl_lsqr_step_full_dev(const double* Ri, int64_t n, const double* z, double* v,
                                      double* v_raw, double* y, double* w, double* x,
                                      double* state, void* stream) {
  clear_error();
  SKL_REQUIRE(Ri && z && v && v_raw && y && w && x && state && n >= 1 && n <= LQ_FULL_MAX,
              SKL_ERR_INVALID, "lsqr_step_full_dev: bad arguments");
  const size_t smem = 2 * (size_t)n * sizeof(double);
  SKL_CUDA(launch_k(lsqr_step_kernel, dim3(1), dim3(LT_NT), smem, (cudaStream_t)stream, true,
                    (const double*)nullptr, (int64_t)n, (int)n, (const double*)nullptr, z, v, v_raw,
                    y, w, x, state, Ri));
  return SKL_OK;
}

extern "C" int64_t skl_lsqr_state_size(void) { return LS_STATE; }

extern "C" int skl_lsqr_spmv(const int64_t* indptr, const int64_t* indices, const double* values,
                             int64_t m, const double* y, double s, double alpha,
                             const double* u_in, double* u_out, double* norm2, double* work,
                             unsigned int* counters, void* stream) {
  clear_error();
  SKL_REQUIRE(indptr && indices && values && y && u_out && norm2 && work && counters && m >= 1,
              SKL_ERR_INVALID, "lsqr_spmv: bad arguments");
  const int blocks = (int)std::max<int64_t>(
      1, std::min<int64_t>((m + LQ_NT - 1) / LQ_NT, 4LL * sm_count_lq()));
  lsqr_spmv_kernel<<<blocks, LQ_NT, 0, (cudaStream_t)stream>>>(indptr, indices, values, m, y, s,
                                                               alpha, u_in, u_out, work, norm2,
                                                               counters);
  SKL_CUDA_LAUNCH();
  return SKL_OK;
}

extern "C" int skl_lsqr_csc_t(const int64_t* colptr, const int32_t* rowidx, const double* cval,
                              int64_t m, int64_t n, const double* u_raw, double beta, double* u_n,
                              double* z, void* stream) {
  clear_error();
  SKL_REQUIRE(colptr && rowidx && cval && u_raw && u_n && z && m >= 1 && n >= 1 && beta > 0.0,
              SKL_ERR_INVALID, "lsqr_csc_t: bad arguments");
  cudaStream_t st = (cudaStream_t)stream;
  const int sblocks = (int)std::min<int64_t>((m + 255) / 256, 8LL * sm_count_lq());
  lsqr_scale_kernel<<<sblocks, 256, 0, st>>>(u_raw, beta, m, u_n);
  SKL_CUDA_LAUNCH();
  const int blocks = (int)std::max<int64_t>(
      1, std::min<int64_t>((n * 32 + LQ_NT - 1) / LQ_NT, 8LL * sm_count_lq()));
  lsqr_csc_t_kernel<<<blocks, LQ_NT, 0, st>>>(colptr, rowidx, cval, n, u_n, z);
  SKL_CUDA_LAUNCH();
  return SKL_OK;
}
