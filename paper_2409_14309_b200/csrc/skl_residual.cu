// ||A x - b||_2 on device (reference: /root/reference/pkg/src/sketchls/
// solvers.py:102-107, `A.data @ x - b.data` then np.linalg.norm).  This is
// the second full HBM pass over A of every SAA solve.  Dense A is column-
// major: each thread owns two adjacent rows (16-byte loads, coalesced
// across the warp) and folds the columns in ascending order with FMA, the
// column-axpy order of dgemv 'N'.  Squares are reduced per CTA and then in
// a fixed order (deterministic).
#include <cuda_runtime.h>

#include <algorithm>

#include "skl_common.h"

namespace skl {

constexpr int RS_NT = 256;
constexpr int RS_XMAX = 8192;  // x staged in shared memory up to this n

__device__ __forceinline__ double rs_block_sum(double v, double* red) {
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

__global__ void __launch_bounds__(RS_NT) residual_dense_kernel(const double* __restrict__ A,
                                                               int64_t m, int64_t n, int64_t lda,
                                                               const double* __restrict__ x,
                                                               const double* __restrict__ b,
                                                               double* part) {
  extern __shared__ double xs[];
  __shared__ double red[32];
  const bool stage = n <= RS_XMAX;
  if (stage)
    for (int64_t c = threadIdx.x; c < n; c += RS_NT) xs[c] = x[c];
  __syncthreads();
  const double* xv = stage ? xs : x;
  double ss = 0.0;
  const int64_t pairs = (m + 1) / 2;
  for (int64_t pr = blockIdx.x * (int64_t)RS_NT + threadIdx.x; pr < pairs;
       pr += (int64_t)gridDim.x * RS_NT) {
    const int64_t j = 2 * pr;
    double a0 = 0.0, a1 = 0.0;
    if (j + 1 < m) {
      const double* col = A + j;
      int64_t c = 0;
      for (; c + 8 <= n; c += 8) {
        double2 v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u)
          v[u] = __ldcs(reinterpret_cast<const double2*>(col + (c + u) * lda));
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          a0 = fma(v[u].x, xv[c + u], a0);
          a1 = fma(v[u].y, xv[c + u], a1);
        }
      }
      for (; c < n; ++c) {
        const double2 v = __ldcs(reinterpret_cast<const double2*>(col + c * lda));
        a0 = fma(v.x, xv[c], a0);
        a1 = fma(v.y, xv[c], a1);
      }
      const double r0 = a0 - b[j], r1 = a1 - b[j + 1];
      ss += r0 * r0;
      ss += r1 * r1;
    } else {
      for (int64_t c = 0; c < n; ++c) a0 = fma(A[j + c * lda], xv[c], a0);
      const double r0 = a0 - b[j];
      ss += r0 * r0;
    }
  }
  ss = rs_block_sum(ss, red);
  if (threadIdx.x == 0) part[blockIdx.x] = ss;
}

__global__ void __launch_bounds__(RS_NT) residual_dense_scalar_kernel(
    const double* __restrict__ A, int64_t m, int64_t n, int64_t lda, const double* __restrict__ x,
    const double* __restrict__ b, double* part) {
  __shared__ double red[32];
  double ss = 0.0;
  for (int64_t j = blockIdx.x * (int64_t)RS_NT + threadIdx.x; j < m;
       j += (int64_t)gridDim.x * RS_NT) {
    double a = 0.0;
    for (int64_t c = 0; c < n; ++c) a = fma(A[j + c * lda], x[c], a);
    const double r = a - b[j];
    ss += r * r;
  }
  ss = rs_block_sum(ss, red);
  if (threadIdx.x == 0) part[blockIdx.x] = ss;
}

__global__ void __launch_bounds__(RS_NT) residual_csr_kernel(const int64_t* __restrict__ indptr,
                                                             const int64_t* __restrict__ indices,
                                                             const double* __restrict__ values,
                                                             int64_t m, const double* __restrict__ x,
                                                             const double* __restrict__ b,
                                                             double* part) {
  __shared__ double red[32];
  double ss = 0.0;
  for (int64_t j = blockIdx.x * (int64_t)RS_NT + threadIdx.x; j < m;
       j += (int64_t)gridDim.x * RS_NT) {
    double a = 0.0;
    for (int64_t q = indptr[j]; q < indptr[j + 1]; ++q) a = fma(values[q], __ldg(x + indices[q]), a);
    const double r = a - b[j];
    ss += r * r;
  }
  ss = rs_block_sum(ss, red);
  if (threadIdx.x == 0) part[blockIdx.x] = ss;
}

__global__ void rs_finish_kernel(const double* part, int nparts, double* out) {
  __shared__ double red[32];
  double s = 0.0;
  for (int i = threadIdx.x; i < nparts; i += blockDim.x) s += part[i];
  s = rs_block_sum(s, red);
  if (threadIdx.x == 0) *out = sqrt(s);
}

static int rs_grid(int64_t work) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return (int)std::max<int64_t>(1, std::min<int64_t>((work + RS_NT - 1) / RS_NT, (int64_t)sms * 8));
}

// sync = false: *out (pinned host or device) is written in stream order and
// read by the caller once the stream has passed it (batched solves).
static int rs_finish(double* part, int blocks, double* out, cudaStream_t st, bool sync = true) {
  double* res = part + blocks;
  rs_finish_kernel<<<1, RS_NT, 0, st>>>(part, blocks, res);
  SKL_CUDA_LAUNCH();
  SKL_CUDA(cudaMemcpyAsync(out, res, sizeof(double), cudaMemcpyDefault, st));
  if (sync) SKL_CUDA(cudaStreamSynchronize(st));
  return SKL_OK;
}

}  // namespace skl

using namespace skl;

static int residual_dense_impl(const double* A, int64_t m, int64_t n, int64_t lda,
                               const double* x, const double* b, double* out, cudaStream_t st,
                               bool sync) {
  SKL_REQUIRE(A && x && b && out && m >= 1 && n >= 1 && lda >= m, SKL_ERR_SHAPE,
              "residual: bad arguments");
  const bool vec = ((uintptr_t)A & 15) == 0 && lda % 2 == 0;
  const int blocks = rs_grid(vec ? (m + 1) / 2 : m);
  double* part = nullptr;
  SKL_CUDA(malloc_async(&part, (blocks + 1) * sizeof(double), st));
  if (vec) {
    const size_t smem = n <= RS_XMAX ? n * sizeof(double) : 0;
    if (smem > 48 * 1024) SKL_CUDA(raise_smem_limit(residual_dense_kernel, smem));
    residual_dense_kernel<<<blocks, RS_NT, smem, st>>>(A, m, n, lda, x, b, part);
  } else {
    residual_dense_scalar_kernel<<<blocks, RS_NT, 0, st>>>(A, m, n, lda, x, b, part);
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    cudaFreeAsync(part, st);
    SKL_FAIL(SKL_ERR_CUDA, "residual kernel: %s", cudaGetErrorString(e));
  }
  int rc = rs_finish(part, blocks, out, st, sync);
  cudaFreeAsync(part, st);
  return rc;
}

extern "C" int skl_residual_dense(const double* A, int64_t m, int64_t n, int64_t lda,
                                  const double* x, const double* b, double* out, void* stream) {
  clear_error();
  return residual_dense_impl(A, m, n, lda, x, b, out, (cudaStream_t)stream, true);
}

extern "C" int skl_residual_dense_async(const double* A, int64_t m, int64_t n, int64_t lda,
                                        const double* x, const double* b, double* out,
                                        void* stream) {
  clear_error();
  return residual_dense_impl(A, m, n, lda, x, b, out, (cudaStream_t)stream, false);
}

static int residual_csr_impl(const int64_t* indptr, const int64_t* indices, const double* values,
                             int64_t m, int64_t n, const double* x, const double* b, double* out,
                             cudaStream_t st, bool sync) {
  SKL_REQUIRE(indptr && x && b && out && m >= 1 && n >= 1, SKL_ERR_SHAPE,
              "residual_csr: bad arguments");
  const int blocks = rs_grid(m);
  double* part = nullptr;
  SKL_CUDA(malloc_async(&part, (blocks + 1) * sizeof(double), st));
  residual_csr_kernel<<<blocks, RS_NT, 0, st>>>(indptr, indices, values, m, x, b, part);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    cudaFreeAsync(part, st);
    SKL_FAIL(SKL_ERR_CUDA, "residual_csr kernel: %s", cudaGetErrorString(e));
  }
  int rc = rs_finish(part, blocks, out, st, sync);
  cudaFreeAsync(part, st);
  return rc;
}

extern "C" int skl_residual_csr(const int64_t* indptr, const int64_t* indices,
                                const double* values, int64_t m, int64_t n, const double* x,
                                const double* b, double* out, void* stream) {
  clear_error();
  return residual_csr_impl(indptr, indices, values, m, n, x, b, out, (cudaStream_t)stream, true);
}

extern "C" int skl_residual_csr_async(const int64_t* indptr, const int64_t* indices,
                                      const double* values, int64_t m, int64_t n,
                                      const double* x, const double* b, double* out,
                                      void* stream) {
  clear_error();
  return residual_csr_impl(indptr, indices, values, m, n, x, b, out, (cudaStream_t)stream, false);
}
