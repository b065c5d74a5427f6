// Ordered bucket walk for CountSketch / sparse-sign applies to a few long
// columns (a vector S*b, or n <= a handful of columns).
//
// Reference: /root/reference/pkg/src/sketchls/sketch.py:209,212 --
// `sparse_map @ b` is scipy's csr_matvec: for every bucket i the products
// s_j * b[j] of its source rows j are added in ascending j starting from
// +0.0.  The register-owned and lane-list dense kernels reproduce that fold
// with one CTA per column; for one long column that leaves most SMs idle,
// so they split the rows into P partitions and add the partials in a fixed
// order -- deterministic but not the reference's bits.  This kernel keeps
// the fold order and still fills the GPU by parallelising over buckets: a
// warp owns one (bucket, column), walks the bucket's source rows (the CSR of
// S built with the operator, rows ascending within a bucket) 128 entries at
// a time -- each lane gathers four entries, the next block's gathers are in
// flight while the current one is folded -- and lane 0 folds them in order
// out of a per-warp shared-memory stage (16-byte loads; a warp shuffle per
// term made the fold MIO-bound).  Bitwise-equal to csr_matvec / csr_matvecs.
//
// Bound: latency of the dependent fold (~512 entries per bucket at the
// BASELINE configs) and the gathers; the column itself is read once from HBM
// (sectors are shared by neighbouring buckets through L2).
#include <cuda_runtime.h>

#include "skl_common.h"

namespace skl {

constexpr int ORD_WARPS = 8;   // warps (buckets) per CTA
constexpr int ORD_PER_LANE = 4;
constexpr int ORD_BLOCK = 32 * ORD_PER_LANE;

struct OrdBlock {
  double v[ORD_PER_LANE];  // sign * value of entry base + lane + 32 q (0 past the end)
};

__device__ __forceinline__ OrdBlock ord_fetch(int64_t base, int64_t end, int lane,
                                              const int32_t* __restrict__ brow,
                                              const int8_t* __restrict__ bsign,
                                              const double* __restrict__ col, double scale) {
  OrdBlock b;
#pragma unroll
  for (int q = 0; q < ORD_PER_LANE; ++q) {
    const int64_t e = base + lane + 32 * q;
    double v = 0.0;
    if (e < end) {
      const double s = (double)__ldg(bsign + e) * scale;
      // csr_matvec's `Ax[jj] * Xx[j]` rounded on its own (no FMA with the add)
      v = __dmul_rn(s, __ldg(col + __ldg(brow + e)));
    }
    b.v[q] = v;
  }
  return b;
}

__global__ void __launch_bounds__(32 * ORD_WARPS)
countsketch_ordered_kernel(const double* __restrict__ A, int64_t lda, int64_t n,
                           const double* __restrict__ b, const int32_t* __restrict__ brow,
                           const int64_t* __restrict__ bptr, const int8_t* __restrict__ bsign,
                           double scale, int d, double* __restrict__ out, int64_t ldo,
                           double* __restrict__ outb, int accumulate) {
  __shared__ __align__(16) double stage[ORD_WARPS][ORD_BLOCK];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t bucket = (int64_t)blockIdx.x * ORD_WARPS + warp;
  const int64_t c = blockIdx.y;  // column (n == the b column when b != null)
  if (bucket >= d) return;
  const double* col = c < n ? A + c * lda : b;
  double* dst = c < n ? out + c * ldo + bucket : outb + bucket;
  const int64_t p0 = __ldg(bptr + bucket), p1 = __ldg(bptr + bucket + 1);
  double* buf = stage[warp];
  double s = 0.0;  // csr_matvec starts every output from +0.0
  OrdBlock cur = ord_fetch(p0, p1, lane, brow, bsign, col, scale);
  for (int64_t base = p0; base < p1; base += ORD_BLOCK) {
    const OrdBlock nxt = ord_fetch(base + ORD_BLOCK, p1, lane, brow, bsign, col, scale);
    const int cnt = p1 - base < ORD_BLOCK ? (int)(p1 - base) : ORD_BLOCK;
    // the block's products go through shared memory and lane 0 folds them
    // in order: 16-byte loads by one lane instead of a warp shuffle per term
    __syncwarp();
#pragma unroll
    for (int q = 0; q < ORD_PER_LANE; ++q) buf[lane + 32 * q] = cur.v[q];
    __syncwarp();
    if (lane == 0) {
      const double2* b2 = reinterpret_cast<const double2*>(buf);
      int i = 0;
      for (; i + 1 < cnt; i += 2) {
        const double2 v = b2[i >> 1];
        s = __dadd_rn(__dadd_rn(s, v.x), v.y);
      }
      if (i < cnt) s = __dadd_rn(s, buf[i]);
    }
    cur = nxt;
  }
  if (lane == 0) *dst = accumulate ? __dadd_rn(*dst, s) : s;
}

static int ordered_launch(const double* A, int64_t m, int64_t n, int64_t lda, const double* b,
                          const int32_t* brow, const int64_t* bptr, const int8_t* bsign,
                          double scale, int64_t d, double* SA, int64_t ldsa, double* Sb,
                          int accumulate, cudaStream_t st) {
  SKL_REQUIRE(m >= 1 && n >= 0 && d >= 1 && (n == 0 || (lda >= m && ldsa >= d)), SKL_ERR_SHAPE,
              "countsketch (ordered): bad shape m=%lld n=%lld d=%lld", (long long)m,
              (long long)n, (long long)d);
  SKL_REQUIRE(n + (b ? 1 : 0) >= 1 && n + 1 < 65535, SKL_ERR_SHAPE,
              "countsketch (ordered): bad column count %lld", (long long)n);
  SKL_REQUIRE(brow && bptr && bsign && (n == 0 || (A && SA)) && (!b || Sb), SKL_ERR_INVALID,
              "countsketch (ordered): null pointer");
  SKL_REQUIRE(d < (1LL << 31) - ORD_WARPS, SKL_ERR_SPEC, "countsketch (ordered): d too large");
  const int64_t ncols = n + (b ? 1 : 0);
  dim3 grid((unsigned)((d + ORD_WARPS - 1) / ORD_WARPS), (unsigned)ncols);
  countsketch_ordered_kernel<<<grid, 32 * ORD_WARPS, 0, st>>>(A, lda, n, b, brow, bptr, bsign,
                                                              scale, (int)d, SA, ldsa, Sb,
                                                              accumulate);
  SKL_CUDA_LAUNCH();
  return SKL_OK;
}

}  // namespace skl

using namespace skl;

extern "C" int skl_countsketch_dense_ordered(const double* A, int64_t m, int64_t n, int64_t lda,
                                             const double* b, const int32_t* bucket_rows,
                                             const int64_t* bucket_ptr, const int8_t* signs,
                                             double scale, int64_t d, double* SA, int64_t ldsa,
                                             double* Sb, int accumulate, void* stream) {
  clear_error();
  return ordered_launch(A, m, n, lda, b, bucket_rows, bucket_ptr, signs, scale, d, SA, ldsa, Sb,
                        accumulate, (cudaStream_t)stream);
}
