// CountSketch apply S*A for CSR A (reference: /root/reference/pkg/src/
// sketchls/sketch.py:210-211, `(sparse_map @ A_csr).toarray()`).  scipy's
// csr_matmat (Gustavson) builds output row i of S*A by walking the source
// rows j of bucket i in ascending order and adding s_j * A[j, c] into each
// column c; densifying keeps those sums.  Reproducing that per-(i, c) fold
// order makes the device result bitwise-equal.
//
// Design (B200): a CTA owns 8 buckets x Cw output columns held as a dense
// tile in shared memory (bucket-major, odd row stride); one warp per bucket
// walks the bucket's source rows (the operator's bucket-sorted row list, i.e.
// the CSR of S) 32 rows at a time, fetching the next 32 rows' CSR extents
// while committing the current ones.  The warp flattens those rows'
// nonzeros in (row, position) order, lanes gather one nonzero each, and
// commit into the tile in flattened order: lanes hitting the same column are
// serialised by lane rank (__match_any_sync), distinct columns commit
// together.  The tile is then written once; the output needs no memset and
// no atomics.
#include <cuda_runtime.h>

#include <algorithm>
#include <vector>

#include "skl_common.h"

namespace skl {

constexpr int CSR_B = 8;   // buckets (warps) per CTA

__global__ void __launch_bounds__(CSR_B * 32)
    countsketch_csr_kernel(const int64_t* __restrict__ indptr, const int64_t* __restrict__ indices,
                           const double* __restrict__ values, const int32_t* __restrict__ brow,
                           const int64_t* __restrict__ bptr, const int8_t* __restrict__ bsign,
                           int64_t d, int64_t n, int64_t Cw, double* __restrict__ SA,
                           int64_t ldsa, double scale) {
  extern __shared__ double tile[];  // [CSR_B][cw + 1] (bucket-major, odd stride)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t i0 = (int64_t)blockIdx.x * CSR_B;
  const int64_t c0 = (int64_t)blockIdx.y * Cw;
  const int64_t cw = min(Cw, n - c0);
  const int64_t ldt = cw + 1;
  for (int64_t k = threadIdx.x; k < ldt * CSR_B; k += blockDim.x) tile[k] = 0.0;
  __syncthreads();

  const int64_t i = i0 + warp;
  if (i < d) {
    const int64_t r_beg = bptr[i], r_end = bptr[i + 1];
    double* my = tile + warp * ldt;  // column c at my[c - c0]
    // Software pipeline over rounds of 32 rows: the bucket-row index of
    // round r+2 (coalesced) and the CSR extent of round r+1 (dependent on
    // it) are in flight while round r commits; the signs come pre-gathered
    // in bucket order, so they stream.
    // raw loads of the next round; converted only when the round starts, so
    // nothing waits on them early
    int64_t np0 = 0, np1 = 0;
    int8_t nsg = 0;
    int32_t nj = -1;  // bucket row of round r+2 for this lane
    {
      const int64_t r = r_beg + lane;
      if (r < r_end) {
        const int32_t j = brow[r];
        np0 = indptr[j];
        np1 = indptr[j + 1];
        nsg = bsign[r];
      }
      const int64_t r2 = r_beg + 32 + lane;
      if (r2 < r_end) nj = brow[r2];
    }
    for (int64_t base = r_beg; base < r_end; base += 32) {
      const int64_t p0 = np0, cnt = np1 - np0;
      const double s = (double)nsg * scale;  // +-1 (CountSketch) or +-fl(1/sqrt(s))
      np0 = 0;
      np1 = 0;
      nsg = 0;
      if (nj >= 0) {
        np0 = indptr[nj];
        np1 = indptr[nj + 1];
        nsg = bsign[base + 32 + lane];
      }
      nj = -1;
      if (base + 64 + lane < r_end) nj = brow[base + 64 + lane];
      // exclusive scan of counts over the warp (lane order == ascending j)
      int64_t incl = cnt;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int64_t y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      const int64_t start = incl - cnt;
      const int64_t total = __shfl_sync(0xffffffffu, incl, 31);
      for (int64_t f0 = 0; f0 < total; f0 += 32) {
        const int64_t f = f0 + lane;
        // owner lane: largest l with start_l <= f (starts are nondecreasing)
        int lo = 0;
#pragma unroll
        for (int step = 16; step > 0; step >>= 1) {
          const int64_t st = __shfl_sync(0xffffffffu, start, min(lo + step, 31));
          if (lo + step <= 31 && st <= f) lo += step;
        }
        // among equal starts (empty rows) the largest index is the owner
        const int64_t st_o = __shfl_sync(0xffffffffu, start, lo);
        const int64_t p0_o = __shfl_sync(0xffffffffu, p0, lo);
        const double s_o = __shfl_sync(0xffffffffu, s, lo);
        bool valid = f < total;
        int64_t c = -1;
        double v = 0.0;
        if (valid) {
          const int64_t p = p0_o + (f - st_o);
          c = indices[p];
          v = values[p];
          valid = (c >= c0) && (c < c0 + cw);
        }
        const unsigned act = __ballot_sync(0xffffffffu, valid);
        const unsigned peers = __match_any_sync(0xffffffffu, valid ? c : -1);
        const unsigned grp = peers & act;
        const int rank = __popc(grp & ((1u << lane) - 1));
        const int rounds = __reduce_max_sync(0xffffffffu, valid ? __popc(grp) : 0);
        for (int q = 0; q < rounds; ++q) {
          if (valid && rank == q) my[c - c0] += s_o * v;
          __syncwarp();
        }
      }
    }
  }
  __syncthreads();
  // write the tile: column c of the output gets CSR_B consecutive buckets
  const int64_t nb = min((int64_t)CSR_B, d - i0);
  for (int64_t k = threadIdx.x; k < cw * CSR_B; k += blockDim.x) {
    const int64_t cc = k / CSR_B, b = k % CSR_B;
    if (b < nb) SA[(c0 + cc) * ldsa + i0 + b] = tile[b * ldt + cc];
  }
}

}  // namespace skl

using namespace skl;

// Host: bucket-sorted source rows (the CSR of S, sketch.py:100-102).
extern "C" int skl_countsketch_buckets(const int32_t* rows, int64_t m, int64_t d,
                                       int32_t* bucket_rows, int64_t* bucket_ptr) {
  clear_error();
  SKL_REQUIRE(rows && bucket_rows && bucket_ptr && m >= 1 && d >= 1 && m <= 0x7fffffffLL,
              SKL_ERR_INVALID, "countsketch_buckets: bad arguments");
  std::fill(bucket_ptr, bucket_ptr + d + 1, 0);
  for (int64_t j = 0; j < m; ++j) {
    const int32_t r = rows[j];
    SKL_REQUIRE(r >= 0 && r < d, SKL_ERR_INVALID, "bucket index out of range");
    ++bucket_ptr[r + 1];
  }
  for (int64_t i = 0; i < d; ++i) bucket_ptr[i + 1] += bucket_ptr[i];
  std::vector<int64_t> pos(bucket_ptr, bucket_ptr + d);
  for (int64_t j = 0; j < m; ++j) bucket_rows[pos[rows[j]]++] = (int32_t)j;
  return SKL_OK;
}

static int csr_launch(const int64_t* indptr, const int64_t* indices, const double* values,
                      int64_t m, int64_t n, const int32_t* bucket_rows, const int64_t* bucket_ptr,
                      const int8_t* signs, double scale, int64_t d, double* SA, int64_t ldsa,
                      cudaStream_t st) {
  SKL_REQUIRE(indptr && bucket_rows && bucket_ptr && signs && SA && m >= 1 && n >= 1 && d >= 1 &&
                  ldsa >= d,
              SKL_ERR_SHAPE, "countsketch_csr: bad arguments");
  // shared tile budget: up to 192 KiB
  const int64_t max_cw = (192 * 1024) / (CSR_B * 8) - 1;
  const int64_t Cw = std::min<int64_t>(n, max_cw);
  const size_t smem = (size_t)(Cw + 1) * CSR_B * sizeof(double);
  SKL_CUDA(cudaFuncSetAttribute(countsketch_csr_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)smem));
  dim3 grid((unsigned)((d + CSR_B - 1) / CSR_B), (unsigned)((n + Cw - 1) / Cw));
  countsketch_csr_kernel<<<grid, CSR_B * 32, smem, st>>>(indptr, indices, values, bucket_rows,
                                                         bucket_ptr, signs, d, n, Cw, SA, ldsa,
                                                         scale);
  SKL_CUDA_LAUNCH();
  (void)m;
  return SKL_OK;
}

extern "C" int skl_countsketch_csr(const int64_t* indptr, const int64_t* indices,
                                   const double* values, int64_t m, int64_t n,
                                   const int32_t* bucket_rows, const int64_t* bucket_ptr,
                                   const int8_t* signs, int64_t d, double* SA, int64_t ldsa,
                                   void* stream) {
  clear_error();
  return csr_launch(indptr, indices, values, m, n, bucket_rows, bucket_ptr, signs, 1.0, d, SA,
                    ldsa, (cudaStream_t)stream);
}

extern "C" int skl_sparsesign_csr(const int64_t* indptr, const int64_t* indices,
                                  const double* values, int64_t m, int64_t n,
                                  const int32_t* bucket_rows, const int64_t* bucket_ptr,
                                  const int8_t* signs, double scale, int64_t d, double* SA,
                                  int64_t ldsa, void* stream) {
  clear_error();
  return csr_launch(indptr, indices, values, m, n, bucket_rows, bucket_ptr, signs, scale, d, SA,
                    ldsa, (cudaStream_t)stream);
}
