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
// the CSR of S) 32 rows at a time.  The warp flattens those rows'
// nonzeros in (row, position) order and lanes gather them, one round ahead
// of the commit (software pipeline: bucket rows 3 rounds, CSR extents 2
// rounds and nonzeros 1 round ahead), then commit into the tile in
// flattened order: lanes hitting the same column are
// serialised by lane rank (__match_any_sync), distinct columns commit
// together.  The tile is then written once; the output needs no memset and
// no atomics.
#include <cuda_runtime.h>

#include <algorithm>
#include <vector>

#include "skl_common.h"

namespace skl {

constexpr int CSR_B = 8;   // buckets (warps) per CTA

// One round = 32 consecutive source rows of a bucket (lane l: row base + l).
struct CsrRound {
  int64_t q;      // first nonzero of my row minus start (nonzero f sits at q + f)
  int start;      // exclusive scan of the rows' nonzero counts (flattened index)
  int total;      // nonzeros of the round (< 2^31: n < 2^26 is checked at launch)
  int sg;         // my row's sign (+-1; 0 for a row past the bucket)
};

// A prefetched nonzero of a round's flattened order: column, value, row sign.
struct CsrSlot {
  int64_t c;
  double v, s;
  bool ok;
};

__device__ __forceinline__ CsrRound csr_round(int64_t np0, int64_t np1, int8_t sg) {
  CsrRound r;
  const int lane = threadIdx.x & 31;
  const int cnt = (int)(np1 - np0);  // 32-bit scan: one SHFL per step
  int incl = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  r.start = incl - cnt;
  r.q = np0 - r.start;
  r.total = __shfl_sync(0xffffffffu, incl, 31);
  r.sg = sg;
  return r;
}

// Issue the loads of flattened nonzero f of round r (owner lane = the
// largest l with start_l <= f; among equal starts, i.e. empty rows, the
// largest index).  The values are consumed a round later.
__device__ __forceinline__ CsrSlot csr_fetch(const CsrRound& r, int f,
                                             const int64_t* __restrict__ indices,
                                             const double* __restrict__ values, double scale) {
  int lo = 0;
#pragma unroll
  for (int step = 16; step > 0; step >>= 1) {
    const int st = __shfl_sync(0xffffffffu, r.start, min(lo + step, 31));
    if (lo + step <= 31 && st <= f) lo += step;
  }
  const int64_t q_o = __shfl_sync(0xffffffffu, r.q, lo);
  CsrSlot sl;
  // +-1 (CountSketch) or +-fl(1/sqrt(s)) (sparse sign): the same product as
  // forming the signed scale per row
  sl.s = (double)__shfl_sync(0xffffffffu, r.sg, lo) * scale;
  sl.ok = f < r.total;
  sl.c = -1;
  sl.v = 0.0;
  if (sl.ok) {
    const int64_t p = q_o + f;
    sl.c = indices[p];
    sl.v = values[p];
  }
  return sl;
}

__device__ __forceinline__ CsrSlot csr_empty() {
  CsrSlot sl;
  sl.c = -1;
  sl.v = 0.0;
  sl.s = 0.0;
  sl.ok = false;
  return sl;
}

// Add the slot into the bucket's tile row: lanes hitting the same column
// commit in lane (= flattened, = ascending source row) order.
__device__ __forceinline__ void csr_commit(const CsrSlot& sl, double* my, int64_t c0, int64_t cw) {
  const int lane = threadIdx.x & 31;
  const bool valid = sl.ok && sl.c >= c0 && sl.c < c0 + cw;
  const unsigned act = __ballot_sync(0xffffffffu, valid);
  if (!act) return;
  const unsigned peers = __match_any_sync(0xffffffffu, valid ? sl.c : -1);
  const unsigned grp = peers & act;
  const int rank = __popc(grp & ((1u << lane) - 1));
  const int rounds = __reduce_max_sync(0xffffffffu, valid ? __popc(grp) : 0);
  for (int q = 0; q < rounds; ++q) {
    if (valid && rank == q) my[sl.c - c0] += sl.s * sl.v;
    __syncwarp();
  }
}

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
    // Software pipeline over rounds of 32 rows, one round of latency for
    // every dependent load: while round r commits, the nonzeros of round
    // r+1 (two flattened passes, 64 entries), the CSR extents of round r+2
    // and the bucket-row indices of round r+3 are in flight.
    auto brow_at = [&](int64_t base) -> int32_t {
      const int64_t r = base + lane;
      return r < r_end ? brow[r] : -1;
    };
    int64_t np0 = 0, np1 = 0;
    int8_t nsg = 0;
    auto extent = [&](int32_t j, int64_t base) {
      np0 = 0;
      np1 = 0;
      nsg = 0;
      if (j >= 0) {
        np0 = indptr[j];
        np1 = indptr[j + 1];
        nsg = bsign[base + lane];
      }
    };
    // prologue: round 0 extents (dependent), round 0 nonzeros, round 1
    // extents, round 2 rows
    extent(brow_at(r_beg), r_beg);
    CsrRound cur = csr_round(np0, np1, nsg);
    CsrSlot a = csr_fetch(cur, lane, indices, values, scale);
    CsrSlot b = cur.total > 32 ? csr_fetch(cur, 32 + lane, indices, values, scale) : csr_empty();
    extent(brow_at(r_beg + 32), r_beg + 32);
    int32_t nj = brow_at(r_beg + 64);
    for (int64_t base = r_beg; base < r_end; base += 32) {
      // round r+1: extents arrived last iteration -> scan, issue its nonzeros
      const CsrRound nxt = csr_round(np0, np1, nsg);
      const CsrSlot na = csr_fetch(nxt, lane, indices, values, scale);
      // the second flattened pass only when the round has > 32 nonzeros
    // (warp-uniform; about half the rounds at ~1 nonzero per row)
      const CsrSlot nb = nxt.total > 32 ? csr_fetch(nxt, 32 + lane, indices, values, scale) : csr_empty();
      // round r+2 extents, round r+3 rows
      extent(nj, base + 64);
      nj = brow_at(base + 96);
      // commit round r
      csr_commit(a, my, c0, cw);
      if (cur.total > 32) csr_commit(b, my, c0, cw);
      for (int f0 = 64; f0 < cur.total; f0 += 32)  // rare: > 64 nonzeros in 32 rows
        csr_commit(csr_fetch(cur, f0 + lane, indices, values, scale), my, c0, cw);
      cur = nxt;
      a = na;
      b = nb;
    }
  }
  __syncthreads();
  // write the tile: column c of the output gets CSR_B consecutive buckets
  const int64_t nbk = min((int64_t)CSR_B, d - i0);
  for (int64_t k = threadIdx.x; k < cw * CSR_B; k += blockDim.x) {
    const int64_t cc = k / CSR_B, bb = k % CSR_B;
    if (bb < nbk) SA[(c0 + cc) * ldsa + i0 + bb] = tile[bb * ldt + cc];
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
  SKL_REQUIRE(n < (int64_t(1) << 26), SKL_ERR_SHAPE,
              "countsketch_csr: n = %lld columns exceeds the 2^26 limit", (long long)n);
  // shared tile budget: up to 192 KiB
  const int64_t max_cw = (192 * 1024) / (CSR_B * 8) - 1;
  int64_t Cw = std::min<int64_t>(n, max_cw);
  static const int64_t cw_knob = env_int("SKL_CSR_CW", 0);  // A/B knob: narrower column tiles
  if (cw_knob >= 8) Cw = std::min<int64_t>(Cw, cw_knob);
  const size_t smem = (size_t)(Cw + 1) * CSR_B * sizeof(double);
  SKL_CUDA(raise_smem_limit(countsketch_csr_kernel, smem));
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
