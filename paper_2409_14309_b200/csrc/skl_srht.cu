// SRHT apply and device FWHT.
//
// Reference (/root/reference/pkg/src/sketchls/sketch.py:213-223, fwht
// :152-177): pad A to m_pad = 2^L rows, multiply row j by sign_diag[j], run
// an unnormalised Sylvester-order FWHT down the rows, keep rows row_sample
// and divide by sqrt(d).  That is O(m_pad n log m_pad) flops over a padded
// m_pad x n copy of A.
//
// B200 design (fused, one pass over A): with H[p, j] = (-1)^popc(p & j) and
// j = (j_hi, j_lo) split at B = 2^b rows,
//     out[k, c] = sum_{j_hi} (-1)^popc(p_hi(k) & j_hi) * Y_{j_hi}[p_lo(k), c],
//     Y_{j_hi} = FWHT_B(sign .* A[j_hi*B : (j_hi+1)*B, c]).
// A CTA owns one column of A and streams it top to bottom in blocks of
// B = 4096 rows: a producer warp bulk-copies (cp.async.bulk) each block and
// its signs into a 2-stage smem ring; the consumers apply the signs and the
// 12 in-block butterfly stages as three register passes of 4 stages each
// (16 elements per thread, XOR-swizzled smem work buffer: conflict-free),
// then every thread gathers its KPT sampled rows p_lo(k) and accumulates them
// with the sign (-1)^popc(p_hi(k) & j_hi) in registers.  A is read from HBM
// once; nothing of size m_pad is ever written.  Row sharding across GPUs is a
// block offset (j_hi of the first local block).
//
// The butterfly here is (a+b, a-b) and the high stages are a direct signed
// sum, so results agree with the reference to rounding (~1e-15 relative),
// not bitwise.  skl_fwht_device (the fwht_inplace API) instead reproduces
// the reference's butterfly (a+b, (a+b)-2b) in its ascending stage order and
// is bitwise-equal.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>

#include "skl_common.h"
#include "skl_ptx.cuh"

extern "C" int64_t skl_srht_sign_words(int64_t B);

namespace skl {

constexpr int SR_NT = 256;
constexpr int SR_STAGES = 2;
constexpr int SR_BMAX = 4096;

__device__ __forceinline__ int sr_swz(int e) { return e ^ ((e >> 4) & 15); }

struct SrParams {
  const double* A;
  int64_t lda;
  int64_t m;          // local rows
  int64_t n;
  const uint16_t* sbits;  // packed signs: per block, one word per first-pass task
  const int64_t* sample;
  int64_t d;
  int b;              // log2 B
  int64_t jhi0;       // j_hi of the first local block
  int P;
  double* out;
  int64_t ldo;
  double* part;       // [P][n][d]
  double inv_scale_div;  // sqrt(d) (division at the end)
  int sw_block;         // packed sign words per block (multiple of 8)
  // column nA (when bcol != null) is b: the [A | b] pass of the SAA solve
  int64_t nA;
  const double* bcol;
  double* outb;
};

__device__ __forceinline__ const double* sr_src(const SrParams& p, int64_t col) {
  return col < p.nA ? p.A + col * p.lda : p.bcol;
}
__device__ __forceinline__ double* sr_dst(const SrParams& p, int64_t col) {
  return col < p.nA ? p.out + col * p.ldo : p.outb;
}

// One pass of NB butterfly stages at bits [lo, lo+NB).  FIRST reads the
// natural-layout stage buffer, applies the signs (bit i of the task's packed
// word flips element i: an XOR into the sign bit, exact) and the tail mask,
// and writes the swizzled work buffer; later passes work in place.
template <int NB, bool FIRST>
__device__ __forceinline__ void sr_pass(const double* __restrict__ in,
                                        const uint16_t* __restrict__ sw, int len,
                                        double* __restrict__ work, int lo, int B) {
  constexpr int CNT = 1 << NB;
  const int ntask = B >> NB;
  for (int task = threadIdx.x; task < ntask; task += SR_NT) {
    const int base = ((task >> lo) << (lo + NB)) | (task & ((1 << lo) - 1));
    const uint32_t mask = FIRST ? (uint32_t)sw[task] : 0u;
    double v[CNT];
#pragma unroll
    for (int i = 0; i < CNT; ++i) {
      const int e = base + (i << lo);
      if (FIRST) {
        const uint2 w = *reinterpret_cast<const uint2*>(in + e);
        const double x = __hiloint2double((int)(w.y ^ (((mask >> i) & 1u) << 31)), (int)w.x);
        v[i] = e < len ? x : 0.0;
      } else {
        v[i] = work[sr_swz(e)];
      }
    }
#pragma unroll
    for (int h = 1; h < CNT; h <<= 1) {
#pragma unroll
      for (int i = 0; i < CNT; ++i) {
        if (!(i & h)) {
          const double a = v[i], c = v[i + h];
          v[i] = a + c;
          v[i + h] = a - c;
        }
      }
    }
#pragma unroll
    for (int i = 0; i < CNT; ++i) work[sr_swz(base + (i << lo))] = v[i];
  }
}

template <bool FIRST>
__device__ __forceinline__ void sr_pass_any(int nb, const double* in, const uint16_t* sw, int len,
                                            double* work, int lo, int B) {
  switch (nb) {
    case 0: sr_pass<0, FIRST>(in, sw, len, work, lo, B); break;
    case 1: sr_pass<1, FIRST>(in, sw, len, work, lo, B); break;
    case 2: sr_pass<2, FIRST>(in, sw, len, work, lo, B); break;
    case 3: sr_pass<3, FIRST>(in, sw, len, work, lo, B); break;
    default: sr_pass<4, FIRST>(in, sw, len, work, lo, B); break;
  }
}

__device__ __forceinline__ void consumer_bar() {
  asm volatile("bar.sync 1, %0;" ::"n"(SR_NT) : "memory");
}

// FULL: B = 4096, three passes of 4 stages at bits 8, 4, 0 (compile-time);
// otherwise the generic pass plan for small m_pad.
template <int KPT, bool FULL>
__global__ void __launch_bounds__(SR_NT + 32, 1) srht_dense_kernel(const SrParams p) {
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);
  uint64_t* empty = full + SR_STAGES;
  const int B = 1 << p.b;
  const size_t soff = ((size_t)B * 8 + 15) & ~(size_t)15;  // sign words (16-byte aligned)
  const size_t stage_bytes = (soff + (size_t)p.sw_block * 2 + 127) & ~(size_t)127;
  unsigned char* ring = smem + 128;
  double* work = reinterpret_cast<double*>(ring + SR_STAGES * stage_bytes);

  const int tid = threadIdx.x;
  const int64_t col = blockIdx.x;
  const int64_t nblk = (p.m + B - 1) / B;
  const int64_t q0 = nblk * blockIdx.y / p.P, q1 = nblk * (blockIdx.y + 1) / p.P;
  const int64_t niter = q1 - q0;

  if (tid == 0) {
    for (int s = 0; s < SR_STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], SR_NT / 32);
    }
    fence_mbar_init();
  }
  __syncthreads();

  if (tid >= SR_NT) {
    if (tid == SR_NT) {
      const uint64_t pol_stream = policy_evict_first();
      const uint64_t pol_keep = policy_evict_last();
      const double* colp = sr_src(p, col);
      for (int64_t it = 0; it < niter; ++it) {
        const int s = (int)(it % SR_STAGES);
        if (it >= SR_STAGES) mbar_wait(&empty[s], (uint32_t)(((it / SR_STAGES) + 1) & 1));
        const int64_t r0 = (q0 + it) * (int64_t)B;
        const int len = (int)min((int64_t)B, p.m - r0);
        const int len_even = len & ~1;
        unsigned char* st = ring + s * stage_bytes;
        double* As = reinterpret_cast<double*>(st);
        uint16_t* Ss = reinterpret_cast<uint16_t*>(st + soff);
        const uint32_t sbytes = (uint32_t)(p.sw_block * 2);
        if (len & 1) As[len - 1] = __ldg(colp + r0 + len - 1);
        mbar_arrive_expect_tx(&full[s], (uint32_t)(len_even * 8) + sbytes);
        if (len_even) bulk_g2s(As, colp + r0, (uint32_t)(len_even * 8), &full[s], pol_stream);
        bulk_g2s(Ss, p.sbits + (q0 + it) * (int64_t)p.sw_block, sbytes, &full[s], pol_keep);
      }
    }
    return;
  }

  // sampled rows owned by this thread (row index < m_pad <= 2^32)
  double acc[KPT];
  uint32_t ps[KPT];
#pragma unroll
  for (int k = 0; k < KPT; ++k) {
    acc[k] = 0.0;
    const int64_t i = (int64_t)k * SR_NT + tid;
    ps[k] = i < p.d ? (uint32_t)p.sample[i] : 0u;
  }
  // pass plan: first pass = highest bit group (natural-layout friendly)
  const int nb_hi = p.b > 8 ? p.b - 8 : 0;
  const int nb_mid = p.b > 4 ? std::min(p.b, 8) - 4 : 0;
  const int nb_lo = std::min(p.b, 4);

  for (int64_t it = 0; it < niter; ++it) {
    const int s = (int)(it % SR_STAGES);
    mbar_wait(&full[s], (uint32_t)((it / SR_STAGES) & 1));
    const int64_t q = q0 + it;
    const int64_t r0 = q * (int64_t)B;
    const int len = (int)min((int64_t)B, p.m - r0);
    const unsigned char* st = ring + s * stage_bytes;
    const double* As = reinterpret_cast<const double*>(st);
    const uint16_t* Ss = reinterpret_cast<const uint16_t*>(st + soff);
    if (FULL) {
      sr_pass<4, true>(As, Ss, len, work, 8, SR_BMAX);
    } else if (nb_hi) {
      sr_pass_any<true>(nb_hi, As, Ss, len, work, 8, B);
    } else if (nb_mid) {
      sr_pass_any<true>(nb_mid, As, Ss, len, work, 4, B);
    } else {
      sr_pass_any<true>(nb_lo, As, Ss, len, work, 0, B);
    }
    __syncwarp();
    if ((tid & 31) == 0) mbar_arrive(&empty[s]);
    consumer_bar();
    if (FULL) {
      sr_pass<4, false>(nullptr, nullptr, 0, work, 4, SR_BMAX);
      consumer_bar();
      sr_pass<4, false>(nullptr, nullptr, 0, work, 0, SR_BMAX);
      consumer_bar();
    } else if (nb_hi && nb_mid) {
      sr_pass_any<false>(nb_mid, nullptr, nullptr, 0, work, 4, B);
      consumer_bar();
    }
    if (!FULL && (nb_hi || nb_mid)) {
      sr_pass_any<false>(nb_lo, nullptr, nullptr, 0, work, 0, B);
      consumer_bar();
    }
    const uint32_t jhi = (uint32_t)(p.jhi0 + q);
#pragma unroll
    for (int k = 0; k < KPT; ++k) {
      const uint2 w = *reinterpret_cast<const uint2*>(work + sr_swz((int)(ps[k] & (B - 1))));
      const uint32_t flip = (uint32_t)(__popc((ps[k] >> p.b) & jhi) & 1) << 31;
      acc[k] += __hiloint2double((int)(w.y ^ flip), (int)w.x);
    }
    consumer_bar();
  }

#pragma unroll
  for (int k = 0; k < KPT; ++k) {
    const int64_t i = (int64_t)k * SR_NT + tid;
    if (i >= p.d) continue;
    if (p.P == 1)
      sr_dst(p, col)[i] = acc[k] / p.inv_scale_div;
    else
      p.part[((int64_t)blockIdx.y * p.n + col) * p.d + i] = acc[k];
  }
}

// Register-resident SRHT for full 4096-row blocks (m_pad >= 4096).
//
// A group of 64 threads transforms one 4096-row block of a column; a CTA
// holds SR2_G groups (blocks q, q+1, ...).  Element e of a block (12 bits):
// thread t of the group loads e = t + 64 i, i = 0..63, straight from global
// memory (each warp load is one coalesced 256-byte segment), flips signs
// from its own 64-bit word, and runs the 12 butterfly stages as
//   bits 6..11 : in registers (over i),
//   one shared-memory transpose (rows padded to 65 doubles: conflict-free
//                both ways, immediate offsets):
//                thread t then holds e = 64 t + i,
//   bits 0..5  : in registers.
// Each thread writes back only elements some output row samples, and the
// output rows (KPT per thread) gather with the (-1)^popc(p_hi & j_hi) sign.
// The next blocks' loads are issued before the gather, so HBM streams under
// the sampling.  Shared-memory traffic: one transpose plus the sampled
// values, ~0.24 wavefronts per element (a three-pass smem FWHT needs ~0.53).
constexpr int SR2_G = 2;              // blocks (64-thread groups) per CTA
constexpr int SR2_NT = 64 * SR2_G;

// Work buffer: a 64 x 64 tile with rows padded to 65 doubles.  Element
// e = 64 r + c lives at 65 r + c, so both the row-order writes (fixed r,
// consecutive c) and the column-order reads (fixed c, consecutive r) of a warp
// hit every bank pair once, and every access is a thread base plus an
// immediate offset (no per-element address arithmetic).
constexpr int SR2_LD = 65;
constexpr int SR2_BUF = 64 * SR2_LD;
__device__ __forceinline__ int sr2_pad(int e) { return e + (e >> 6); }

template <int KPT>
__global__ void __launch_bounds__(SR2_NT, 2) srht_reg_kernel(const SrParams p) {
  extern __shared__ __align__(16) double work2[];  // [SR2_G][SR2_BUF], then sps[KPT * SR2_NT]
  __shared__ uint32_t sbm[SR_BMAX / 32];
  uint32_t* sps = reinterpret_cast<uint32_t*>(work2 + SR2_G * SR2_BUF);  // sample positions
  const int tid = threadIdx.x, g = tid >> 6, t = tid & 63;
  double* wk = work2 + g * SR2_BUF;
  const int64_t col = blockIdx.x;
  const int64_t nblk = (p.m + SR_BMAX - 1) / SR_BMAX;
  const int64_t q0 = nblk * blockIdx.y / p.P, q1 = nblk * (blockIdx.y + 1) / p.P;

  // Output rows are processed in order of their in-block position p_lo
  // (counting sort in shared memory), so a warp's 32 gathers fall in a few
  // 128-byte rows instead of 32 random ones.  skk[] keeps the output index.
  uint32_t* skk = sps + KPT * SR2_NT;
  uint32_t* cnt = reinterpret_cast<uint32_t*>(work2);  // scratch before first use
  for (int i = tid; i < SR_BMAX / 32; i += SR2_NT) sbm[i] = 0u;
  for (int i = tid; i < SR_BMAX; i += SR2_NT) cnt[i] = 0u;
  __syncthreads();
  for (int64_t i = tid; i < p.d; i += SR2_NT) {
    const uint32_t pl = (uint32_t)p.sample[i] & (SR_BMAX - 1);
    atomicAdd(&cnt[pl], 1u);
    atomicOr(&sbm[pl >> 5], 1u << (pl & 31));
  }
  __syncthreads();
  if (tid < 32) {  // exclusive scan of the 4096 counts by one warp
    uint32_t run = 0;
    for (int c = 0; c < SR_BMAX / 32; ++c) {
      const uint32_t x = cnt[c * 32 + tid];
      uint32_t y = x;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t z = __shfl_up_sync(0xffffffffu, y, o);
        if (tid >= o) y += z;
      }
      cnt[c * 32 + tid] = run + y - x;
      run += __shfl_sync(0xffffffffu, y, 31);
    }
  }
  __syncthreads();
  for (int64_t i = tid; i < p.d; i += SR2_NT) {
    const uint32_t ps = (uint32_t)p.sample[i];
    const uint32_t slot = atomicAdd(&cnt[ps & (SR_BMAX - 1)], 1u);
    sps[slot] = ps;
    skk[slot] = (uint32_t)i;
  }
  for (int64_t i = p.d + tid; i < (int64_t)KPT * SR2_NT; i += SR2_NT) {
    sps[i] = 0u;
    skk[i] = 0xffffffffu;
  }
  double acc[KPT];
#pragma unroll
  for (int k = 0; k < KPT; ++k) acc[k] = 0.0;
  __syncthreads();
  // after the transpose thread t holds e = 64 t + i: sampled bits i
  const uint64_t smask = ((uint64_t)sbm[2 * t + 1] << 32) | sbm[2 * t];
  const double* colp = sr_src(p, col);
  const uint64_t* sw64 = reinterpret_cast<const uint64_t*>(p.sbits);

  double v[64];
  auto load = [&](int64_t q) {
    const int64_t r0 = q * SR_BMAX;
    const int64_t len = q < q1 ? min((int64_t)SR_BMAX, p.m - r0) : 0;
    const double* src = colp + r0 + t;
    if (len == SR_BMAX) {  // full block: unpredicated, immediate offsets
#pragma unroll
      for (int i = 0; i < 64; ++i) v[i] = __ldcs(src + 64 * i);
    } else {
#pragma unroll
      for (int i = 0; i < 64; ++i) v[i] = t + 64 * i < len ? __ldcs(src + 64 * i) : 0.0;
    }
  };
  load(q0 + g);
  for (int64_t qb = q0; qb < q1; qb += SR2_G) {
    const int64_t q = qb + g;  // my block (may be past q1: all zeros)
    const uint64_t sw = q < q1 ? sw64[q * 64 + t] : 0ull;
#pragma unroll
    for (int i = 0; i < 64; ++i)
      v[i] = __hiloint2double(__double2hiint(v[i]) ^ (int)(((sw >> i) & 1ull) << 31),
                              __double2loint(v[i]));
    // bits 6..11
#pragma unroll
    for (int h = 1; h < 64; h <<= 1)
#pragma unroll
      for (int i = 0; i < 64; ++i)
        if (!(i & h)) {
          const double a = v[i], c = v[i + h];
          v[i] = a + c;
          v[i + h] = a - c;
        }
    __syncthreads();  // the previous iteration's gathers are done with wk
#pragma unroll
    for (int i = 0; i < 64; ++i) wk[SR2_LD * i + t] = v[i];
    asm volatile("bar.sync %0, 64;" ::"r"(1 + g) : "memory");  // group barrier
#pragma unroll
    for (int i = 0; i < 64; ++i) v[i] = wk[SR2_LD * t + i];
    // bits 0..5
#pragma unroll
    for (int h = 1; h < 64; h <<= 1)
#pragma unroll
      for (int i = 0; i < 64; ++i)
        if (!(i & h)) {
          const double a = v[i], c = v[i + h];
          v[i] = a + c;
          v[i + h] = a - c;
        }
    // owner-only rewrite of the sampled elements (no barrier needed)
#pragma unroll
    for (int i = 0; i < 64; ++i)
      if ((smask >> i) & 1ull) wk[SR2_LD * t + i] = v[i];
    load(qb + SR2_G + g);  // next blocks stream in under the gather
    __syncthreads();
#pragma unroll
    for (int gg = 0; gg < SR2_G; ++gg) {
      const int64_t qq = qb + gg;
      if (qq >= q1) break;
      const uint32_t jhi = (uint32_t)(p.jhi0 + qq);
      const double* w = work2 + gg * SR2_BUF;
#pragma unroll
      for (int k = 0; k < KPT; ++k) {
        const uint32_t ps = sps[k * SR2_NT + tid];
        const double y = w[sr2_pad((int)(ps & (SR_BMAX - 1)))];
        const uint32_t flip = (uint32_t)(__popc((ps >> 12) & jhi) & 1) << 31;
        acc[k] += __hiloint2double(__double2hiint(y) ^ (int)flip, __double2loint(y));
      }
    }
  }
#pragma unroll
  for (int k = 0; k < KPT; ++k) {
    const uint32_t kk = skk[k * SR2_NT + tid];
    if (kk == 0xffffffffu) continue;
    const int64_t i = kk;
    if (p.P == 1)
      sr_dst(p, col)[i] = acc[k] / p.inv_scale_div;
    else
      p.part[((int64_t)blockIdx.y * p.n + col) * p.d + i] = acc[k];
  }
}

__global__ void srht_reduce_kernel(const double* part, int P, int64_t n, int64_t d, double* out,
                                   int64_t ldo, double div, int64_t nA, double* outb) {
  const int64_t total = n * d;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t col = idx / d, i = idx % d;
    double s = 0.0;
    for (int q = 0; q < P; ++q) s += part[((int64_t)q * n + col) * d + i];
    (col < nA ? out + col * ldo : outb)[i] = s / div;
  }
}

// First-pass geometry for a block of B = 2^b rows: (lo bit, stages).
static void first_pass(int b, int* lo, int* nb) {
  if (b > 8) {
    *lo = 8;
    *nb = b - 8;
  } else if (b > 4) {
    *lo = 4;
    *nb = b - 4;
  } else {
    *lo = 0;
    *nb = b;
  }
}

static int block_log2(int64_t m_pad) {
  int b = 0;
  while ((1LL << (b + 1)) <= std::min<int64_t>(m_pad, SR_BMAX)) ++b;
  return b;
}

template <int KPT>
static cudaError_t launch_srht(const SrParams& p, dim3 grid, size_t smem, cudaStream_t st) {
  if (p.b == 12) {  // full blocks: register-resident kernel, KPT = d / 128 per thread
    constexpr int K2 = KPT * SR_NT / SR2_NT;
    auto kern = srht_reg_kernel<K2>;
    const int sm2 = SR2_G * SR2_BUF * 8 + 2 * K2 * SR2_NT * 4;
    cudaError_t e = raise_smem_limit(kern, (size_t)sm2);
    if (e != cudaSuccess) return e;
    kern<<<grid, SR2_NT, sm2, st>>>(p);
    return cudaGetLastError();
  }
  auto kern = srht_dense_kernel<KPT, false>;
  cudaError_t e = raise_smem_limit(kern, smem);
  if (e != cudaSuccess) return e;
  kern<<<grid, SR_NT + 32, smem, st>>>(p);
  return cudaGetLastError();
}

int srht_launch(const double* A, int64_t m, int64_t n, int64_t lda, const uint16_t* sbits,
                const int64_t* sample, int64_t m_pad, int64_t d, double* SA, int64_t ldsa,
                int64_t row_offset, int partitions, cudaStream_t st, int64_t d_scale = 0,
                const double* bvec = nullptr, double* Sb = nullptr) {
  // d_scale: the embedding dimension the 1/sqrt(d) normalisation uses (the
  // whole d when this launch covers a slice of the sampled rows)
  if (d_scale <= 0) d_scale = d;
  const int64_t* sample_ = sample;
  SKL_REQUIRE(A && sbits && sample && SA && m >= 1 && n >= 1 && d >= 1 && lda >= m && ldsa >= d,
              SKL_ERR_SHAPE, "srht: bad arguments");
  SKL_REQUIRE(!bvec == !Sb, SKL_ERR_INVALID, "srht: b and Sb go together");
  const int64_t nA = n;
  if (bvec) n = nA + 1;  // b rides along as the last column
  SKL_REQUIRE(m_pad >= 1 && (m_pad & (m_pad - 1)) == 0, SKL_ERR_SHAPE,
              "srht: padded dimension %lld is not a power of two", (long long)m_pad);
  if (d > 32 * SR_NT) {
    // more sampled rows than one launch holds in registers: one pass over A
    // per 8192 output rows (each pass samples a slice of row_sample)
    for (int64_t k0 = 0; k0 < d; k0 += 32 * SR_NT) {
      const int64_t dk = std::min<int64_t>(32 * SR_NT, d - k0);
      const int rc = srht_launch(A, m, n, lda, sbits, sample + k0, m_pad, dk, SA + k0, ldsa,
                                 row_offset, partitions, st, d_scale, bvec,
                                 Sb ? Sb + k0 : nullptr);
      if (rc) return rc;
    }
    return SKL_OK;
  }
  SKL_REQUIRE(((uintptr_t)A & 15) == 0 && (lda % 2 == 0 || n == 1) && ((uintptr_t)sbits & 15) == 0,
              SKL_ERR_INVALID, "srht: A/signs must be 16-byte aligned with an even leading dimension");
  SKL_REQUIRE(m_pad <= 0x100000000LL, SKL_ERR_SPEC, "srht: padded dimension > 2^32");
  (void)sample_;
  const int b = block_log2(m_pad);
  const int64_t B = 1LL << b;
  SKL_REQUIRE(row_offset % B == 0, SKL_ERR_INVALID, "srht: row offset not block aligned");
  int kpt = 1;
  while ((int64_t)kpt * SR_NT < d) kpt <<= 1;
  const int sw_block = (int)skl_srht_sign_words(B);
  const size_t stage = ((((size_t)B * 8 + 15) & ~(size_t)15) + (size_t)sw_block * 2 + 127) & ~(size_t)127;
  const size_t smem = 128 + SR_STAGES * stage + (size_t)B * 8;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t nblk = (m + B - 1) / B;
  int P = partitions;
  if (P <= 0) {
    if (b == 12 && 2 * n < 2 * (int64_t)sms) {
      // few long columns (a vector S b): split each column's blocks over
      // enough CTAs to fill the GPU
      P = (int)((2 * (int64_t)sms + n - 1) / n);
    } else if (b == 12) {
      // the register kernel runs 2 CTAs per SM: split the blocks of each
      // column so the grid fills whole waves (the few partial sums are
      // reduced in fixed order afterwards)
      const int64_t slots = (int64_t)sms * 2;
      double best = -1.0;
      for (int cand = 1; cand <= 8; ++cand) {
        const int64_t ctas = n * cand;
        const double eff = (double)ctas / (double)(((ctas + slots - 1) / slots) * slots);
        if (eff > best + 0.02) {
          best = eff;
          P = cand;
        }
      }
    } else {
      P = n * 2 >= sms ? 1 : (int)((2 * sms + n - 1) / n);
    }
  }
  P = (int)std::max<int64_t>(1, std::min<int64_t>(P, nblk));
  SrParams p;
  p.A = A; p.lda = lda; p.m = m; p.n = n; p.sbits = sbits; p.sample = sample; p.d = d; p.b = b;
  p.sw_block = sw_block;
  p.jhi0 = row_offset >> b; p.P = P; p.out = SA; p.ldo = ldsa; p.part = nullptr;
  p.inv_scale_div = std::sqrt((double)d_scale);
  p.nA = nA; p.bcol = bvec; p.outb = Sb;
  double* part = nullptr;
  if (P > 1) {
    SKL_CUDA(malloc_async(&part, (size_t)P * n * d * sizeof(double), st));
    p.part = part;
  }
  dim3 grid((unsigned)n, (unsigned)P);
  cudaError_t e;
  switch (kpt) {
    case 1: e = launch_srht<1>(p, grid, smem, st); break;
    case 2: e = launch_srht<2>(p, grid, smem, st); break;
    case 4: e = launch_srht<4>(p, grid, smem, st); break;
    case 8: e = launch_srht<8>(p, grid, smem, st); break;
    case 16: e = launch_srht<16>(p, grid, smem, st); break;
    default: e = launch_srht<32>(p, grid, smem, st); break;
  }
  if (e != cudaSuccess) {
    if (part) cudaFreeAsync(part, st);
    SKL_FAIL(SKL_ERR_CUDA, "srht kernel launch failed: %s", cudaGetErrorString(e));
  }
  if (P > 1) {
    const int64_t total = n * d;
    const int blocks = (int)std::min<int64_t>((total + 255) / 256, 4LL * sms);
    srht_reduce_kernel<<<blocks, 256, 0, st>>>(part, P, n, d, SA, ldsa, std::sqrt((double)d_scale),
                                               nA, Sb);
    SKL_CUDA_LAUNCH();
    SKL_CUDA(cudaFreeAsync(part, st));
  }
  return SKL_OK;
}

// ---------------------------------------------------------------- fwht_inplace
// Stages [lo, lo+nb) of the reference's FWHT, in ascending order, with its
// butterfly x' = x + y, y' = x' - 2y (sketch.py:172-175).
template <int NB>
__global__ void fwht_ref_pass_kernel(double* X, int64_t m_pad, int64_t n, int64_t lda, int lo) {
  constexpr int CNT = 1 << NB;
  const int64_t ntask = (m_pad >> NB) * n;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < ntask;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t col = t / (m_pad >> NB), task = t % (m_pad >> NB);
    const int64_t base = ((task >> lo) << (lo + NB)) | (task & ((1LL << lo) - 1));
    double* x = X + col * lda;
    double v[CNT];
#pragma unroll
    for (int i = 0; i < CNT; ++i) v[i] = x[base + ((int64_t)i << lo)];
#pragma unroll
    for (int h = 1; h < CNT; h <<= 1) {
#pragma unroll
      for (int i = 0; i < CNT; ++i) {
        if (!(i & h)) {
          const double s = v[i] + v[i + h];
          v[i + h] = s + (-2.0 * v[i + h]);
          v[i] = s;
        }
      }
    }
#pragma unroll
    for (int i = 0; i < CNT; ++i) x[base + ((int64_t)i << lo)] = v[i];
  }
}

}  // namespace skl

using namespace skl;

extern "C" int skl_srht_dense(const double* A, int64_t m, int64_t n, int64_t lda,
                              const uint16_t* sign_bits, const int64_t* row_sample, int64_t m_pad,
                              int64_t d, double* SA, int64_t ldsa, void* stream) {
  clear_error();
  return srht_launch(A, m, n, lda, sign_bits, row_sample, m_pad, d, SA, ldsa, 0, 0,
                     (cudaStream_t)stream);
}

extern "C" int skl_srht_dense_ab(const double* A, int64_t m, int64_t n, int64_t lda,
                                 const double* b, const uint16_t* sign_bits,
                                 const int64_t* row_sample, int64_t m_pad, int64_t d,
                                 int64_t row_offset, double* SA, int64_t ldsa, double* Sb,
                                 int partitions, void* stream) {
  clear_error();
  SKL_REQUIRE(b && Sb, SKL_ERR_INVALID, "srht_dense_ab: b and Sb are required");
  return srht_launch(A, m, n, lda, sign_bits, row_sample, m_pad, d, SA, ldsa, row_offset,
                     partitions, (cudaStream_t)stream, 0, b, Sb);
}

extern "C" int skl_srht_dense_shard(const double* A, int64_t m_local, int64_t n, int64_t lda,
                                    const uint16_t* signs_local, const int64_t* row_sample,
                                    int64_t m_pad, int64_t d, int64_t row_offset, double* partial,
                                    int64_t ldp, void* stream) {
  clear_error();
  // partial sums of one row block; the caller sums partials across ranks.
  // Scaling by 1/sqrt(d) is applied here as well (it is linear).
  return srht_launch(A, m_local, n, lda, signs_local, row_sample, m_pad, d, partial, ldp,
                     row_offset, 1, (cudaStream_t)stream);
}

extern "C" int skl_fwht_device(double* X, int64_t m_pad, int64_t n, int64_t lda, void* stream) {
  clear_error();
  cudaStream_t st = (cudaStream_t)stream;
  SKL_REQUIRE(X && n >= 1 && lda >= m_pad && m_pad >= 1 && (m_pad & (m_pad - 1)) == 0,
              SKL_ERR_SHAPE, "fwht requires a power-of-two length, got %lld", (long long)m_pad);
  int L = 0;
  while ((1LL << L) < m_pad) ++L;
  for (int lo = 0; lo < L; lo += 4) {
    const int nb = std::min(4, L - lo);
    const int64_t ntask = (m_pad >> nb) * n;
    const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>((ntask + 255) / 256, 4096));
    switch (nb) {
      case 1: fwht_ref_pass_kernel<1><<<blocks, 256, 0, st>>>(X, m_pad, n, lda, lo); break;
      case 2: fwht_ref_pass_kernel<2><<<blocks, 256, 0, st>>>(X, m_pad, n, lda, lo); break;
      case 3: fwht_ref_pass_kernel<3><<<blocks, 256, 0, st>>>(X, m_pad, n, lda, lo); break;
      default: fwht_ref_pass_kernel<4><<<blocks, 256, 0, st>>>(X, m_pad, n, lda, lo); break;
    }
    SKL_CUDA_LAUNCH();
  }
  return SKL_OK;
}

// Packed signs for the SRHT kernels (host): per block of B = min(m_pad, 4096)
// rows, 16-bit words (1 = negative).  Full 4096-row blocks use the register
// kernel's layout (64-bit word t, bit i = element t + 64 i, stored as four
// u16); smaller blocks one word per first-pass task, bit i = that task's
// element i.  Padded to a multiple of 8 words.
extern "C" int64_t skl_srht_sign_words(int64_t B) {
  int b = 0;
  while ((1LL << (b + 1)) <= B) ++b;
  int lo, nb;
  first_pass(b, &lo, &nb);
  const int64_t tasks = B >> nb;
  return (tasks + 7) / 8 * 8;
}

extern "C" int skl_srht_pack_signs(const int8_t* signs, int64_t m_pad, uint16_t* packed) {
  clear_error();
  SKL_REQUIRE(signs && packed && m_pad >= 1 && (m_pad & (m_pad - 1)) == 0, SKL_ERR_INVALID,
              "srht_pack_signs: bad arguments");
  const int b = block_log2(m_pad);
  const int64_t B = 1LL << b;
  int lo, nb;
  first_pass(b, &lo, &nb);
  const int64_t tasks = B >> nb, words = skl_srht_sign_words(B);
  if (b == 12) {
    // register kernel layout: per block 64 little-endian 64-bit words, word
    // t bit i = element t + 64 i of the block (as 256 u16 words)
    for (int64_t blk = 0; blk < m_pad / B; ++blk) {
      uint16_t* w = packed + blk * words;
      for (int64_t t = 0; t < 64; ++t) {
        uint64_t mask = 0;
        for (int i = 0; i < 64; ++i)
          if (signs[blk * B + t + 64 * i] < 0) mask |= 1ull << i;
        for (int h = 0; h < 4; ++h) w[t * 4 + h] = (uint16_t)(mask >> (16 * h));
      }
    }
    return SKL_OK;
  }
  for (int64_t blk = 0; blk < m_pad / B; ++blk) {
    uint16_t* w = packed + blk * words;
    for (int64_t t = 0; t < words; ++t) {
      uint32_t mask = 0;
      if (t < tasks) {
        const int64_t base = ((t >> lo) << (lo + nb)) | (t & ((1LL << lo) - 1));
        for (int i = 0; i < (1 << nb); ++i)
          if (signs[blk * B + base + ((int64_t)i << lo)] < 0) mask |= 1u << i;
      }
      w[t] = (uint16_t)mask;
    }
  }
  return SKL_OK;
}
