// CountSketch apply S*A, S*b for dense column-major fp64 A on sm_100a.
//
// Reference semantics (/root/reference/pkg/src/sketchls/sketch.py:209-212):
// `op.sparse_map @ A` with the CSR map built at sketch.py:100-102; scipy's
// csr_matvecs folds, for every bucket i and column c, the signed source rows
// j with rows[j] == i in ascending j starting from +0.0.  Multiplying by a
// sign is exact, so reproducing that fold order reproduces SA bit for bit.
//
// Design (B200): one CTA owns C columns of [A | b] and streams them once,
// top to bottom, in chunks of T rows.  A producer warp issues 1-D bulk
// copies (cp.async.bulk -> UBLKCP) of each chunk's column segments and the
// chunk's block of the plan (L2-resident, shared by all CTAs) into an
// S-stage shared-memory ring guarded by full/empty mbarriers.  The running
// bucket sums live in shared memory (C x (d+1) doubles; slot d is a dummy).
// Bucket b always belongs to warp b / ceil(d/W); per chunk the plan deals
// each warp's buckets to its 32 lanes so that every lane walks the same
// number of entries ("lane lists", interleaved so a warp reads 32
// consecutive words).  An entry carries the row's byte offset, the sign and
// the bucket: when the bucket differs from the one the lane holds, the lane
// writes the held sum back and loads the new one (a lane keeps its bucket
// across chunks when the plan continues it), then every entry is one masked
// load, one XOR (exact negation) and one add -- in ascending row order per
// bucket, as scipy's csr_matvecs folds.  The plan schedules lanes so each
// step's shared-memory gathers spread over the banks.  A bucket never leaves
// its warp, so __syncwarp orders its updates across chunks; no CTA barrier
// and no atomics.  A is read from HBM exactly once with evict-first L2 hints.
// With P > 1 row partitions (few columns, long input), partial sums go to a
// workspace and are reduced in fixed partition order (deterministic, not
// bitwise).
#include <cstdlib>
#include <algorithm>
#include <vector>

#include <cuda_runtime.h>

#include "skl_common.h"
#include "skl_ptx.cuh"

namespace skl {

constexpr int CS_STAGES = 3;   // smem ring depth

struct CsParams {
  const double* A;
  int64_t lda;
  const double* b;
  int64_t n;        // columns of A
  int64_t ncols;    // n + (b != nullptr)
  int64_t row_begin, row_end;  // rows handled by this launch (row_begin % T == 0)
  const uint32_t* lanes;
  const int64_t* chunk_off;
  int max_block;    // words
  int d;
  int T;
  int head;         // per-chunk warp-offset header (u32 words)
  int P;
  double* out;      // SA (P == 1)
  int64_t ldo;
  double* outb;     // Sb (P == 1)
  double* part;     // [P][ncols][d] (P > 1)
  int accumulate;
  double scale;     // entry magnitude (sparse sign: fl(1/sqrt(s))), SCALED kernels only
};

__device__ __forceinline__ const double* cs_col(const CsParams& p, int64_t c) {
  return c < p.n ? p.A + c * p.lda : p.b;
}

template <int NT>
__device__ __forceinline__ void cs_consumer_bar() {
  asm volatile("bar.sync 1, %0;" ::"n"(NT) : "memory");
}

template <int NT, int C, bool SCALED>
__global__ void __launch_bounds__(NT + 32, 2)
    countsketch_dense_kernel(const CsParams p) {
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);
  uint64_t* empty = full + CS_STAGES;
  const int T = p.T, d = p.d;
  const int ldacc = d + 1;
  double* acc_s = reinterpret_cast<double*>(smem + 128);
  unsigned char* ring = smem + 128 + (((size_t)C * ldacc * sizeof(double) + 127) & ~(size_t)127);
  const size_t a_bytes = (size_t)C * (T + 2) * sizeof(double);
  const size_t stage_bytes = (a_bytes + (size_t)p.max_block * sizeof(uint32_t) + 127) & ~(size_t)127;

  const int tid = threadIdx.x;
  const int64_t col0 = (int64_t)blockIdx.x * C;
  const int ncol_here = (int)(p.ncols - col0 < C ? p.ncols - col0 : C);
  const int64_t ch_first = p.row_begin / T;
  const int64_t nch = (p.row_end - p.row_begin + T - 1) / T;
  const int64_t it0 = nch * blockIdx.y / p.P, it1 = nch * (blockIdx.y + 1) / p.P;
  const int64_t niter = it1 - it0;

  if (tid == 0) {
    for (int s = 0; s < CS_STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NT / 32);
    }
    fence_mbar_init();
  }
  // zero slot (index T of every staged column; never written by the copies)
  if (tid < CS_STAGES * C) {
    double* As = reinterpret_cast<double*>(ring + (tid / C) * stage_bytes);
    As[(tid % C) * (T + 2) + T] = 0.0;
  }
  __syncthreads();

  if (tid >= NT) {
    // ------------------------------ producer warp
    if (tid == NT) {
      const uint64_t pol_stream = policy_evict_first();
      const uint64_t pol_keep = policy_evict_last();
      for (int64_t it = 0; it < niter; ++it) {
        const int s = (int)(it % CS_STAGES);
        if (it >= CS_STAGES) mbar_wait(&empty[s], (uint32_t)(((it / CS_STAGES) + 1) & 1));
        const int64_t ch = ch_first + it0 + it;
        const int64_t r0 = ch * T;
        const int len = (int)(p.row_end - r0 < T ? p.row_end - r0 : T);
        const int len_even = len & ~1;
        const int64_t o0 = __ldg(p.chunk_off + ch), o1 = __ldg(p.chunk_off + ch + 1);
        unsigned char* st = ring + s * stage_bytes;
        double* As = reinterpret_cast<double*>(st);
        uint32_t* Ls = reinterpret_cast<uint32_t*>(st + a_bytes);
        const uint32_t lbytes = (uint32_t)((o1 - o0) * sizeof(uint32_t));
        if (len & 1) {
          for (int c = 0; c < ncol_here; ++c)
            As[c * (T + 2) + len - 1] = __ldg(cs_col(p, col0 + c) + r0 + len - 1);
        }
        const uint32_t total = (uint32_t)(ncol_here * len_even * sizeof(double)) + lbytes;
        mbar_arrive_expect_tx(&full[s], total);
        if (len_even) {
          for (int c = 0; c < ncol_here; ++c)
            bulk_g2s(As + c * (T + 2), cs_col(p, col0 + c) + r0,
                     (uint32_t)(len_even * sizeof(double)), &full[s], pol_stream);
        }
        bulk_g2s(Ls, p.lanes + o0, lbytes, &full[s], pol_keep);
      }
    }
    return;
  }

  // -------------------------------- consumers
  for (int i = tid; i < d; i += NT) {
#pragma unroll
    for (int c = 0; c < C; ++c) {
      double v = 0.0;
      const int64_t col = col0 + c;
      if (p.P == 1 && p.accumulate && c < ncol_here) v = col < p.n ? p.out[col * p.ldo + i] : p.outb[i];
      acc_s[c * ldacc + i] = v;
    }
  }
  cs_consumer_bar<NT>();

  const int wid = tid >> 5, lane = tid & 31;
  // The lane's current bucket and its running sum stay in registers across
  // chunks; the sum goes back to shared memory only when the plan switches
  // the lane to another bucket (or to the dummy slot d).
  int cur = d;
  double a[C];
#pragma unroll
  for (int c = 0; c < C; ++c) a[c] = 0.0;
  for (int64_t it = 0; it < niter; ++it) {
    const int s = (int)(it % CS_STAGES);
    mbar_wait(&full[s], (uint32_t)((it / CS_STAGES) & 1));
    const unsigned char* st = ring + s * stage_bytes;
    const unsigned char* Ab = st;
    const uint32_t* H = reinterpret_cast<const uint32_t*>(st + a_bytes);
    const uint32_t* Lr = H + p.head + lane;
    const int r0 = (int)H[wid], r1 = (int)H[wid + 1];
#pragma unroll 2
    for (int r = r0; r < r1; ++r) {
      const uint32_t e = Lr[r * 32];
      const unsigned char* src = Ab + (e & 0x7fffu);
      double x[C];
#pragma unroll
      for (int c = 0; c < C; ++c) {
        const uint2 w = *reinterpret_cast<const uint2*>(src + (size_t)c * (T + 2) * 8);
        x[c] = __hiloint2double((int)(w.y ^ (e & 0x80000000u)), (int)w.x);
        // fl(+-1/sqrt(s) * a) rounded on its own, as csr_matvecs forms it (no FMA)
        if (SCALED) x[c] = __dmul_rn(p.scale, x[c]);
      }
      const int b = (int)((e >> 16) & 0x7fffu);
      if (b != cur) {
#pragma unroll
        for (int c = 0; c < C; ++c) acc_s[c * ldacc + cur] = a[c];
        cur = b;
#pragma unroll
        for (int c = 0; c < C; ++c) a[c] = acc_s[c * ldacc + cur];
      }
#pragma unroll
      for (int c = 0; c < C; ++c) a[c] += x[c];
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }
#pragma unroll
  for (int c = 0; c < C; ++c) acc_s[c * ldacc + cur] = a[c];
  cs_consumer_bar<NT>();

#pragma unroll
  for (int c = 0; c < C; ++c) {
    if (c >= ncol_here) break;
    const int64_t col = col0 + c;
    for (int i = tid; i < d; i += NT) {
      const double v = acc_s[c * ldacc + i];
      if (p.P == 1) {
        if (col < p.n)
          p.out[col * p.ldo + i] = v;
        else
          p.outb[i] = v;
      } else {
        p.part[((int64_t)blockIdx.y * p.ncols + col) * d + i] = v;
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Register-owned variant (d <= 128 * warps): bucket b lives for the whole
// apply in a register of lane (b/4) % 32 of warp b/128 (slot b % 4), so no
// accumulator ever touches shared memory; per chunk each lane walks the
// union of its four buckets' rows (skl_countsketch_plan_owned), one masked
// gather + XOR + predicated add per entry.  Same fold order per bucket ->
// bitwise-equal to the reference.
constexpr int OW_MAX_STAGES = 6;  // ring depth: as many as fit in shared memory

struct OwParams {
  const double* A;
  int64_t lda;
  const double* b;
  int64_t n, ncols;
  int64_t row_begin, row_end;
  const uint16_t* lanes;
  const int64_t* chunk_off;
  int max_block;  // u16 words
  int d, T, head, P, stages;
  double* out;
  int64_t ldo;
  double* outb;
  double* part;
  int accumulate;
  double scale;  // entry value magnitude (sparse sign embedding: fl(1/sqrt(s)))
};

// SCALED: every entry is (+-scale) * A[j] rounded once, as scipy's
// csr_matvecs computes val * x for val = +-scale (sparse sign embeddings);
// CountSketch entries are +-1 (exact sign flips, no multiply).
// Predicated add into slot K of the thread's accumulators: a branch around
// the add, so ptxas emits a predicated DADD (an if-chain or predicated PTX
// add comes out as DADD + FSEL select chains, 3x the issue slots).
template <int K>
__device__ __forceinline__ void ow_add(double& a, uint32_t slot, double x) {
  asm("{\n\t.reg .pred q;\n\t"
      "setp.ne.u32 q, %1, %3;\n\t@q bra SK%=;\n\tadd.rn.f64 %0, %0, %2;\n\tSK%=:\n\t}"
      : "+d"(a)
      : "r"(slot), "d"(x), "n"(K));
}

template <int SL, int K = 0>
__device__ __forceinline__ void ow_add_all(double (&a)[SL], uint32_t slot, double x) {
  if constexpr (K < SL) {
    ow_add<K>(a[K], slot, x);
    ow_add_all<SL, K + 1>(a, slot, x);
  }
}

template <int NT, bool SCALED, int SL>
__global__ void __launch_bounds__(NT + 32, 2) countsketch_owned_kernel(const OwParams p) {
  constexpr int RB = SL == 4 ? 13 : SL == 8 ? 12 : 11;  // owned_row_bits
  constexpr uint32_t RMASK = (1u << RB) - 1u;
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);
  uint64_t* empty = full + OW_MAX_STAGES;
  const int NS = p.stages;
  const int T = p.T;
  unsigned char* ring = smem + 128;
  const size_t a_bytes = (size_t)(T + 2) * sizeof(double);
  const size_t stage_bytes = (a_bytes + (size_t)p.max_block * 2 + 127) & ~(size_t)127;
  const int tid = threadIdx.x;
  const int64_t col = blockIdx.x;
  const double* colp = col < p.n ? p.A + col * p.lda : p.b;
  const int64_t ch_first = p.row_begin / T;
  const int64_t nch = (p.row_end - p.row_begin + T - 1) / T;
  const int64_t it0 = nch * blockIdx.y / p.P, it1 = nch * (blockIdx.y + 1) / p.P;
  const int64_t niter = it1 - it0;

  if (tid == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NT / 32);
    }
    fence_mbar_init();
  }
  if (tid < NS) reinterpret_cast<double*>(ring + tid * stage_bytes)[T] = 0.0;
  __syncthreads();

  if (tid >= NT) {
    if (tid == NT) {
      const uint64_t pol_stream = policy_evict_first();
      const uint64_t pol_keep = policy_evict_last();
      int s = 0;
      uint32_t ph = 1;  // phase of empty[s] to wait for (first pass: none)
      for (int64_t it = 0; it < niter; ++it) {
        if (it >= NS) mbar_wait(&empty[s], ph);
        const int64_t ch = ch_first + it0 + it;
        const int64_t r0 = ch * T;
        const int len = (int)(p.row_end - r0 < T ? p.row_end - r0 : T);
        const int len_even = len & ~1;
        const int64_t o0 = __ldg(p.chunk_off + ch), o1 = __ldg(p.chunk_off + ch + 1);
        unsigned char* st = ring + s * stage_bytes;
        double* As = reinterpret_cast<double*>(st);
        const uint32_t lbytes = (uint32_t)((o1 - o0) * 2);
        if (len & 1) As[len - 1] = __ldg(colp + r0 + len - 1);
        mbar_arrive_expect_tx(&full[s], (uint32_t)(len_even * sizeof(double)) + lbytes);
        if (len_even)
          bulk_g2s(As, colp + r0, (uint32_t)(len_even * sizeof(double)), &full[s], pol_stream);
        bulk_g2s(st + a_bytes, p.lanes + o0, lbytes, &full[s], pol_keep);
        if (++s == NS) {
          s = 0;
          ph ^= 1u;
        }
      }
    }
    return;
  }

  const int wid = tid >> 5, lane = tid & 31;
  // slot q of this thread owns bucket tid + q * NT
  double a[SL];
#pragma unroll
  for (int q = 0; q < SL; ++q) a[q] = 0.0;
  if (p.P == 1 && p.accumulate) {
    const double* src = col < p.n ? p.out + col * p.ldo : p.outb;
#pragma unroll
    for (int q = 0; q < SL; ++q)
      if (tid + q * NT < p.d) a[q] = src[tid + q * NT];
  }
  int s = 0;
  uint32_t ph = 0;
  for (int64_t it = 0; it < niter; ++it) {
    mbar_wait(&full[s], ph);
    const unsigned char* st = ring + s * stage_bytes;
    const uint16_t* L = reinterpret_cast<const uint16_t*>(st + a_bytes);
    const int r0 = L[wid], r1 = L[wid + 1];
    const uint16_t* Lr = L + p.head + lane;
#pragma unroll 4
    for (int r = r0; r < r1; ++r) {
      const uint32_t e = Lr[r * 32];
      const uint2 w = *reinterpret_cast<const uint2*>(st + (e & RMASK) * 8);
      double x = __hiloint2double((int)(w.y ^ ((e & 0x8000u) << 16)), (int)w.x);
      if (SCALED) x = __dmul_rn(x, p.scale);
      // exactly one slot accumulates (predicated DADDs, see ow_add)
      ow_add_all<SL>(a, (e >> RB) & (SL - 1), x);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
    if (++s == NS) {
      s = 0;
      ph ^= 1u;
    }
  }
#pragma unroll
  for (int q = 0; q < SL; ++q) {
    const int bkt = tid + q * NT;
    if (bkt >= p.d) continue;
    if (p.P == 1) {
      if (col < p.n)
        p.out[col * p.ldo + bkt] = a[q];
      else
        p.outb[bkt] = a[q];
    } else {
      p.part[((int64_t)blockIdx.y * p.ncols + col) * p.d + bkt] = a[q];
    }
  }
}

// Fixed-order reduction of the P partial sketches.
__global__ void countsketch_reduce_kernel(const double* part, int P, int64_t ncols, int d,
                                          int64_t n, double* out, int64_t ldo, double* outb,
                                          int accumulate) {
  const int64_t total = ncols * d;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t col = idx / d;
    const int i = (int)(idx % d);
    double* dst = col < n ? out + col * ldo + i : outb + i;
    double s = accumulate ? *dst : 0.0;
    for (int q = 0; q < P; ++q) s += part[((int64_t)q * ncols + col) * d + i];
    *dst = s;
  }
}

static int sm_count() { return sm_count_cached(); }

template <int NT, int C>
static cudaError_t launch_cs(const CsParams& p, dim3 grid, size_t smem, cudaStream_t st) {
  auto kern = p.scale != 1.0 ? countsketch_dense_kernel<NT, C, true>
                             : countsketch_dense_kernel<NT, C, false>;
  cudaError_t e = raise_smem_limit(kern, smem);
  if (e != cudaSuccess) return e;
  e = prefer_max_shared(kern);
  if (e != cudaSuccess) return e;
  kern<<<grid, NT + 32, smem, st>>>(p);
  return cudaGetLastError();
}

static cudaError_t dispatch_cs(int nt, int C, const CsParams& p, dim3 grid, size_t smem,
                               cudaStream_t st) {
  if (nt == 256 && C == 1) return launch_cs<256, 1>(p, grid, smem, st);
  if (nt == 512 && C == 1) return launch_cs<512, 1>(p, grid, smem, st);
  if (nt == 256 && C == 2) return launch_cs<256, 2>(p, grid, smem, st);
  if (nt == 512 && C == 2) return launch_cs<512, 2>(p, grid, smem, st);
  return cudaErrorInvalidValue;
}

// Core launcher shared by the device and host-streaming entry points.
static int countsketch_launch(const double* A, int64_t m, int64_t n, int64_t lda, const double* b,
                              const uint32_t* lanes, const int64_t* chunk_off, int64_t max_block,
                              int64_t d, int64_t chunk, int warps, double* SA, int64_t ldsa,
                              double* Sb, int partitions, int accumulate, int64_t row_begin,
                              int64_t row_end, cudaStream_t st, double scale = 1.0) {
  // rows are addressed absolutely in [row_begin, row_end): the columns of
  // that window must not overlap (the host-streaming ring passes a base
  // pointer offset by -row_begin with lda = the slot height)
  SKL_REQUIRE(m >= 1 && n >= 1 && d >= 1 && lda >= row_end - row_begin && ldsa >= d, SKL_ERR_SHAPE,
              "countsketch: bad shape m=%lld n=%lld d=%lld lda=%lld ldsa=%lld", (long long)m,
              (long long)n, (long long)d, (long long)lda, (long long)ldsa);
  SKL_REQUIRE(d <= 32767, SKL_ERR_SPEC, "countsketch: embed_dim %lld > 32767 not supported",
              (long long)d);
  SKL_REQUIRE(chunk >= 8 && chunk <= 4088 && chunk % 8 == 0, SKL_ERR_INVALID,
              "countsketch: bad plan chunk %lld", (long long)chunk);
  SKL_REQUIRE(A && lanes && chunk_off && SA && (!b || Sb) && max_block > 0, SKL_ERR_INVALID,
              "countsketch: null pointer");
  SKL_REQUIRE(((uintptr_t)A & 15) == 0 && (lda % 2 == 0 || n == 1) && (!b || ((uintptr_t)b & 15) == 0),
              SKL_ERR_INVALID,
              "countsketch: A/b must be 16-byte aligned with an even leading dimension");
  SKL_REQUIRE(((uintptr_t)lanes & 15) == 0, SKL_ERR_INVALID,
              "countsketch: plan arrays must be 16-byte aligned");
  SKL_REQUIRE(row_begin % chunk == 0 && row_end > row_begin && row_end <= m, SKL_ERR_INVALID,
              "countsketch: bad row range");

  SKL_REQUIRE(warps == 8 || warps == 16, SKL_ERR_INVALID,
              "countsketch: plan built for %d warps; kernels exist for 8 and 16", warps);
  const int nthr = 32 * warps;
  const int64_t ncols = n + (b ? 1 : 0);
  int C = 1;
  const int T = (int)chunk;
  const size_t stage = ((size_t)C * (T + 2) * 8 + (size_t)max_block * 4 + 127) & ~(size_t)127;
  const size_t smem = 128 + (((size_t)C * (d + 1) * 8 + 127) & ~(size_t)127) + CS_STAGES * stage;
  SKL_REQUIRE(smem <= 227 * 1024, SKL_ERR_INVALID,
              "countsketch: chunk %d / embed_dim %lld too large for shared memory", T, (long long)d);

  const int64_t groups = (ncols + C - 1) / C;
  const int64_t nch = (row_end - row_begin + T - 1) / T;
  int P = partitions;
  if (P <= 0) {
    // Ordered single pass (bitwise-equal to the reference) unless the
    // column count leaves most SMs idle on a long input.
    const int sms = sm_count();
    const bool ordered = groups * 2 >= sms || (row_end - row_begin) <= (1 << 18);
    P = ordered ? 1 : (int)((2 * sms + groups - 1) / groups);
  }
  P = (int)std::max<int64_t>(1, std::min<int64_t>(P, nch));

  CsParams p;
  p.A = A; p.lda = lda; p.b = b; p.n = n; p.ncols = ncols;
  p.row_begin = row_begin; p.row_end = row_end;
  p.lanes = lanes; p.chunk_off = chunk_off; p.max_block = (int)max_block;
  p.d = (int)d; p.T = T; p.P = P;
  p.head = (warps + 1 + 3) / 4 * 4;
  p.out = SA; p.ldo = ldsa; p.outb = Sb; p.part = nullptr; p.accumulate = accumulate;
  p.scale = scale;

  double* part = nullptr;
  if (P > 1) {
    SKL_CUDA(malloc_async(&part, (size_t)P * ncols * d * sizeof(double), st));
    p.part = part;
  }
  dim3 grid((unsigned)groups, (unsigned)P);
  cudaError_t e = dispatch_cs(nthr, C, p, grid, smem, st);
  if (e != cudaSuccess) {
    if (part) cudaFreeAsync(part, st);
    SKL_FAIL(SKL_ERR_CUDA, "countsketch kernel launch failed: %s", cudaGetErrorString(e));
  }
  if (P > 1) {
    const int64_t total = ncols * d;
    int blocks = (int)std::min<int64_t>((total + 255) / 256, 4 * sm_count());
    countsketch_reduce_kernel<<<blocks, 256, 0, st>>>(part, P, ncols, (int)d, n, SA, ldsa, Sb,
                                                      accumulate);
    SKL_CUDA_LAUNCH();
    SKL_CUDA(cudaFreeAsync(part, st));
  }
  return SKL_OK;
}

template <int NT, bool SC, int SL>
static cudaError_t launch_owned(const OwParams& p, dim3 grid, size_t smem, cudaStream_t st) {
  auto k = countsketch_owned_kernel<NT, SC, SL>;
  cudaError_t e = raise_smem_limit(k, smem);
  if (e == cudaSuccess)
    e = prefer_max_shared(k);
  if (e != cudaSuccess) return e;
  k<<<grid, NT + 32, smem, st>>>(p);
  return cudaGetLastError();
}

template <int NT, bool SC>
static cudaError_t dispatch_owned_sl(int nsl, const OwParams& p, dim3 grid, size_t smem,
                                     cudaStream_t st) {
  switch (nsl) {
    case 4: return launch_owned<NT, SC, 4>(p, grid, smem, st);
    case 8: return launch_owned<NT, SC, 8>(p, grid, smem, st);
    default: return cudaErrorInvalidValue;
  }
}

static cudaError_t dispatch_owned(int nt, int nsl, bool scaled, const OwParams& p, dim3 grid,
                                  size_t smem, cudaStream_t st) {
  if (nt == 512)
    return scaled ? dispatch_owned_sl<512, true>(nsl, p, grid, smem, st)
                  : dispatch_owned_sl<512, false>(nsl, p, grid, smem, st);
  return scaled ? dispatch_owned_sl<256, true>(nsl, p, grid, smem, st)
                : dispatch_owned_sl<256, false>(nsl, p, grid, smem, st);
}

static int countsketch_owned_launch(const double* A, int64_t m, int64_t n, int64_t lda,
                                    const double* b, const uint16_t* lanes,
                                    const int64_t* chunk_off, int64_t max_block, int64_t d,
                                    int64_t chunk, int warps, double* SA, int64_t ldsa, double* Sb,
                                    int partitions, int accumulate, int64_t row_begin,
                                    int64_t row_end, cudaStream_t st, double scale = 1.0) {
  // rows are addressed absolutely in [row_begin, row_end): the columns of
  // that window must not overlap (the host-streaming ring passes a base
  // pointer offset by -row_begin with lda = the slot height)
  SKL_REQUIRE(m >= 1 && n >= 1 && d >= 1 && lda >= row_end - row_begin && ldsa >= d, SKL_ERR_SHAPE,
              "countsketch: bad shape m=%lld n=%lld d=%lld", (long long)m, (long long)n,
              (long long)d);
  const int nsl = owned_slots(d, warps);
  SKL_REQUIRE((warps == 8 || warps == 16) && nsl > 0, SKL_ERR_SPEC,
              "countsketch (owned): d=%lld does not fit %d warps", (long long)d, warps);
  SKL_REQUIRE(chunk >= 8 && chunk <= owned_max_chunk(nsl) && chunk % 8 == 0, SKL_ERR_INVALID,
              "countsketch: bad plan chunk %lld", (long long)chunk);
  SKL_REQUIRE(A && lanes && chunk_off && SA && (!b || Sb) && max_block > 0, SKL_ERR_INVALID,
              "countsketch: null pointer");
  SKL_REQUIRE(((uintptr_t)A & 15) == 0 && (lda % 2 == 0 || n == 1) &&
                  (!b || ((uintptr_t)b & 15) == 0) && ((uintptr_t)lanes & 15) == 0,
              SKL_ERR_INVALID,
              "countsketch: A/b/plan must be 16-byte aligned with an even leading dimension");
  SKL_REQUIRE(row_begin % chunk == 0 && row_end > row_begin && row_end <= m, SKL_ERR_INVALID,
              "countsketch: bad row range");
  const int64_t ncols = n + (b ? 1 : 0);
  const int T = (int)chunk;
  const size_t stage = ((size_t)(T + 2) * 8 + (size_t)max_block * 2 + 127) & ~(size_t)127;
  // Deepest ring that fits; with 16 warps two CTAs share an SM when the
  // ring fits half the shared memory.
  const size_t budget = 227 * 1024 - 128;
  int stages = (int)std::min<size_t>(OW_MAX_STAGES, budget / stage);
  SKL_REQUIRE(stages >= 2, SKL_ERR_INVALID, "countsketch: plan blocks too large");
  const int64_t nch = (row_end - row_begin + T - 1) / T;
  // a short column stream gains nothing from a deep ring; two stages let
  // several column CTAs share an SM so the grid fits one wave
  if (nch <= 5) stages = std::min(stages, 2);
  if (env_int("SKL_OWNED_STAGES", 0) > 0) stages = std::max(2, std::min(stages, (int)env_int("SKL_OWNED_STAGES", 0)));
  const size_t smem = 128 + stages * stage;
  int P = partitions;
  if (P <= 0) {
    const int sms = sm_count();
    const bool ordered = ncols * 2 >= sms || (row_end - row_begin) <= (1 << 18);
    P = ordered ? 1 : (int)((2 * sms + ncols - 1) / ncols);
  }
  P = (int)std::max<int64_t>(1, std::min<int64_t>(P, nch));
  OwParams p;
  p.A = A; p.lda = lda; p.b = b; p.n = n; p.ncols = ncols; p.row_begin = row_begin;
  p.row_end = row_end; p.lanes = lanes; p.chunk_off = chunk_off; p.max_block = (int)max_block;
  p.d = (int)d; p.T = T; p.head = (warps + 1 + 7) / 8 * 8; p.P = P; p.stages = stages; p.out = SA; p.ldo = ldsa;
  p.outb = Sb; p.part = nullptr; p.accumulate = accumulate; p.scale = scale;
  double* part = nullptr;
  if (P > 1) {
    SKL_CUDA(malloc_async(&part, (size_t)P * ncols * d * sizeof(double), st));
    p.part = part;
  }
  dim3 grid((unsigned)ncols, (unsigned)P);
  const bool scaled = scale != 1.0;
  const cudaError_t e = dispatch_owned(warps == 16 ? 512 : 256, nsl, scaled, p, grid, smem, st);
  if (e != cudaSuccess) {
    if (part) cudaFreeAsync(part, st);
    SKL_FAIL(SKL_ERR_CUDA, "countsketch (owned) launch failed: %s", cudaGetErrorString(e));
  }
  if (P > 1) {
    const int64_t total = ncols * d;
    int blocks = (int)std::min<int64_t>((total + 255) / 256, 4 * sm_count());
    countsketch_reduce_kernel<<<blocks, 256, 0, st>>>(part, P, ncols, (int)d, n, SA, ldsa, Sb,
                                                      accumulate);
    SKL_CUDA_LAUNCH();
    SKL_CUDA(cudaFreeAsync(part, st));
  }
  return SKL_OK;
}

}  // namespace skl

using namespace skl;

extern "C" int skl_countsketch_dense_owned(const double* A, int64_t m, int64_t n, int64_t lda,
                                           const double* b, const uint16_t* lanes,
                                           const int64_t* chunk_off, int64_t max_block, int64_t d,
                                           int64_t chunk, int warps, double* SA, int64_t ldsa,
                                           double* Sb, int partitions, int accumulate,
                                           void* stream) {
  clear_error();
  return countsketch_owned_launch(A, m, n, lda, b, lanes, chunk_off, max_block, d, chunk, warps,
                                  SA, ldsa, Sb, partitions, accumulate, 0, m, (cudaStream_t)stream);
}

extern "C" int skl_sparsesign_dense_owned(const double* A, int64_t m, int64_t n, int64_t lda,
                                          const double* b, const uint16_t* lanes,
                                          const int64_t* chunk_off, int64_t max_block, int64_t d,
                                          int64_t chunk, int warps, double scale, double* SA,
                                          int64_t ldsa, double* Sb, int partitions,
                                          int accumulate, void* stream) {
  clear_error();
  return countsketch_owned_launch(A, m, n, lda, b, lanes, chunk_off, max_block, d, chunk, warps,
                                  SA, ldsa, Sb, partitions, accumulate, 0, m, (cudaStream_t)stream,
                                  scale);
}

extern "C" int skl_sparsesign_dense(const double* A, int64_t m, int64_t n, int64_t lda,
                                    const double* b, const uint32_t* lanes,
                                    const int64_t* chunk_off, int64_t max_block, int64_t d,
                                    int64_t chunk, int warps, double scale, double* SA,
                                    int64_t ldsa, double* Sb, int partitions, int accumulate,
                                    void* stream) {
  clear_error();
  return countsketch_launch(A, m, n, lda, b, lanes, chunk_off, max_block, d, chunk, warps, SA, ldsa,
                            Sb, partitions, accumulate, 0, m, (cudaStream_t)stream, scale);
}

extern "C" int skl_countsketch_dense(const double* A, int64_t m, int64_t n, int64_t lda,
                                     const double* b, const uint32_t* lanes,
                                     const int64_t* chunk_off, int64_t max_block, int64_t d,
                                     int64_t chunk, int warps, double* SA,
                                     int64_t ldsa, double* Sb, int partitions, int accumulate,
                                     void* stream) {
  clear_error();
  return countsketch_launch(A, m, n, lda, b, lanes, chunk_off, max_block, d, chunk, warps, SA, ldsa,
                            Sb,
                            partitions,
                            accumulate, 0, m, (cudaStream_t)stream);
}

// Host-buffer apply: row blocks of A are copied host->device on a side
// stream while the kernel sketches the previous block (ordered pass,
// accumulate across blocks, so the result stays bitwise-equal).
//
// Without A_dev_keep the blocks land in a two-slot ring (2 x ~128 MiB, not a
// device copy of all of A): block k is sketched out of slot k % 2 through
// the pointer A_slot - r0 (the kernels address rows absolutely), and the copy
// of block k + 2 waits for the kernel of block k.  With A_dev_keep the blocks
// land in place and the full device copy is left for the residual pass.
// The copy stream and events are per thread and device (created once), and
// SA_out / Sb_out may be host or device memory (cudaMemcpyDefault).
struct HostStreamCtx {
  cudaStream_t cp = nullptr;
  std::vector<cudaEvent_t> ev;
};

static int host_stream_ctx(HostStreamCtx** out, size_t nev) {
  static thread_local HostStreamCtx per_dev[64];
  int dev = 0;
  SKL_CUDA(cudaGetDevice(&dev));
  SKL_REQUIRE(dev >= 0 && dev < 64, SKL_ERR_CUDA, "countsketch_host: device %d out of range", dev);
  HostStreamCtx& c = per_dev[dev];
  if (!c.cp) SKL_CUDA(cudaStreamCreateWithFlags(&c.cp, cudaStreamNonBlocking));
  while (c.ev.size() < nev) {
    cudaEvent_t e;
    SKL_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    c.ev.push_back(e);
  }
  *out = &c;
  return SKL_OK;
}

template <class Launch>
static int countsketch_host_stream(const double* A_host, int64_t m, int64_t n, int64_t lda,
                                   const double* b_host, int64_t d, int64_t chunk,
                                   double* SA_out, int64_t ldsa, double* Sb_out,
                                   double* A_dev_keep, int64_t ld_keep, double* b_dev_keep,
                                   cudaStream_t st, Launch&& launch) {
  SKL_REQUIRE(A_host && SA_out && m >= 1 && n >= 1 && lda >= m && ldsa >= d, SKL_ERR_SHAPE,
              "countsketch_host: bad arguments");
  SKL_REQUIRE(!b_host || Sb_out, SKL_ERR_INVALID, "countsketch_host: Sb_out missing");
  SKL_REQUIRE(!A_dev_keep || (ld_keep >= m && ld_keep % 2 == 0 &&
                              ((uintptr_t)A_dev_keep & 15) == 0),
              SKL_ERR_INVALID, "countsketch_host: bad A_dev_keep / ld_keep");
  // blocks of whole plan chunks, ~128 MiB of A each (chunk is even, so every
  // block start keeps the slot pointer A_slot - r0 16-byte aligned)
  static const int64_t block_mb = env_int("SKL_HOST_BLOCK_MB", 128);
  const int64_t rows_per_block =
      std::min<int64_t>((m + chunk - 1) / chunk * chunk,
                        std::max<int64_t>(chunk, ((block_mb << 20) / (8 * n)) / chunk * chunk));
  const int64_t nblk = (m + rows_per_block - 1) / rows_per_block;
  HostStreamCtx* cx = nullptr;
  int rc = host_stream_ctx(&cx, (size_t)(2 * nblk + 1));
  if (rc) return rc;
  cudaEvent_t* copied = cx->ev.data();         // [nblk]: block k on the device
  cudaEvent_t* used = cx->ev.data() + nblk;    // [nblk]: kernel of block k done
  cudaEvent_t ready = cx->ev.data()[2 * nblk];
  const int64_t ld_ring = (rows_per_block + 1) / 2 * 2;
  double* ring = nullptr;
  double* b_dev = b_dev_keep;
  double *SA_dev = nullptr, *Sb_dev = nullptr;
  if (!A_dev_keep)
    SKL_CUDA(malloc_async(&ring, (size_t)2 * ld_ring * n * sizeof(double), st));
  if (b_host && !b_dev) SKL_CUDA(malloc_async(&b_dev, (size_t)m * sizeof(double), st));
  SKL_CUDA(malloc_async(&SA_dev, (size_t)d * n * sizeof(double), st));
  if (b_host) SKL_CUDA(malloc_async(&Sb_dev, (size_t)d * sizeof(double), st));
  SKL_CUDA(cudaEventRecord(ready, st));  // allocations visible to the copy stream
  SKL_CUDA(cudaStreamWaitEvent(cx->cp, ready, 0));

  for (int64_t k = 0; k < nblk && rc == SKL_OK; ++k) {
    const int64_t r0 = k * rows_per_block, r1 = std::min(m, r0 + rows_per_block);
    double* dst;
    int64_t ld_dst;
    const double* A_base;  // pointer the kernel indexes with absolute rows
    if (A_dev_keep) {
      dst = A_dev_keep + r0;
      ld_dst = ld_keep;
      A_base = A_dev_keep;
    } else {
      double* slot = ring + (size_t)(k & 1) * ld_ring * n;
      dst = slot;
      ld_dst = ld_ring;
      A_base = slot - r0;
    }
    cudaError_t e = cudaSuccess;
    if (!A_dev_keep && k >= 2) e = cudaStreamWaitEvent(cx->cp, used[k - 2], 0);
    if (e == cudaSuccess)
      e = cudaMemcpy2DAsync(dst, ld_dst * sizeof(double), A_host + r0, lda * sizeof(double),
                            (r1 - r0) * sizeof(double), n, cudaMemcpyHostToDevice, cx->cp);
    if (e == cudaSuccess && b_host)
      e = cudaMemcpyAsync(b_dev + r0, b_host + r0, (r1 - r0) * sizeof(double),
                          cudaMemcpyHostToDevice, cx->cp);
    if (e == cudaSuccess) e = cudaEventRecord(copied[k], cx->cp);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(st, copied[k], 0);
    if (e != cudaSuccess) {
      set_error("countsketch_host: copy failed: %s", cudaGetErrorString(e));
      rc = SKL_ERR_CUDA;
      break;
    }
    rc = launch(A_base, A_dev_keep ? ld_keep : ld_ring, b_host ? b_dev : nullptr, SA_dev, Sb_dev,
                k > 0 ? 1 : 0, r0, r1);
    if (rc == SKL_OK && cudaEventRecord(used[k], st) != cudaSuccess) {
      set_error("countsketch_host: event record failed");
      rc = SKL_ERR_CUDA;
    }
  }
  // the copy stream never runs ahead of this call: join it before returning
  if (cudaEventRecord(ready, cx->cp) == cudaSuccess) cudaStreamWaitEvent(st, ready, 0);
  if (rc == SKL_OK) {
    cudaError_t e = cudaMemcpy2DAsync(SA_out, ldsa * sizeof(double), SA_dev, d * sizeof(double),
                                      d * sizeof(double), n, cudaMemcpyDefault, st);
    if (e == cudaSuccess && b_host)
      e = cudaMemcpyAsync(Sb_out, Sb_dev, d * sizeof(double), cudaMemcpyDefault, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) {
      set_error("countsketch_host: %s", cudaGetErrorString(e));
      rc = SKL_ERR_CUDA;
    }
  }
  if (ring) cudaFreeAsync(ring, st);
  if (b_host && !b_dev_keep) cudaFreeAsync(b_dev, st);
  cudaFreeAsync(SA_dev, st);
  if (Sb_dev) cudaFreeAsync(Sb_dev, st);
  return rc;
}

extern "C" int skl_countsketch_dense_host(const double* A_host, int64_t m, int64_t n, int64_t lda,
                                          const double* b_host, const uint32_t* lanes,
                                          const int64_t* chunk_off, int64_t max_block,
                                          int64_t d, int64_t chunk, int warps,
                                          double* SA_out, int64_t ldsa, double* Sb_out,
                                          double* A_dev_keep, int64_t ld_keep, double* b_dev_keep,
                                          void* stream) {
  clear_error();
  cudaStream_t st = (cudaStream_t)stream;
  return countsketch_host_stream(
      A_host, m, n, lda, b_host, d, chunk, SA_out, ldsa, Sb_out, A_dev_keep, ld_keep,
      b_dev_keep, st,
      [&](const double* A_dev, int64_t ld_dev, const double* b_dev, double* SA_dev, double* Sb_dev,
          int acc, int64_t r0, int64_t r1) {
        return countsketch_launch(A_dev, m, n, ld_dev, b_dev, lanes, chunk_off, max_block, d,
                                  chunk, warps, SA_dev, d, Sb_dev, 1, acc, r0, r1, st);
      });
}

extern "C" int skl_countsketch_dense_owned_host(
    const double* A_host, int64_t m, int64_t n, int64_t lda, const double* b_host,
    const uint16_t* lanes, const int64_t* chunk_off, int64_t max_block, int64_t d, int64_t chunk,
    int warps, double* SA_out, int64_t ldsa, double* Sb_out, double* A_dev_keep,
    int64_t ld_keep, double* b_dev_keep, void* stream) {
  clear_error();
  cudaStream_t st = (cudaStream_t)stream;
  return countsketch_host_stream(
      A_host, m, n, lda, b_host, d, chunk, SA_out, ldsa, Sb_out, A_dev_keep, ld_keep,
      b_dev_keep, st,
      [&](const double* A_dev, int64_t ld_dev, const double* b_dev, double* SA_dev, double* Sb_dev,
          int acc, int64_t r0, int64_t r1) {
        return countsketch_owned_launch(A_dev, m, n, ld_dev, b_dev, lanes, chunk_off, max_block,
                                        d, chunk, warps, SA_dev, d, Sb_dev, 1, acc, r0, r1, st);
      });
}
