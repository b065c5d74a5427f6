// Gaussian sketch entries on device, bit-exact to the reference's
// `stream(key).standard_normal((d, m)) / sqrt(d)`
// (/root/reference/pkg/src/sketchls/sketch.py:94-96; generator rng.py:43-45).
//
// numpy 2.3.5's standard_normal is a 256-strip ziggurat over full 64-bit
// Philox words: the fast path consumes one word, the wedge test one more
// word per attempt, the tail (strip 0) two words per attempt, so the i-th
// normal sits at a data-dependent stream position.  Parallel generation:
//   A. the stream is cut into segments of S words; every segment is parsed
//      speculatively as if a normal started at its first word, recording
//      the start positions it finds (bitmask) and where it exits;
//   B. the true entry of segment k is the exit of segment k-1; parsing from
//      there re-synchronises with the speculative parse at the first shared
//      start (almost always within a word or two), which gives the true
//      number of normals starting in the segment;
//   C. an exclusive scan gives each segment its output offset and the
//      segment is parsed again, writing G[i, j] (row-major, ld ldg).
// Strip-0 tail values depend on log1p; the device computes them, records
// their positions, and the host recomputes those (~2.5e-4 of all draws)
// with the same libm numpy uses and patches them in.  Arithmetic follows
// numpy's C expression order with explicit _rn intrinsics (no FMA
// contraction).  The tables come from the installed numpy (_ziggurat.py).
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <mutex>
#include <thread>
#include <vector>

#include "skl_common.h"
#include "skl_philox.h"

namespace skl {

constexpr double ZIG_R = 3.6541528853610087963519472518;
constexpr double ZIG_INV_R = 0.27366123732975827203338247596;
constexpr int ZIG_S = 1024;  // words per segment
constexpr int ZIG_MASKW = ZIG_S / 32;

__constant__ uint64_t c_ki[256];
__constant__ double c_wi[256];
__constant__ double c_fi[256];
// Per-CTA shared copies: the ziggurat strip index is random per thread, and
// divergent __constant__ reads serialise across the warp (up to 32 ways).
__shared__ uint64_t s_ki[256];
__shared__ double s_wi[256];
__shared__ double s_fi[256];

__device__ __forceinline__ void zig_load_tables() {
  for (int i = threadIdx.x; i < 256; i += blockDim.x) {
    s_ki[i] = c_ki[i];
    s_wi[i] = c_wi[i];
    s_fi[i] = c_fi[i];
  }
  __syncthreads();
}

static std::mutex g_tab_mu;
static bool g_tab_set = false;
static uint64_t h_ki[256];
static double h_wi[256], h_fi[256];

struct WordStream {
  uint64_t key, blk, w0, w1, w2, w3;
  __host__ __device__ WordStream(uint64_t k) : key(k), blk(~0ULL), w0(0), w1(0), w2(0), w3(0) {}
  __host__ __device__ __forceinline__ uint64_t at(uint64_t pos) {
    const uint64_t b = pos >> 2;
    if (b != blk) {
      uint64_t w[4];
      philox_block(key, b, w);
      w0 = w[0]; w1 = w[1]; w2 = w[2]; w3 = w[3];
      blk = b;
    }
    const int q = (int)(pos & 3);
    return q == 0 ? w0 : q == 1 ? w1 : q == 2 ? w2 : w3;
  }
};

__host__ __device__ __forceinline__ double next_double_of(uint64_t w) {
  return (double)(w >> 11) * (1.0 / 9007199254740992.0);
}

#ifdef __CUDA_ARCH__
#define ZMUL(a, b) __dmul_rn((a), (b))
#define ZADD(a, b) __dadd_rn((a), (b))
#define ZSUB(a, b) __dsub_rn((a), (b))
#define ZKI s_ki
#define ZWI s_wi
#define ZFI s_fi
#else
#define ZMUL(a, b) ((a) * (b))
#define ZADD(a, b) ((a) + (b))
#define ZSUB(a, b) ((a) - (b))
#define ZKI h_ki
#define ZWI h_wi
#define ZFI h_fi
#endif

// One standard normal starting at word `pos` (numpy random_standard_normal).
// Returns the position after it; *tail is set when the strip-0 tail (log1p)
// produced the value.
template <class Stream>
__host__ __device__ __forceinline__ uint64_t zig_parse(Stream& ws, uint64_t pos, double* val,
                                                       bool* tail) {
  *tail = false;
  for (;;) {
    uint64_t r = ws.at(pos++);
    const int idx = (int)(r & 0xff);
    r >>= 8;
    const int sign = (int)(r & 1);
    const uint64_t rabs = (r >> 1) & 0x000fffffffffffffULL;
    double x = ZMUL((double)rabs, ZWI[idx]);
    if (sign) x = -x;
    if (rabs < ZKI[idx]) {
      *val = x;
      return pos;
    }
    if (idx == 0) {
      *tail = true;
      for (;;) {
        const double xx = ZMUL(-ZIG_INV_R, log1p(-next_double_of(ws.at(pos++))));
        const double yy = -log1p(-next_double_of(ws.at(pos++)));
        if (ZADD(yy, yy) > ZMUL(xx, xx)) {
          *val = ((rabs >> 8) & 1) ? -(ZADD(ZIG_R, xx)) : ZADD(ZIG_R, xx);
          return pos;
        }
      }
    }
    const double u = next_double_of(ws.at(pos++));
    const double lhs = ZADD(ZMUL(ZSUB(ZFI[idx - 1], ZFI[idx]), u), ZFI[idx]);
    if (lhs < exp(ZMUL(ZMUL(-0.5, x), x))) {
      *val = x;
      return pos;
    }
  }
}

// Per-thread window of the word stream in shared memory, refilled 16 words
// (four Philox blocks) at a time by all threads of the warp together.  A
// segment parse that pulled each word through WordStream computed a Philox
// block whenever ANY lane of the warp crossed a 4-word boundary (the lanes'
// positions drift apart as normals take 1 or more words), i.e. nearly every
// normal; here the parse runs in rounds: a converged refill, then every lane
// parses while 4 words are left in its window.  Words outside the window
// (a strip-0 tail running past it, rare) are computed directly.
constexpr int ZR_SLOTS = 32;   // window words per thread
constexpr int ZR_FILL = 16;    // words added per round
constexpr int ZR_NT = 128;     // threads per CTA of the parse kernels

struct RingStream {
  uint64_t key, hi;  // window: words [hi - ZR_SLOTS, hi) that were written
  uint64_t* ring;    // [ZR_SLOTS][ZR_NT]: word w of this thread at ring[(w % 32) * ZR_NT + tid]
  int tid;
  __device__ RingStream(uint64_t k, uint64_t start, uint64_t* r)
      : key(k), hi(start & ~3ULL), ring(r), tid(threadIdx.x) {}
  __device__ __forceinline__ void refill() {
#pragma unroll
    for (int b = 0; b < ZR_FILL / 4; ++b) {
      uint64_t w[4];
      philox_block(key, (hi >> 2) + b, w);
#pragma unroll
      for (int q = 0; q < 4; ++q) ring[((hi + 4 * b + q) & (ZR_SLOTS - 1)) * ZR_NT + tid] = w[q];
    }
    hi += ZR_FILL;
  }
  __device__ __forceinline__ uint64_t at(uint64_t pos) {
    if (pos < hi && pos + ZR_SLOTS >= hi)
      return ring[(pos & (ZR_SLOTS - 1)) * ZR_NT + tid];
    uint64_t w[4];
    philox_block(key, pos >> 2, w);
    return w[pos & 3];
  }
};

// A: speculative parse of each segment.
__global__ void __launch_bounds__(ZR_NT) zig_spec_kernel(uint64_t key, uint64_t base,
                                                         int64_t nseg, uint32_t* mask,
                                                         uint64_t* exitpos) {
  __shared__ uint64_t ring[ZR_SLOTS * ZR_NT];
  zig_load_tables();
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= nseg) return;
  const uint64_t s0 = base + (uint64_t)k * ZIG_S;
  RingStream ws(key, s0, ring);
  uint64_t pos = s0;
  uint32_t* mk = mask + k * ZIG_MASKW;
  int cur = 0;
  uint32_t bits = 0;
  while (pos < s0 + ZIG_S) {
    ws.refill();
    while (pos < s0 + ZIG_S && pos + 4 <= ws.hi) {
      const int off = (int)(pos - s0);
      const int w = off >> 5;
      while (cur < w) {
        mk[cur++] = bits;
        bits = 0;
      }
      bits |= 1u << (off & 31);
      double v;
      bool t;
      pos = zig_parse(ws, pos, &v, &t);
    }
  }
  while (cur < ZIG_MASKW) {
    mk[cur++] = bits;
    bits = 0;
  }
  exitpos[k] = pos;
}

__device__ __forceinline__ int zig_count_from(const uint32_t* mk, int off) {
  int c = __popc(mk[off >> 5] & (0xffffffffu << (off & 31)));
  for (int w = (off >> 5) + 1; w < ZIG_MASKW; ++w) c += __popc(mk[w]);
  return c;
}

// B: true per-segment counts from the true entries; flags a broken chain.
__global__ void zig_count_kernel(uint64_t key, uint64_t base, int64_t nseg, const uint32_t* mask,
                                 const uint64_t* exitpos, int64_t* count, int* bad) {
  zig_load_tables();
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= nseg) return;
  const uint64_t s0 = base + (uint64_t)k * ZIG_S;
  const uint64_t entry = k == 0 ? base : exitpos[k - 1];
  const uint32_t* mk = mask + k * ZIG_MASKW;
  int64_t cnt = 0;
  uint64_t pos = entry;
  bool synced = false;
  WordStream ws(key);
  while (pos < s0 + ZIG_S) {
    const int off = (int)(pos - s0);
    if ((mk[off >> 5] >> (off & 31)) & 1u) {
      cnt += zig_count_from(mk, off);
      synced = true;
      break;
    }
    double v;
    bool t;
    pos = zig_parse(ws, pos, &v, &t);
    ++cnt;
  }
  if (!synced && pos != exitpos[k]) atomicExch(bad, 1);
  count[k] = cnt;
}

// Exclusive scan of the per-segment counts in two passes: (1) every CTA
// scans its tile of SC_TILE counts (8 consecutive per thread, warp shuffles,
// then the warps' totals) into local prefixes and writes the tile total;
// (2) every CTA adds the sum of the tiles before it (at most a few hundred
// totals) and the last CTA writes the grand total.  (A single-CTA walk over
// the ~5e5 segments of config 3's operator took 1.15 ms.)
constexpr int SC_NT = 1024;
constexpr int SC_PER = 8;
constexpr int SC_TILE = SC_NT * SC_PER;

__global__ void __launch_bounds__(SC_NT) zig_scan_tiles_kernel(const int64_t* __restrict__ count,
                                                               int64_t nseg,
                                                               int64_t* __restrict__ offset,
                                                               int64_t* __restrict__ tile_sum) {
  __shared__ int64_t wsum[SC_NT / 32];
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  const int64_t base = (int64_t)blockIdx.x * SC_TILE + (int64_t)t * SC_PER;
  int64_t v[SC_PER];
  int64_t mine = 0;
#pragma unroll
  for (int q = 0; q < SC_PER; ++q) {
    v[q] = base + q < nseg ? count[base + q] : 0;
    mine += v[q];
  }
  int64_t incl = mine;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int64_t y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) wsum[w] = incl;
  __syncthreads();
  if (w == 0) {
    int64_t x = wsum[lane];
    int64_t xi = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t y = __shfl_up_sync(0xffffffffu, xi, o);
      if (lane >= o) xi += y;
    }
    wsum[lane] = xi - x;  // exclusive prefix of the warps
    if (lane == 31) tile_sum[blockIdx.x] = xi;
  }
  __syncthreads();
  int64_t run = wsum[w] + incl - mine;
#pragma unroll
  for (int q = 0; q < SC_PER; ++q) {
    if (base + q < nseg) offset[base + q] = run;
    run += v[q];
  }
}

__global__ void __launch_bounds__(SC_NT) zig_scan_add_kernel(int64_t* __restrict__ offset,
                                                             int64_t nseg,
                                                             const int64_t* __restrict__ tile_sum,
                                                             int ntiles, int64_t* total) {
  __shared__ int64_t pre;
  if (threadIdx.x < 32) {
    int64_t s = 0;
    for (int i = threadIdx.x; i < (int)blockIdx.x; i += 32) s += tile_sum[i];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (threadIdx.x == 0) {
      pre = s;
      if ((int)blockIdx.x == ntiles - 1) *total = s + tile_sum[blockIdx.x];
    }
  }
  __syncthreads();
  const int64_t base = (int64_t)blockIdx.x * SC_TILE;
  for (int i = threadIdx.x; i < SC_TILE; i += SC_NT)
    if (base + i < nseg) offset[base + i] += pre;
}

// offset = exclusive scan of count[0 .. nseg), *total = the sum; tile_sum
// holds ceil(nseg / SC_TILE) scratch entries.
static void zig_scan(const int64_t* count, int64_t nseg, int64_t* offset, int64_t* total,
                     int64_t* tile_sum, cudaStream_t st) {
  const int ntiles = (int)((nseg + SC_TILE - 1) / SC_TILE);
  zig_scan_tiles_kernel<<<ntiles, SC_NT, 0, st>>>(count, nseg, offset, tile_sum);
  zig_scan_add_kernel<<<ntiles, SC_NT, 0, st>>>(offset, nseg, tile_sum, ntiles, total);
}

// C: write the normals of each segment (normal t at G[(t / m) * ldg + t % m],
// divided by `div`); record strip-0 tail positions and the word after the
// last normal.
// (t_base, row0: the band variant -- normal t of the band is global normal
// t_base + t and lands at row (t_base + t) / m - row0 of G.)
__global__ void __launch_bounds__(ZR_NT) zig_write_kernel(uint64_t key, uint64_t base, int64_t nseg,
                                 const uint64_t* exitpos, const int64_t* count,
                                 const int64_t* offset, int64_t N, int64_t m, double* G,
                                 int64_t ldg, double div, int64_t* tail_t, uint64_t* tail_pos,
                                 int* tail_n, int tail_cap, uint64_t* end_word,
                                 int64_t t_base = 0, int64_t row0 = 0) {
  __shared__ uint64_t ring[1];
  zig_load_tables();
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= nseg) return;
  int64_t t = t_base + offset[k];
  const int64_t cnt = count[k];
  if (t >= N || cnt == 0) return;
  uint64_t pos = k == 0 ? base : exitpos[k - 1];
  const int64_t nq = min(cnt, N - t);  // normals this segment writes
  int64_t i = t / m - row0, j = t % m;
  // (the shared-memory window of zig_spec_kernel measured 2.2x slower here:
  // 11.9 G instructions, the refill executed ~11x more often than the
  // parse needs -- not understood; the per-word Philox path is kept)
  WordStream ws(key);
  (void)ring;
  int64_t q = 0;
  {
    while (q < nq) {
      double v;
      bool tail;
      const uint64_t start = pos;
      pos = zig_parse(ws, pos, &v, &tail);
      G[i * ldg + j] = v / div;
      if (tail) {
        const int slot = atomicAdd(tail_n, 1);
        if (slot < tail_cap) {
          tail_t[slot] = t + q;
          tail_pos[slot] = start;
        }
      }
      if (++j == m) {
        j = 0;
        ++i;
      }
      ++q;
    }
  }
  if (t + nq == N) *end_word = pos;
}

__global__ void zig_patch_kernel(const int64_t* tail_t, const double* vals, int n, int64_t m,
                                 double* G, int64_t ldg, int64_t row0 = 0) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= n) return;
  const int64_t t = tail_t[q];
  G[(t / m - row0) * ldg + t % m] = vals[q];
}

static int upload_tables(cudaStream_t st) {
  std::lock_guard<std::mutex> lk(g_tab_mu);
  SKL_REQUIRE(g_tab_set, SKL_ERR_INVALID,
              "ziggurat tables not installed (call skl_gaussian_set_tables first)");
  SKL_CUDA(cudaMemcpyToSymbolAsync(c_ki, h_ki, sizeof(h_ki), 0, cudaMemcpyHostToDevice, st));
  SKL_CUDA(cudaMemcpyToSymbolAsync(c_wi, h_wi, sizeof(h_wi), 0, cudaMemcpyHostToDevice, st));
  SKL_CUDA(cudaMemcpyToSymbolAsync(c_fi, h_fi, sizeof(h_fi), 0, cudaMemcpyHostToDevice, st));
  return SKL_OK;
}

}  // namespace skl

using namespace skl;

extern "C" int skl_gaussian_set_tables(const uint64_t* ki, const double* wi, const double* fi) {
  clear_error();
  SKL_REQUIRE(ki && wi && fi, SKL_ERR_INVALID, "gaussian tables: null pointer");
  std::lock_guard<std::mutex> lk(g_tab_mu);
  std::copy(ki, ki + 256, h_ki);
  std::copy(wi, wi + 256, h_wi);
  std::copy(fi, fi + 256, h_fi);
  g_tab_set = true;
  return SKL_OK;
}

extern "C" int skl_rng_gaussian_host(uint64_t key, int64_t count, double* out) {
  clear_error();
  SKL_REQUIRE(count >= 0 && (count == 0 || out), SKL_ERR_INVALID, "gaussian_host: bad arguments");
  {
    std::lock_guard<std::mutex> lk(g_tab_mu);
    SKL_REQUIRE(g_tab_set, SKL_ERR_INVALID, "ziggurat tables not installed");
  }
  WordStream ws(key);
  uint64_t pos = 0;
  for (int64_t i = 0; i < count; ++i) {
    bool tail;
    pos = zig_parse(ws, pos, &out[i], &tail);
  }
  return SKL_OK;
}

// Recompute strip-0 tail values on the host (the host libm's log1p, as
// numpy's): out[q] = the normal starting at word pos[q], divided by div.
// The ~2.6e-4 of draws that take the tail are independent: spread over the
// host cores (one thread took 9 ms for config 3's ~1.4e5 tails).
static void recompute_tails_host(uint64_t key, const uint64_t* pos, double* out, int ntail,
                                 double div) {
  auto work = [&](int lo, int hi) {
    for (int q = lo; q < hi; ++q) {
      WordStream ws(key);
      bool tl;
      double v;
      zig_parse(ws, pos[q], &v, &tl);
      out[q] = v / div;
    }
  };
  const int nth = std::max(1, std::min(resolve_threads(0), ntail / 2048));
  if (nth == 1) {
    work(0, ntail);
    return;
  }
  std::vector<std::thread> th;
  for (int t = 0; t < nth; ++t)
    th.emplace_back(work, (int)((int64_t)ntail * t / nth), (int)((int64_t)ntail * (t + 1) / nth));
  for (auto& x : th) x.join();
}

// Normals [first normal at word `start`] of Generator(Philox(key)) laid out
// as `rows` x `cols` C-order (normal t at out[(t / cols) * ld + t % cols]),
// divided by `div`; *end_word receives the stream word after the last one.
static int normals_device(uint64_t key, uint64_t start, int64_t rows, int64_t cols, double* G,
                          int64_t ldg, double div, uint64_t* end_word, cudaStream_t st) {
  static const bool probe = env_flag("SKL_ZIG_PROBE");
  const auto t_start = std::chrono::steady_clock::now();
  auto ms_since = [&]() {
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_start)
        .count();
  };
  int rc = upload_tables(st);
  if (rc) return rc;
  const int64_t N = rows * cols;
  const int64_t m = cols;
  // expected words per normal ~1.025; start with 3% slack
  int64_t nseg = (int64_t)((double)N * 1.03 / ZIG_S) + 8;
  for (int attempt = 0; attempt < 4; ++attempt) {
    uint32_t* mask = nullptr;
    uint64_t* exitpos = nullptr;
    int64_t *count = nullptr, *offset = nullptr, *total = nullptr;
    int* flags = nullptr;  // [0] bad chain, [1] tail count
    const int tail_cap = (int)std::min<int64_t>(N / 256 + 4096, 1 << 26);
    int64_t* tail_t = nullptr;
    uint64_t* tail_pos = nullptr;
    uint64_t* endw = nullptr;
    SKL_CUDA(malloc_async(&mask, (size_t)nseg * ZIG_MASKW * 4, st));
    SKL_CUDA(malloc_async(&exitpos, (size_t)nseg * 8, st));
    SKL_CUDA(malloc_async(&count, (size_t)nseg * 8, st));
    SKL_CUDA(malloc_async(&offset, (size_t)nseg * 8, st));
    SKL_CUDA(malloc_async(&total, 8 * (1 + (nseg + SC_TILE - 1) / SC_TILE), st));
    SKL_CUDA(malloc_async(&flags, 8, st));
    SKL_CUDA(malloc_async(&tail_t, (size_t)tail_cap * 8, st));
    SKL_CUDA(malloc_async(&tail_pos, (size_t)tail_cap * 8, st));
    SKL_CUDA(malloc_async(&endw, 8, st));
    SKL_CUDA(cudaMemsetAsync(flags, 0, 8, st));
    const int tb = 128;
    const int blocks = (int)((nseg + tb - 1) / tb);
    zig_spec_kernel<<<blocks, tb, 0, st>>>(key, start, nseg, mask, exitpos);
    zig_count_kernel<<<blocks, tb, 0, st>>>(key, start, nseg, mask, exitpos, count, flags);
    zig_scan(count, nseg, offset, total, total + 1, st);
    int64_t h_total = 0;
    int h_flags[2] = {0, 0};
    SKL_CUDA(cudaMemcpyAsync(&h_total, total, 8, cudaMemcpyDeviceToHost, st));
    SKL_CUDA(cudaMemcpyAsync(h_flags, flags, 8, cudaMemcpyDeviceToHost, st));
    SKL_CUDA(cudaStreamSynchronize(st));
    if (probe) fprintf(stderr, "zig: counts ready %.3f ms\n", ms_since());
    auto release = [&]() {
      cudaFreeAsync(mask, st); cudaFreeAsync(exitpos, st); cudaFreeAsync(count, st);
      cudaFreeAsync(offset, st); cudaFreeAsync(total, st); cudaFreeAsync(flags, st);
      cudaFreeAsync(tail_t, st); cudaFreeAsync(tail_pos, st); cudaFreeAsync(endw, st);
    };
    if (h_flags[0]) {
      release();
      SKL_FAIL(SKL_ERR_CUDA, "gaussian: ziggurat segment chain failed to resynchronise");
    }
    if (h_total < N) {  // not enough words drawn: retry with more segments
      release();
      nseg = nseg + nseg / 8 + 16;
      continue;
    }
    zig_write_kernel<<<blocks, tb, 0, st>>>(key, start, nseg, exitpos, count, offset, N, m, G, ldg,
                                             div, tail_t, tail_pos, flags + 1, tail_cap, endw);
    SKL_CUDA_LAUNCH();
    uint64_t h_end = 0;
    SKL_CUDA(cudaMemcpyAsync(h_flags, flags, 8, cudaMemcpyDeviceToHost, st));
    SKL_CUDA(cudaMemcpyAsync(&h_end, endw, 8, cudaMemcpyDeviceToHost, st));
    SKL_CUDA(cudaStreamSynchronize(st));
    const int ntail = h_flags[1];
    if (probe) fprintf(stderr, "zig: written %.3f ms, %d tails\n", ms_since(), ntail);
    if (ntail > tail_cap) {
      release();
      SKL_FAIL(SKL_ERR_CUDA, "gaussian: tail record overflow (%d > %d)", ntail, tail_cap);
    }
    if (ntail > 0) {
      // host recomputation of the strip-0 tail values with the host libm
      std::vector<int64_t> ht((size_t)ntail);
      std::vector<uint64_t> hp((size_t)ntail);
      std::vector<double> hv((size_t)ntail);
      SKL_CUDA(cudaMemcpyAsync(ht.data(), tail_t, (size_t)ntail * 8, cudaMemcpyDeviceToHost, st));
      SKL_CUDA(cudaMemcpyAsync(hp.data(), tail_pos, (size_t)ntail * 8, cudaMemcpyDeviceToHost, st));
      SKL_CUDA(cudaStreamSynchronize(st));
      recompute_tails_host(key, hp.data(), hv.data(), ntail, div);
      double* dv = nullptr;
      SKL_CUDA(malloc_async(&dv, (size_t)ntail * 8, st));
      SKL_CUDA(cudaMemcpyAsync(dv, hv.data(), (size_t)ntail * 8, cudaMemcpyHostToDevice, st));
      zig_patch_kernel<<<(ntail + 255) / 256, 256, 0, st>>>(tail_t, dv, ntail, m, G, ldg);
      SKL_CUDA_LAUNCH();
      SKL_CUDA(cudaFreeAsync(dv, st));
      SKL_CUDA(cudaStreamSynchronize(st));  // host vectors go out of scope
    }
    release();
    if (end_word) *end_word = h_end;
    if (probe) fprintf(stderr, "zig: done %.3f ms\n", ms_since());
    return SKL_OK;
  }
  SKL_FAIL(SKL_ERR_CUDA, "gaussian: stream segmentation did not converge");
}

extern "C" int skl_rng_gaussian_device(uint64_t key, int64_t d, int64_t m, double* G, int64_t ldg,
                                       void* stream) {
  clear_error();
  SKL_REQUIRE(d >= 1 && m >= 1 && ldg >= m && G, SKL_ERR_SHAPE, "gaussian: bad arguments");
  return normals_device(key, 0, d, m, G, ldg, std::sqrt((double)d), nullptr, (cudaStream_t)stream);
}

extern "C" int skl_rng_normal_device(uint64_t key, uint64_t start_word, int64_t rows, int64_t cols,
                                     double* out, int64_t ld, uint64_t* end_word, void* stream) {
  clear_error();
  SKL_REQUIRE(rows >= 1 && cols >= 1 && ld >= cols && out, SKL_ERR_SHAPE,
              "normal_device: bad arguments");
  return normals_device(key, start_word, rows, cols, out, ld, 1.0, end_word, (cudaStream_t)stream);
}

// ---------------------------------------------------------------------------
// Banded generation for a multi-device operator (multidevice.py): device k
// parses only segments [seg0, seg1) of the stream.  begin(): speculative
// parse of [seg0 - 1, seg1) -- the extra segment gives the true entry of
// seg0, which is the speculative exit of seg0 - 1 because the true chain
// merges with it inside that segment (checked by the count of the device
// owning seg0 - 1, which reports a broken chain otherwise) -- and the true
// counts; *count = normals starting in the band.  After the host's prefix
// sum over the bands, write() stores band normal q (global t = first + q,
// t < N) at G[(t / m - row0) * ldg + t % m], recomputes the strip-0 tails on
// the host, and frees the band.
namespace skl {
struct GaussBand {
  uint64_t key = 0;
  uint64_t base = 0;  // first word parsed (segment seg0 - 1, or 0)
  int64_t nseg = 0;   // segments parsed (incl. the entry segment)
  uint32_t* mask = nullptr;
  uint64_t* exitpos = nullptr;
  int64_t *count = nullptr, *offset = nullptr, *total = nullptr;
  int* flags = nullptr;
  void release(cudaStream_t st) {
    cudaFreeAsync(mask, st); cudaFreeAsync(exitpos, st); cudaFreeAsync(count, st);
    cudaFreeAsync(offset, st); cudaFreeAsync(total, st); cudaFreeAsync(flags, st);
  }
};
}  // namespace skl

extern "C" int64_t skl_gaussian_segment_words(void) { return ZIG_S; }

extern "C" int skl_gaussian_band_begin(uint64_t key, int64_t seg0, int64_t seg1, void** handle,
                                       int64_t* count, void* stream) {
  clear_error();
  SKL_REQUIRE(handle && seg0 >= 0 && seg1 > seg0, SKL_ERR_INVALID,
              "gaussian_band_begin: bad arguments");
  cudaStream_t st = (cudaStream_t)stream;
  int rc = upload_tables(st);
  if (rc) return rc;
  GaussBand* b = new GaussBand();
  b->key = key;
  const int64_t pre = seg0 > 0 ? 1 : 0;
  b->base = (uint64_t)(seg0 - pre) * ZIG_S;
  b->nseg = seg1 - seg0 + pre;
  const int64_t nseg = b->nseg;
  auto fail = [&](const char* what, cudaError_t e) {
    b->release(st);
    delete b;
    SKL_FAIL(SKL_ERR_CUDA, "gaussian_band_begin: %s: %s", what, cudaGetErrorString(e));
  };
  cudaError_t e;
  if ((e = malloc_async(&b->mask, (size_t)nseg * ZIG_MASKW * 4, st)) != cudaSuccess) return fail("alloc", e);
  if ((e = malloc_async(&b->exitpos, (size_t)nseg * 8, st)) != cudaSuccess) return fail("alloc", e);
  if ((e = malloc_async(&b->count, (size_t)nseg * 8, st)) != cudaSuccess) return fail("alloc", e);
  if ((e = malloc_async(&b->offset, (size_t)nseg * 8, st)) != cudaSuccess) return fail("alloc", e);
  if ((e = malloc_async(&b->total, 8 * (1 + (nseg + SC_TILE - 1) / SC_TILE), st)) != cudaSuccess)
    return fail("alloc", e);
  if ((e = malloc_async(&b->flags, 8, st)) != cudaSuccess) return fail("alloc", e);
  cudaMemsetAsync(b->flags, 0, 8, st);
  const int tb = 128;
  const int blocks = (int)((nseg + tb - 1) / tb);
  zig_spec_kernel<<<blocks, tb, 0, st>>>(key, b->base, nseg, b->mask, b->exitpos);
  zig_count_kernel<<<blocks, tb, 0, st>>>(key, b->base, nseg, b->mask, b->exitpos, b->count,
                                          b->flags);
  if (pre) cudaMemsetAsync(b->count, 0, 8, st);  // the entry segment is the previous band's
  zig_scan(b->count, nseg, b->offset, b->total, b->total + 1, st);
  if ((e = cudaGetLastError()) != cudaSuccess) return fail("launch", e);
  *handle = b;
  (void)count;
  return SKL_OK;
}

// The band's normal count (synchronises the stream; fails if the chain of
// this band did not resynchronise).
extern "C" int skl_gaussian_band_count(void* handle, int64_t* count, void* stream) {
  clear_error();
  SKL_REQUIRE(handle && count, SKL_ERR_INVALID, "gaussian_band_count: bad arguments");
  GaussBand* b = static_cast<GaussBand*>(handle);
  cudaStream_t st = (cudaStream_t)stream;
  int h_flags[2] = {0, 0};
  SKL_CUDA(cudaMemcpyAsync(count, b->total, 8, cudaMemcpyDeviceToHost, st));
  SKL_CUDA(cudaMemcpyAsync(h_flags, b->flags, 8, cudaMemcpyDeviceToHost, st));
  SKL_CUDA(cudaStreamSynchronize(st));
  SKL_REQUIRE(!h_flags[0], SKL_ERR_CUDA,
              "gaussian: ziggurat segment chain failed to resynchronise");
  return SKL_OK;
}

extern "C" int skl_gaussian_band_write(void* handle, int64_t first, int64_t N, int64_t m,
                                       int64_t row0, double* G, int64_t ldg, double div,
                                       void* stream) {
  clear_error();
  SKL_REQUIRE(handle && G && m >= 1 && ldg >= m && first >= 0 && N >= 1 && div > 0.0,
              SKL_ERR_INVALID, "gaussian_band_write: bad arguments");
  GaussBand* b = static_cast<GaussBand*>(handle);
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t nseg = b->nseg;
  const int tail_cap = (int)std::min<int64_t>(nseg * ZIG_S / 256 + 4096, 1 << 26);
  int64_t* tail_t = nullptr;
  uint64_t* tail_pos = nullptr;
  uint64_t* endw = nullptr;
  int rc = SKL_OK;
  do {
    cudaError_t e;
    if ((e = malloc_async(&tail_t, (size_t)tail_cap * 8, st)) != cudaSuccess ||
        (e = malloc_async(&tail_pos, (size_t)tail_cap * 8, st)) != cudaSuccess ||
        (e = malloc_async(&endw, 8, st)) != cudaSuccess) {
      set_error("gaussian_band_write: alloc: %s", cudaGetErrorString(e));
      rc = SKL_ERR_CUDA;
      break;
    }
    cudaMemsetAsync(b->flags, 0, 8, st);
    const int tb = 128;
    const int blocks = (int)((nseg + tb - 1) / tb);
    zig_write_kernel<<<blocks, tb, 0, st>>>(b->key, b->base, nseg, b->exitpos, b->count,
                                            b->offset, N, m, G, ldg, div, tail_t, tail_pos,
                                            b->flags + 1, tail_cap, endw, first, row0);
    int h_flags[2] = {0, 0};
    if ((e = cudaGetLastError()) != cudaSuccess ||
        (e = cudaMemcpyAsync(h_flags, b->flags, 8, cudaMemcpyDeviceToHost, st)) != cudaSuccess ||
        (e = cudaStreamSynchronize(st)) != cudaSuccess) {
      set_error("gaussian_band_write: %s", cudaGetErrorString(e));
      rc = SKL_ERR_CUDA;
      break;
    }
    const int ntail = h_flags[1];
    if (ntail > tail_cap) {
      set_error("gaussian: tail record overflow (%d > %d)", ntail, tail_cap);
      rc = SKL_ERR_CUDA;
      break;
    }
    if (ntail > 0) {
      std::vector<int64_t> ht((size_t)ntail);
      std::vector<uint64_t> hp((size_t)ntail);
      std::vector<double> hv((size_t)ntail);
      cudaMemcpyAsync(ht.data(), tail_t, (size_t)ntail * 8, cudaMemcpyDeviceToHost, st);
      cudaMemcpyAsync(hp.data(), tail_pos, (size_t)ntail * 8, cudaMemcpyDeviceToHost, st);
      if ((e = cudaStreamSynchronize(st)) != cudaSuccess) {
        set_error("gaussian_band_write: %s", cudaGetErrorString(e));
        rc = SKL_ERR_CUDA;
        break;
      }
      recompute_tails_host(b->key, hp.data(), hv.data(), ntail, div);
      double* dv = nullptr;
      if ((e = malloc_async(&dv, (size_t)ntail * 8, st)) != cudaSuccess) {
        set_error("gaussian_band_write: alloc: %s", cudaGetErrorString(e));
        rc = SKL_ERR_CUDA;
        break;
      }
      cudaMemcpyAsync(dv, hv.data(), (size_t)ntail * 8, cudaMemcpyHostToDevice, st);
      zig_patch_kernel<<<(ntail + 255) / 256, 256, 0, st>>>(tail_t, dv, ntail, m, G, ldg, row0);
      cudaFreeAsync(dv, st);
      cudaStreamSynchronize(st);  // host vectors go out of scope
    }
  } while (0);
  if (tail_t) cudaFreeAsync(tail_t, st);
  if (tail_pos) cudaFreeAsync(tail_pos, st);
  if (endw) cudaFreeAsync(endw, st);
  b->release(st);
  delete b;
  return rc;
}

extern "C" void skl_gaussian_band_free(void* handle, void* stream) {
  if (!handle) return;
  GaussBand* b = static_cast<GaussBand*>(handle);
  b->release((cudaStream_t)stream);
  delete b;
}
