// CountSketch operator construction on the device: the hash/sign draws
// (sketch.py:97-99: integers(0, d, m), integers(0, 2, m) on numpy's u32
// Philox stream) and the register-owned apply plan (skl_plan_owned.cpp).
// Both are bit-identical to the host builders, which stay the reference
// implementation; this path removes ~5 ms of host work (and the plan's
// host->device copy) from every cold solve, where the reference rebuilds the
// operator each time.
//
// Draws: u32 stream position p is half (p & 1, low first) of u64 word
// (p >> 1) & 3 of Philox block p >> 3.  Row j is Lemire's 32-bit bounded
// draw at position j when no earlier draw was rejected; rejections
// (probability ((2^32 - d) mod d) / 2^32 per draw, 0 for power-of-two d) are
// counted, and in that rare case the host builder is used instead.  Signs
// are the top bits of positions m + R + j.
//
// Plan: one CTA per chunk.  Pass 1 histograms the chunk's buckets and sizes
// each warp's block (longest lane over its four buckets).  Pass 2 sorts the
// chunk's (bucket, row) keys in shared memory (bitonic), so every bucket's
// rows are ascending, and lane 0 of each warp runs the host planner's greedy
// bank-balancing merge of its lanes' four streams, step by step, in the same
// order -- the output words are identical to skl_countsketch_plan_owned.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <vector>

#include "skl_common.h"
#include "skl_philox.h"

extern "C" int skl_rng_countsketch(uint64_t key, int64_t m, int64_t d, int32_t* rows,
                                   int8_t* signs, int threads, uint64_t* u32_consumed);

namespace skl {

__device__ __forceinline__ uint32_t u32_at(const uint64_t w[4], uint64_t p) {
  const uint64_t word = w[(p >> 1) & 3];
  return (p & 1) ? (uint32_t)(word >> 32) : (uint32_t)word;
}

// rows[j] for positions [0, m): 8 positions (one Philox block) per thread.
__global__ void cs_rows_kernel(uint64_t key, int64_t m, uint64_t d, uint32_t threshold,
                               int32_t* __restrict__ rows, unsigned long long* rejections) {
  const int64_t nblk = (m + 7) / 8;
  unsigned long long rej = 0;
  for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < nblk;
       b += (int64_t)gridDim.x * blockDim.x) {
    uint64_t w[4];
    philox_block(key, (uint64_t)b, w);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int64_t j = b * 8 + i;
      if (j >= m) break;
      const uint64_t prod = (uint64_t)u32_at(w, (uint64_t)j) * d;
      if ((uint32_t)prod < threshold) ++rej;
      rows[j] = (int32_t)(prod >> 32);
    }
  }
  if (rej) atomicAdd(rejections, rej);
}

// signs[j] = top bit of u32 at position pos0 + j ? +1 : -1.
__global__ void cs_signs_kernel(uint64_t key, int64_t m, uint64_t pos0, int8_t* __restrict__ signs) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < m;
       j += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t p = pos0 + (uint64_t)j;
    uint64_t w[4];
    philox_block(key, p >> 3, w);
    signs[j] = (u32_at(w, p) >> 31) ? 1 : -1;
  }
}

constexpr int PB_NT = 512;
constexpr int PB_KEYS = 8192;  // chunk <= 8184 rows (+ pads), power of two

__device__ __forceinline__ int pb_head(int warps) { return (warps + 1 + 7) / 8 * 8; }

// Pass 1: per-warp list lengths and block size of every chunk.
__global__ void __launch_bounds__(PB_NT) owned_sizes_kernel(const int32_t* __restrict__ rows,
                                                            int64_t m, int d, int chunk, int warps,
                                                            int nsl, int32_t* __restrict__ maxlen,
                                                            int64_t* __restrict__ sizes) {
  extern __shared__ int32_t cnt[];  // [d]
  __shared__ int32_t wmax[32];
  const int64_t k = blockIdx.x, r0 = k * chunk;
  const int len = (int)min((int64_t)chunk, m - r0);
  for (int b = threadIdx.x; b < d; b += PB_NT) cnt[b] = 0;
  __syncthreads();
  for (int j = threadIdx.x; j < len; j += PB_NT) atomicAdd(&cnt[rows[r0 + j]], 1);
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int w = wid; w < warps; w += PB_NT / 32) {
    int tot = 0;
    for (int s = 0; s < nsl; ++s) {
      const int b = w * 32 + lane + s * 32 * warps;
      if (b < d) tot += cnt[b];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) tot = max(tot, __shfl_xor_sync(0xffffffffu, tot, o));
    if (lane == 0) {
      maxlen[k * warps + w] = tot;
      wmax[w] = tot;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int64_t total = 0;
    for (int w = 0; w < warps; ++w) total += wmax[w];
    sizes[k] = pb_head(warps) + total * 32;
  }
}

// exclusive scan of the chunk sizes -> chunk_off[0..nch], max size -> *mx
__global__ void owned_scan_kernel(const int64_t* __restrict__ sizes, int64_t nch,
                                  int64_t* __restrict__ off, int64_t* mx) {
  if (threadIdx.x != 0) return;
  int64_t run = 0, best = 0;
  for (int64_t k = 0; k < nch; ++k) {
    off[k] = run;
    run += sizes[k];
    best = max(best, sizes[k]);
  }
  off[nch] = run;
  *mx = best;
}

// Pass 2: the plan words of every chunk (same format and greedy as the host).
template <int SL>
__global__ void __launch_bounds__(PB_NT) owned_fill_kernel(
    const int32_t* __restrict__ rows, const int8_t* __restrict__ signs, int64_t m, int d,
    int chunk, int warps, const int32_t* __restrict__ maxlen, const int64_t* __restrict__ off,
    uint16_t* __restrict__ lanes) {
  extern __shared__ uint32_t keys[];  // [PB_KEYS], then start[d], cnt[d], the chunk's signs
  int32_t* start = reinterpret_cast<int32_t*>(keys + PB_KEYS);
  int32_t* cnt = start + d;
  int8_t* sg = reinterpret_cast<int8_t*>(cnt + d);  // [chunk] signs of the chunk's rows
  const int64_t k = blockIdx.x, r0 = k * chunk;
  const int len = (int)min((int64_t)chunk, m - r0);
  const int tid = threadIdx.x;
  for (int i = tid; i < PB_KEYS; i += PB_NT)
    keys[i] = i < len ? ((uint32_t)rows[r0 + i] << 13) | (uint32_t)i : 0xffffffffu;
  for (int i = tid; i < len; i += PB_NT) sg[i] = signs[r0 + i];
  for (int b = tid; b < d; b += PB_NT) cnt[b] = 0;
  __syncthreads();
  // bitonic sort of the keys (ascending: bucket, then row)
  for (int size = 2; size <= PB_KEYS; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = tid; i < PB_KEYS / 2; i += PB_NT) {
        const int lo = 2 * i - (i & (stride - 1));
        const int hi = lo + stride;
        const bool up = ((lo & size) == 0);
        const uint32_t a = keys[lo], c = keys[hi];
        if ((a > c) == up) {
          keys[lo] = c;
          keys[hi] = a;
        }
      }
      __syncthreads();
    }
  }
  for (int j = tid; j < len; j += PB_NT) atomicAdd(&cnt[keys[j] >> 13], 1);
  __syncthreads();
  {
    // exclusive scan of cnt[0..d) into start[]: each thread a run of
    // consecutive buckets, then warp and block scans of the run totals
    __shared__ int32_t wsum[PB_NT / 32];
    const int per = (d + PB_NT - 1) / PB_NT;
    const int b0 = tid * per, b1 = min(d, b0 + per);
    int32_t own = 0;
    for (int b = b0; b < b1; ++b) own += cnt[b];
    const int lane = tid & 31, wid = tid >> 5;
    int32_t incl = own;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int32_t y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    if (lane == 31) wsum[wid] = incl;
    __syncthreads();
    int32_t run = incl - own;
    for (int w = 0; w < wid; ++w) run += wsum[w];
    for (int b = b0; b < b1; ++b) {
      start[b] = run;
      run += cnt[b];
    }
  }
  __syncthreads();
  const int head = pb_head(warps);
  uint16_t* blk = lanes + off[k];
  // head: first list row of each warp, then the total
  if (tid == 0) {
    int32_t tot = 0;
    for (int w = 0; w < warps; ++w) {
      blk[w] = (uint16_t)tot;
      tot += maxlen[k * warps + w];
    }
    for (int w = warps; w < head; ++w) blk[w] = (uint16_t)tot;
  }
  const int lane = tid & 31, wid = tid >> 5;
  const uint16_t pad = (uint16_t)chunk;  // zero slot, slot 0, positive
  for (int w = wid; w < warps; w += PB_NT / 32) {
    int32_t rowbase = 0;
    for (int q = 0; q < w; ++q) rowbase += maxlen[k * warps + q];
    const int ml = maxlen[k * warps + w];
    uint16_t* R = blk + head + (int64_t)rowbase * 32;
    // lane l's four slot lists: next row (register), entries left
    int nxt[SL], cb[SL], st[SL];
    uint32_t cand[SL];
#pragma unroll
    for (int s = 0; s < SL; ++s) {
      const int b = w * 32 + lane + s * 32 * warps;
      cb[s] = b < d ? cnt[b] : 0;
      st[s] = b < d ? start[b] : 0;
      nxt[s] = 0;
      cand[s] = cb[s] > 0 ? (keys[st[s]] & 0x1fffu) : 0u;
    }
    for (int step = 0; step < ml; ++step) {
      // The lanes choose in lane order, each seeing the bank loads of the
      // lanes before it -- exactly the host planner's greedy.  Only register
      // compares sit on this serial chain: the candidates are preloaded, the
      // chosen list advances and the word (with its sign) is formed after.
      uint32_t ld4[4] = {0u, 0u, 0u, 0u};  // 16 bank counters, 8 bits each
      int mine = -1;
#pragma unroll 4
      for (int l = 0; l < 32; ++l) {
        int choice = -1;
        if (lane == l) {
          int bload = 1 << 30;
          int bleft = 0;
#pragma unroll
          for (int s = 0; s < SL; ++s) {
            if (nxt[s] >= cb[s]) continue;
            const int bank = (int)(cand[s] & 15);
            const uint32_t word4 = bank < 8 ? (bank < 4 ? ld4[0] : ld4[1])
                                            : (bank < 12 ? ld4[2] : ld4[3]);
            const int ld = (int)((word4 >> (8 * (bank & 3))) & 255u);
            const int left = cb[s] - nxt[s];
            if (ld < bload || (ld == bload && left > bleft)) {
              choice = s;
              bload = ld;
              bleft = left;
            }
          }
          mine = choice;
        }
        int cbank = -1;
#pragma unroll
        for (int s = 0; s < SL; ++s)
          if (s == choice) cbank = (int)(cand[s] & 15);
        const int bank_l = __shfl_sync(0xffffffffu, cbank, l);
        if (bank_l >= 0) {
          const uint32_t inc = 1u << (8 * (bank_l & 3));
          if (bank_l < 4)
            ld4[0] += inc;
          else if (bank_l < 8)
            ld4[1] += inc;
          else if (bank_l < 12)
            ld4[2] += inc;
          else
            ld4[3] += inc;
        }
      }
      uint16_t word = pad;
      if (mine >= 0) {
        constexpr int RB = SL == 4 ? 13 : SL == 8 ? 12 : 11;  // owned_row_bits
        uint32_t jrow = 0;
#pragma unroll
        for (int s = 0; s < SL; ++s)
          if (s == mine) jrow = cand[s];
        word = (uint16_t)(jrow | ((uint32_t)mine << RB) | ((sg[jrow] < 0 ? 1u : 0u) << 15));
#pragma unroll
        for (int s = 0; s < SL; ++s)
          if (s == mine) {
            ++nxt[s];
            cand[s] = nxt[s] < cb[s] ? (keys[st[s] + nxt[s]] & 0x1fffu) : 0u;
          }
      }
      R[(int64_t)step * 32 + lane] = word;
    }
  }
}

static int sm_count_pb() { return sm_count_cached(); }

}  // namespace skl

using namespace skl;

extern "C" int skl_rng_countsketch_device(uint64_t key, int64_t m, int64_t d, int32_t* rows,
                                          int8_t* signs, void* stream) {
  clear_error();
  cudaStream_t st = (cudaStream_t)stream;
  SKL_REQUIRE(m >= 1 && d >= 1 && d <= 0x7fffffffLL && rows && signs, SKL_ERR_INVALID,
              "rng_countsketch_device: bad arguments");
  uint64_t sign_pos = 0;
  if (d == 1) {
    SKL_CUDA(cudaMemsetAsync(rows, 0, (size_t)m * sizeof(int32_t), st));
  } else {
    const uint64_t dd = (uint64_t)d;
    const uint32_t threshold = (uint32_t)((0x100000000ULL - dd) % dd);
    unsigned long long* rej = nullptr;
    SKL_CUDA(malloc_async(&rej, sizeof(unsigned long long), st));
    SKL_CUDA(cudaMemsetAsync(rej, 0, sizeof(unsigned long long), st));
    const int64_t nblk = (m + 7) / 8;
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((nblk + 255) / 256,
                                                                 8LL * sm_count_pb()));
    cs_rows_kernel<<<grid, 256, 0, st>>>(key, m, dd, threshold, rows, rej);
    SKL_CUDA_LAUNCH();
    unsigned long long nrej = 0;
    if (threshold != 0) {
      SKL_CUDA(cudaMemcpyAsync(&nrej, rej, sizeof(nrej), cudaMemcpyDeviceToHost, st));
      SKL_CUDA(cudaStreamSynchronize(st));
    }
    cudaFreeAsync(rej, st);
    if (nrej) {
      // rare: some draw was rejected -- take the host builder's stream walk
      std::vector<int32_t> hr((size_t)m);
      std::vector<int8_t> hs((size_t)m);
      const int rc = skl_rng_countsketch(key, m, d, hr.data(), hs.data(), 0, nullptr);
      if (rc) return rc;
      SKL_CUDA(cudaMemcpyAsync(rows, hr.data(), (size_t)m * sizeof(int32_t),
                               cudaMemcpyHostToDevice, st));
      SKL_CUDA(cudaMemcpyAsync(signs, hs.data(), (size_t)m, cudaMemcpyHostToDevice, st));
      SKL_CUDA(cudaStreamSynchronize(st));
      return SKL_OK;
    }
    sign_pos = (uint64_t)m;
  }
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((m + 255) / 256,
                                                               8LL * sm_count_pb()));
  cs_signs_kernel<<<grid, 256, 0, st>>>(key, m, sign_pos, signs);
  SKL_CUDA_LAUNCH();
  return SKL_OK;
}

extern "C" int skl_countsketch_plan_owned_device(const int32_t* rows, const int8_t* signs,
                                                 int64_t m, int64_t d, int64_t chunk, int warps,
                                                 uint16_t* lanes, int64_t* chunk_off,
                                                 int32_t* maxlen, int64_t* total_and_max,
                                                 void* stream) {
  clear_error();
  cudaStream_t st = (cudaStream_t)stream;
  SKL_REQUIRE(rows && signs && chunk_off && maxlen && m >= 1 && d >= 1, SKL_ERR_INVALID,
              "plan_owned_device: bad arguments");
  const int nsl = owned_slots(d, warps);
  SKL_REQUIRE(warps >= 1 && warps <= 16 && nsl > 0, SKL_ERR_SPEC,
              "owned plan: embed_dim %lld needs more than %d warps x 32 lanes x 16 slots",
              (long long)d, warps);
  const int64_t cmax = owned_max_chunk(nsl);
  SKL_REQUIRE(chunk >= 8 && chunk <= cmax && chunk % 8 == 0, SKL_ERR_INVALID,
              "owned plan chunk must be a multiple of 8 in [8, %lld], got %lld", (long long)cmax,
              (long long)chunk);
  const int64_t nch = (m + chunk - 1) / chunk;
  if (!lanes) {
    SKL_REQUIRE(total_and_max, SKL_ERR_INVALID, "plan_owned_device: total_and_max missing");
    int64_t* sizes = nullptr;
    SKL_CUDA(malloc_async(&sizes, (size_t)(nch + 1) * sizeof(int64_t), st));
    owned_sizes_kernel<<<(unsigned)nch, PB_NT, (size_t)d * sizeof(int32_t), st>>>(
        rows, m, (int)d, (int)chunk, warps, nsl, maxlen, sizes);
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) {
      owned_scan_kernel<<<1, 32, 0, st>>>(sizes, nch, chunk_off, sizes + nch);
      e = cudaGetLastError();
    }
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(total_and_max, chunk_off + nch, sizeof(int64_t),
                          cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(total_and_max + 1, sizes + nch, sizeof(int64_t),
                          cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    cudaFreeAsync(sizes, st);
    if (e != cudaSuccess) SKL_FAIL(SKL_ERR_CUDA, "plan_owned_device sizes: %s", cudaGetErrorString(e));
    SKL_REQUIRE(total_and_max[1] <= 65535LL * 32, SKL_ERR_SPEC, "owned plan: chunk block too large");
    return SKL_OK;
  }
  const size_t smem = (size_t)PB_KEYS * 4 + (size_t)d * 8 + (size_t)chunk;
  auto fill = nsl == 4 ? owned_fill_kernel<4> : owned_fill_kernel<8>;
  SKL_CUDA(raise_smem_limit(fill, smem));
  fill<<<(unsigned)nch, PB_NT, smem, st>>>(rows, signs, m, (int)d, (int)chunk, warps, maxlen,
                                           chunk_off, lanes);
  SKL_CUDA_LAUNCH();
  return SKL_OK;
}
