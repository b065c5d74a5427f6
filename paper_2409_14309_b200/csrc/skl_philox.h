// Philox4x64-10 and splitmix64, usable from host C++ and CUDA device code.
// This is the counter-based generator numpy 2.3.5 uses for
// Generator(Philox(key)) (sketchls/rng.py:43-45): key words (key, 0),
// counter pre-incremented so stream block q is philox(counter=(q+1,0,0,0)).
// splitmix64 mirrors sketchls/rng.py:19-24.
#pragma once
#include <cstdint>

#ifdef __CUDACC__
#define SKL_HD __host__ __device__ __forceinline__
#else
#define SKL_HD inline
#endif

namespace skl {

SKL_HD uint64_t splitmix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

SKL_HD void mulhilo64(uint64_t a, uint64_t b, uint64_t& hi, uint64_t& lo) {
#ifdef __CUDA_ARCH__
  lo = a * b;
  hi = __umul64hi(a, b);
#else
  unsigned __int128 p = (unsigned __int128)a * b;
  lo = (uint64_t)p;
  hi = (uint64_t)(p >> 64);
#endif
}

// Stream block q (0-based): four u64 words.
SKL_HD void philox_block(uint64_t key, uint64_t q, uint64_t out[4]) {
  uint64_t c0 = q + 1, c1 = (q + 1 == 0) ? 1 : 0, c2 = 0, c3 = 0;
  uint64_t k0 = key, k1 = 0;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r) {
      k0 += 0x9E3779B97F4A7C15ULL;
      k1 += 0xBB67AE8584CAA73BULL;
    }
    uint64_t hi0, lo0, hi1, lo1;
    mulhilo64(0xD2E7470EE14C6C93ULL, c0, hi0, lo0);
    mulhilo64(0xCA5A826395121157ULL, c2, hi1, lo1);
    uint64_t n0 = hi1 ^ c1 ^ k0, n1 = lo1, n2 = hi0 ^ c3 ^ k1, n3 = lo0;
    c0 = n0; c1 = n1; c2 = n2; c3 = n3;
  }
  out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

}  // namespace skl
