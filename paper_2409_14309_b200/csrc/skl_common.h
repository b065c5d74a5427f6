// Shared helpers of the sketchls_b200 native library: status/error plumbing
// (thread-local message, see include/sketchls_b200.h) and CUDA checks.
#pragma once

#include <cstdarg>
#include <cstdint>
#include <cstdio>
#include <string>

#include "../../include/sketchls_b200.h"

namespace skl {

void set_error(const char* fmt, ...);
void clear_error();

// Number of host worker threads for `threads` <= 0 requests.
int resolve_threads(int threads);

// Register-owned CountSketch plan geometry (skl_countsketch_plan_owned):
// every consumer thread owns `slots` buckets (4 or 8: d <= 32 x warps x
// slots), and the u16 entry word is row | slot << row_bits | negative << 15,
// so the chunk (row field incl. the zero slot at index `chunk`) shrinks as
// the slot field grows: 8184 or 4088 rows.  0: d too large.  (16 slots fit
// the format too -- 2040-row chunks -- but were measured slower than the
// lane-list kernel: short lane lists pad heavily and 16 predicated adds per
// entry cost more issue slots than the shared-memory sums.)
inline int owned_slots(int64_t d, int warps) {
  const int64_t per = (d + 32 * (int64_t)warps - 1) / (32 * (int64_t)warps);
  return per <= 4 ? 4 : per <= 8 ? 8 : 0;
}
inline int owned_row_bits(int slots) { return slots == 4 ? 13 : slots == 8 ? 12 : 11; }
inline int64_t owned_max_chunk(int slots) { return (1LL << owned_row_bits(slots)) - 8; }

}  // namespace skl

#define SKL_FAIL(code, ...)          \
  do {                               \
    skl::set_error(__VA_ARGS__);     \
    return (code);                   \
  } while (0)

#define SKL_REQUIRE(cond, code, ...) \
  do {                               \
    if (!(cond)) SKL_FAIL(code, __VA_ARGS__); \
  } while (0)

#ifdef __CUDACC__
#include <cuda_runtime.h>
#define SKL_CUDA(call)                                                          \
  do {                                                                          \
    cudaError_t e__ = (call);                                                   \
    if (e__ != cudaSuccess)                                                     \
      SKL_FAIL(SKL_ERR_CUDA, "%s failed: %s (%s:%d)", #call, cudaGetErrorString(e__), \
               __FILE__, __LINE__);                                             \
  } while (0)
#define SKL_CUDA_LAUNCH()                                                       \
  do {                                                                          \
    cudaError_t e__ = cudaGetLastError();                                       \
    if (e__ != cudaSuccess)                                                     \
      SKL_FAIL(SKL_ERR_CUDA, "kernel launch failed: %s (%s:%d)",               \
               cudaGetErrorString(e__), __FILE__, __LINE__);                    \
  } while (0)

#include <atomic>
#include <mutex>

namespace skl {
// SM count of the current device, cached per device (thread-safe).
inline int sm_count_cached() {
  static std::atomic<int> cache[64];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 148;
  int v = cache[dev].load(std::memory_order_relaxed);
  if (v == 0) {
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    if (v <= 0) v = 148;
    cache[dev].store(v, std::memory_order_relaxed);
  }
  return v;
}

// Runs `f` once per device (thread-safe: concurrent first callers wait for
// it to finish), for one-time setup such as kernel attributes.  Returns the
// status of the run (later calls return SKL_OK).
template <class F>
inline int once_per_device(std::once_flag* flags /* [64] */, F&& f) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return f();
  int rc = 0;
  std::call_once(flags[dev], [&] { rc = f(); });
  return rc;
}

// Stream-ordered workspace allocation.  The first call on a device raises
// the default memory pool's release threshold so freed workspaces stay
// mapped across stream synchronisations (the default threshold of 0 unmaps
// them at every sync and the next call pays the remap, milliseconds for the
// QR's workspaces).
template <class T>
inline cudaError_t malloc_async(T** p, size_t bytes, cudaStream_t st) {
  static std::once_flag retained[64];
  once_per_device(retained, [] {
    int dev = 0;
    cudaMemPool_t pool;
    if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t keep = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
    return 0;
  });
  return cudaMallocAsync(reinterpret_cast<void**>(p), bytes, st);
}
}  // namespace skl
#endif
