// Shared helpers of the sketchls_b200 native library: status/error plumbing
// (thread-local message, see include/sketchls_b200.h) and CUDA checks.
#pragma once

#include <cstdarg>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <string>

#include "../../include/sketchls_b200.h"

namespace skl {

void set_error(const char* fmt, ...);
void clear_error();

// Tuning / A-B knobs from the environment: a flag is set only by a non-empty
// value other than "0"; an integer knob falls back to `dflt` when unset,
// empty or not positive.
inline bool env_flag(const char* name) {
  const char* v = getenv(name);
  return v && *v && !(v[0] == '0' && v[1] == 0);
}
inline long long env_int(const char* name, long long dflt) {
  const char* v = getenv(name);
  if (!v || !*v) return dflt;
  const long long x = atoll(v);
  return x > 0 ? x : dflt;
}

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
#include <map>
#include <mutex>
#include <utility>

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

// Raise (never lower) a kernel's dynamic shared-memory limit on the current
// device.  The attribute is process-global: setting it to each call's own
// size would let a concurrent caller with a smaller size lower it between
// another thread's set and launch, failing that launch.  Only ever raising
// it keeps every request that was granted valid.
inline cudaError_t raise_smem_limit(const void* func, size_t bytes) {
  static std::mutex mu;
  static std::map<std::pair<int, const void*>, size_t> granted;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lk(mu);
  size_t& cur = granted[{dev, func}];
  if (bytes <= cur) return cudaSuccess;
  e = cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e == cudaSuccess) cur = bytes;
  return e;
}
template <class K>
inline cudaError_t raise_smem_limit(K* kernel, size_t bytes) {
  return raise_smem_limit(reinterpret_cast<const void*>(kernel), bytes);
}
// Prefer the largest shared-memory carveout for a kernel, once per device
// (cudaFuncSetAttribute costs microseconds of host time per call: it sat on
// every launch of the sketch kernels).
inline cudaError_t prefer_max_shared(const void* func) {
  static std::mutex mu;
  static std::map<std::pair<int, const void*>, bool> done;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lk(mu);
  bool& d = done[{dev, func}];
  if (d) return cudaSuccess;
  e = cudaFuncSetAttribute(func, cudaFuncAttributePreferredSharedMemoryCarveout,
                           cudaSharedmemCarveoutMaxShared);
  if (e == cudaSuccess) d = true;
  return e;
}
template <class K>
inline cudaError_t prefer_max_shared(K* kernel) {
  return prefer_max_shared(reinterpret_cast<const void*>(kernel));
}

// Stream-ordered workspace allocation from a memory pool the library owns
// (one per device, created on first use), not the device's default pool:
// memory it keeps cached is the library's alone.  Up to kPoolKeepBytes stay
// mapped across stream synchronisations, so the per-call workspaces of the
// QR, split-K partials and host-streaming rings are reused without a remap;
// anything above that (a one-off multi-GiB workspace) goes back to the
// driver at the next synchronisation instead of staying mapped for the life
// of the process, out of reach of torch's allocator.
constexpr uint64_t kPoolKeepBytes = 1ULL << 30;

inline cudaMemPool_t library_pool() {
  static std::once_flag made[64];
  static cudaMemPool_t pools[64] = {};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return nullptr;
  once_per_device(made, [dev] {
    cudaMemPoolProps props = {};
    props.allocType = cudaMemAllocationTypePinned;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = dev;
    cudaMemPool_t pool = nullptr;
    if (cudaMemPoolCreate(&pool, &props) == cudaSuccess) {
      uint64_t keep = kPoolKeepBytes;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
      pools[dev] = pool;
    }
    return 0;
  });
  return pools[dev];
}

template <class T>
inline cudaError_t malloc_async(T** p, size_t bytes, cudaStream_t st) {
  cudaMemPool_t pool = library_pool();
  if (!pool) return cudaMallocAsync(reinterpret_cast<void**>(p), bytes, st);
  return cudaMallocFromPoolAsync(reinterpret_cast<void**>(p), bytes, pool, st);
}
// Launch with programmatic stream serialization (see pdl_enter in
// skl_ptx.cuh) when `pdl`: only for a kernel whose sole dependency is the
// kernel launched just before it in the same stream (never right after a
// cudaStreamWaitEvent), and that calls pdl_enter() before touching global
// memory.  SKL_NO_PDL=1 turns it off (A/B knob).
template <typename... KArgs, typename... Args>
inline cudaError_t launch_k(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                            cudaStream_t st, bool pdl, Args... args) {
  static const bool off = env_flag("SKL_NO_PDL");
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = (pdl && !off) ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kernel, args...);
}
inline bool pdl_enabled() {
  static const bool off = env_flag("SKL_NO_PDL");
  return !off;
}
}  // namespace skl
#endif
