// Fixed-order sum of per-rank partial sketches (the reduce step of the
// row-sharded apply).
//
// Each rank's sketch kernel writes its d x (n+1) partial straight into its
// own slot of the destination rank's symmetric buffer (NVLink peer stores
// from the kernel's epilogue, so the transfer overlaps the other CTAs'
// work); after a device-side barrier the destination sums the slots in rank
// order.  The result is deterministic for a given world size -- unlike a
// reduction whose order follows the collective library's algorithm choice.
#include <cuda_runtime.h>

#include <algorithm>

#include "skl_common.h"

namespace skl {

__global__ void sum_slots_kernel(const double* __restrict__ slots, int64_t nslots,
                                 int64_t slot_stride, int64_t rows, int64_t cols, int64_t ld,
                                 double* __restrict__ out, int64_t ldo) {
  const int64_t total = rows * cols;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = idx / rows, i = idx % rows;
    const double* p = slots + c * ld + i;
    double s = p[0];
    for (int64_t q = 1; q < nslots; ++q) s += p[q * slot_stride];
    out[c * ldo + i] = s;
  }
}

}  // namespace skl

using namespace skl;

extern "C" int skl_sum_slots(const double* slots, int64_t nslots, int64_t slot_stride,
                             int64_t rows, int64_t cols, int64_t ld, double* out, int64_t ldo,
                             void* stream) {
  clear_error();
  SKL_REQUIRE(slots && out && nslots >= 1 && rows >= 1 && cols >= 1 && ld >= rows &&
                  ldo >= rows && slot_stride >= ld * cols,
              SKL_ERR_SHAPE, "sum_slots: bad arguments");
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t total = rows * cols;
  const int blocks = (int)std::min<int64_t>((total + 255) / 256, 8LL * sms);
  sum_slots_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(slots, nslots, slot_stride, rows,
                                                              cols, ld, out, ldo);
  SKL_CUDA_LAUNCH();
  return SKL_OK;
}
