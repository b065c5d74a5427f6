// Fixed-order sums of per-rank partial sketches (the reduce step of the
// row-sharded apply).
//
// skl_reduce_peers (the multi-GPU data plane): every rank's sketch kernel
// writes its d x (n+1) partial into its own symmetric buffer; after a
// device-side barrier rank r sums element block r of the N partials --
// loading the peers' blocks over NVLink, adding in rank order -- and stores
// the block straight into the destination's result buffer.  A reduce-
// scatter whose gather is the destination's inbox: every rank moves
// ~(N-1)/N of one partial in and 1/N out, instead of the destination
// pulling N full partials.  skl_sum_slots: the same fixed-order sum over
// slots of one buffer.  Both are deterministic for a given world size --
// unlike a reduction whose order follows the collective library's algorithm
// choice -- and give the same bits.
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

constexpr int MAX_PEERS = 16;
struct PeerPtrs {
  const double* p[MAX_PEERS];
};

// out[i] = in.p[0][i] + in.p[1][i] + ... (rank order) for i in [begin, end);
// 16-byte loads/stores where the block is aligned (grid-stride over pairs).
__global__ void reduce_peers_kernel(PeerPtrs in, int npeers, int64_t begin, int64_t end,
                                    double* __restrict__ out, int vec) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (vec) {
    const int64_t pairs = (end - begin) / 2;
    for (int64_t k = t; k < pairs; k += stride) {
      const int64_t i = begin + 2 * k;
      double2 s = __ldcv(reinterpret_cast<const double2*>(in.p[0] + i));
      for (int q = 1; q < npeers; ++q) {
        const double2 v = __ldcv(reinterpret_cast<const double2*>(in.p[q] + i));
        s.x = __dadd_rn(s.x, v.x);
        s.y = __dadd_rn(s.y, v.y);
      }
      *reinterpret_cast<double2*>(out + i) = s;
    }
    if (t == 0 && ((end - begin) & 1)) {
      const int64_t i = end - 1;
      double s = __ldcv(in.p[0] + i);
      for (int q = 1; q < npeers; ++q) s = __dadd_rn(s, __ldcv(in.p[q] + i));
      out[i] = s;
    }
    return;
  }
  for (int64_t i = begin + t; i < end; i += stride) {
    double s = __ldcv(in.p[0] + i);
    for (int q = 1; q < npeers; ++q) s = __dadd_rn(s, __ldcv(in.p[q] + i));
    out[i] = s;
  }
}

}  // namespace skl

using namespace skl;

extern "C" int skl_reduce_peers(const double* const* peers, int npeers, int64_t begin,
                                int64_t end, double* out, void* stream) {
  clear_error();
  SKL_REQUIRE(peers && out && npeers >= 1 && npeers <= MAX_PEERS && begin >= 0 && end >= begin,
              SKL_ERR_SHAPE, "reduce_peers: bad arguments (npeers=%d, [%lld, %lld))", npeers,
              (long long)begin, (long long)end);
  if (end == begin) return SKL_OK;
  PeerPtrs in{};
  bool aligned = (begin % 2) == 0 && ((uintptr_t)out & 15) == 0;
  for (int q = 0; q < npeers; ++q) {
    SKL_REQUIRE(peers[q], SKL_ERR_INVALID, "reduce_peers: null peer %d", q);
    in.p[q] = peers[q];
    aligned = aligned && ((uintptr_t)peers[q] & 15) == 0;
  }
  const int64_t work = aligned ? (end - begin + 1) / 2 : end - begin;
  const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>((work + 255) / 256,
                                                                 4LL * sm_count_cached()));
  reduce_peers_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(in, npeers, begin, end, out,
                                                                aligned ? 1 : 0);
  SKL_CUDA_LAUNCH();
  return SKL_OK;
}

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
