// cq_factor alone vs cq_factor with cq_lockstep_solve running beside it in a
// second warp (clock64, one CTA; csrc/skl_cholqr.cu).
#include "../../paper_2409_14309_b200/csrc/skl_cholqr.cu"
#include <cstdio>
namespace skl {
void set_error(const char*, ...) {}
void clear_error() {}
}
__global__ void __launch_bounds__(256, 1) bench(const double* G, double* Rg, int* flag, long long* out) {
  __shared__ __align__(16) double T[2 * skl::CQ_TILE + 64];
  __shared__ __align__(16) double Gn[skl::CQ_TILE];
  __shared__ __align__(16) double srow[128];
  __shared__ __align__(16) double up[1100];
  __shared__ int prog;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int mode = 0; mode < 2; ++mode) {
    for (int rep = 0; rep < 3; ++rep) {
      for (int e = tid; e < 1024; e += 256) {
        T[(e >> 5) * skl::CQ_LD + (e & 31)] = G[e];
        Gn[(e >> 5) * skl::CQ_LD + (e & 31)] = G[e] * 0.5;
      }
      if (tid == 0) prog = 0;
      __syncthreads();
      long long t0 = clock64();
      if (warp == 0) skl::cq_factor(T, srow, Rg, flag, &prog, up);
      else if (warp == 1 && mode == 1) skl::cq_lockstep_solve(Gn, T, up, &prog, Rg + 1024);
      long long t1 = clock64();
      __syncthreads();
      long long t2 = clock64();
      if ((tid & 31) == 0 && warp < 2 && rep == 2) out[mode * 4 + warp] = t1 - t0;
      if (tid == 0 && rep == 2) out[mode * 4 + 2] = t2 - t0;
    }
  }
}
int main() {
  double h[1024];
  for (int c = 0; c < 32; ++c) for (int r = 0; r < 32; ++r) h[c * 32 + r] = (r == c ? 40.0 : 0.0) + 1.0 / (1 + r + c);
  double *G, *R; int* f; long long* o;
  cudaMalloc(&G, 8192); cudaMalloc(&R, 16384); cudaMalloc(&f, 4); cudaMalloc(&o, 64);
  cudaMemcpy(G, h, 8192, cudaMemcpyHostToDevice);
  bench<<<1, 256>>>(G, R, f, o);
  long long ho[8]; cudaMemcpy(ho, o, 64, cudaMemcpyDeviceToHost);
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  printf("factor alone: warp0 %lld cycles (block %lld)\n", ho[0], ho[2]);
  printf("with lockstep: factor %lld  lockstep %lld  (block %lld)\n", ho[4], ho[5], ho[6]);
}
