// Microbenchmark of the CholeskyQR tile routines (csrc/skl_cholqr.cu): one
// CTA, clock64 around the first (cold instruction cache) and the following
// (warm) calls of cq_factor / cq_rowsolve / cq_tile_update.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include \
//        tools/micro/cq_factor_bench.cu -o /tmp/cqfb && /tmp/cqfb
#define CQ_FACTOR_CLOCKS
#include "../../paper_2409_14309_b200/csrc/skl_cholqr.cu"
#include <cstdio>

__global__ void __launch_bounds__(256, 1) bench(const double* G, double* Rg, int* flag, long long* out) {
  __shared__ __align__(16) double T[skl::CQ_TILE + 32];
  __shared__ __align__(16) double U[skl::CQ_TILE + 32];
  __shared__ __align__(16) double srow[128];
  const int tid = threadIdx.x;
  for (int rep = 0; rep < 4; ++rep) {
    for (int e = tid; e < 1024; e += 256) T[(e >> 5) * skl::CQ_LD + (e & 31)] = G[e];
    __syncthreads();
    long long t0 = clock64();
    if (tid < 32) skl::cq_factor(T, srow, Rg, flag);
    __syncthreads();
    long long t1 = clock64();
    for (int e = tid; e < skl::CQ_TILE + 32; e += 256) U[e] = T[e];
    for (int e = tid; e < 1024; e += 256) T[(e >> 5) * skl::CQ_LD + (e & 31)] = G[e];
    __syncthreads();
    long long t2 = clock64();
    if (tid < 32) skl::cq_rowsolve(T, U, Rg);
    __syncthreads();
    long long t3 = clock64();
    if (tid < 32) skl::cq_tile_update<2, 4>(T, U, false, 0, U, 0, 0);
    __syncthreads();
    long long t4 = clock64();
    if (tid < 32) skl::cq_diag_inverse(U, Rg, T);
    __syncthreads();
    long long t5 = clock64();
    if (tid == 0) {
      out[rep * 4 + 0] = t1 - t0;
      out[rep * 4 + 1] = t3 - t2;
      out[rep * 4 + 2] = t4 - t3;
      out[rep * 4 + 3] = t5 - t4;
    }
  }
}

int main() {
  double h[1024];
  for (int c = 0; c < 32; ++c)
    for (int r = 0; r < 32; ++r) h[c * 32 + r] = (r == c ? 40.0 : 0.0) + 1.0 / (1 + r + c);
  double *G, *R; int* f; long long* o;
  cudaMalloc(&G, 8192); cudaMalloc(&R, 8192); cudaMalloc(&f, 4); cudaMalloc(&o, 16 * 8);
  cudaMemcpy(G, h, 8192, cudaMemcpyHostToDevice);
  bench<<<1, 256>>>(G, R, f, o);
  long long ho[16];
  cudaMemcpy(ho, o, sizeof(ho), cudaMemcpyDeviceToHost);
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  long long fc[17];
  cudaMemcpyFromSymbol(fc, skl::cq_factor_clocks, sizeof(fc));
  printf("pair cycles:");
  for (int i = 1; i < 17; ++i) printf(" %lld", fc[i] - fc[i - 1]);
  printf("\n");
  for (int r = 0; r < 4; ++r)
    printf("rep %d: factor %lld  rowsolve %lld  tile_update %lld  diag_inverse %lld cycles\n", r,
           ho[r * 4], ho[r * 4 + 1], ho[r * 4 + 2], ho[r * 4 + 3]);
  return 0;
}
namespace skl {
void set_error(const char*, ...) {}
void clear_error() {}
}
