// Where the cycles of cq_factor's pivot step go: the full step, the pivot
// chain alone (no rank-1 update), and the update alone (pivot not carried).
#include <cstdio>
#define LDT 33
template <int MODE>  // 0 full, 1 chain only, 2 update only
__device__ __noinline__ void factor(double* T, double* srow, double* out) {
  const int lane = threadIdx.x & 31;
  double c[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) c[i] = T[lane * LDT + i];
  srow[32 + lane] = 0.0;
  double pk = __shfl_sync(0xffffffffu, c[0], 0), rk = 1.0 / pk, myd = 0;
#pragma unroll 1
  for (int k = 0; k < 32; ++k) {
    const double gk = c[0];
    double pn = fma(-(gk * gk), rk, c[1]);
    double pnext = MODE == 2 ? pk : __shfl_sync(0xffffffffu, pn, (k + 1) & 31);
    double rn;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(rn) : "d"(pnext));
    const double u = gk * rk;
    if (MODE != 1) {
      if (lane > k) T[lane * LDT + k] = u;
      srow[lane] = lane > k ? gk : 0.0;
      __syncwarp();
      const double* sr = srow + k + 1;
#pragma unroll
      for (int i = 0; i < 31; ++i) c[i] = fma(-sr[i], u, c[i + 1]);
      __syncwarp();
    } else {
      c[0] = c[1]; c[1] = fma(-gk, u, c[1]);
    }
    rn = fma(rn, fma(-pnext, rn, 1.0), rn);
    rn = fma(rn, fma(-pnext, rn, 1.0), rn);
    if (lane == k) myd = pk;
    pk = pnext;
    rk = rn;
  }
  out[lane] = myd + c[0];
}
__global__ void bench(const double* G, double* out, long long* cyc) {
  __shared__ double T[32 * LDT];
  __shared__ __align__(16) double srow[64];
  for (int rep = 0; rep < 3; ++rep) {
    for (int v = 0; v < 3; ++v) {
      for (int e = threadIdx.x; e < 1024; e += 32) T[(e >> 5) * LDT + (e & 31)] = G[e];
      __syncwarp();
      long long t0 = clock64();
      if (v == 0) factor<0>(T, srow, out);
      if (v == 1) factor<1>(T, srow, out);
      if (v == 2) factor<2>(T, srow, out);
      __syncwarp();
      long long t1 = clock64();
      if (threadIdx.x == 0 && rep == 2) cyc[v] = t1 - t0;
    }
  }
}
int main() {
  double h[1024];
  for (int c = 0; c < 32; ++c) for (int r = 0; r < 32; ++r) h[c * 32 + r] = (r == c ? 40.0 : 0.0) + 1.0 / (1 + r + c);
  double *G, *o; long long* cy;
  cudaMalloc(&G, 8192); cudaMalloc(&o, 8192); cudaMalloc(&cy, 64);
  cudaMemcpy(G, h, 8192, cudaMemcpyHostToDevice);
  bench<<<1, 32>>>(G, o, cy);
  long long c[3]; cudaMemcpy(c, cy, 24, cudaMemcpyDeviceToHost);
  printf("full %lld  chain-only %lld  update-only %lld cycles (32 steps)\n", c[0], c[1], c[2]);
}
