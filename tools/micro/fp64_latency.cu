// Microbenchmark: dependent-chain latency (SM cycles) of FP64 and FP32 ops,
// shared-memory loads and shuffles on one warp (tools/micro, not product code).
#include <cstdio>
#include <cuda_runtime.h>

__global__ void lat(double* out, long long* cyc, double a, double b, int n) {
  __shared__ double sm[64];
  sm[threadIdx.x] = a + threadIdx.x;
  __syncwarp();
  double x = a;
  float xf = (float)a;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = fma(x, b, a);
  long long t1 = clock64();
  for (int i = 0; i < n; ++i) x = x + b;
  long long t2 = clock64();
  for (int i = 0; i < n; ++i) xf = fmaf(xf, (float)b, (float)a);
  long long t3 = clock64();
  int idx = threadIdx.x;
  for (int i = 0; i < n; ++i) { double v = sm[idx & 63]; idx = (int)v & 31; }
  long long t4 = clock64();
  for (int i = 0; i < n; ++i) x = __shfl_sync(0xffffffffu, x, (i + 1) & 31);
  long long t5 = clock64();
  for (int i = 0; i < n; ++i) x = sqrt(x + 2.0);
  long long t6 = clock64();
  for (int i = 0; i < n; ++i) x = 1.0 / (x + 3.0);
  long long t7 = clock64();
  // DMMA m16n8k4 f64: dependent chain on the accumulator
  double c[4] = {x, x, x, x};
  for (int i = 0; i < n; ++i)
    asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                 : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3]) : "d"(a), "d"(b), "d"(a));
  long long t8 = clock64();
  // rsqrt.approx.f64 and rcp.approx.ftz.f64 chains
  for (int i = 0; i < n; ++i) { double y; asm("rsqrt.approx.f64 %0, %1;" : "=d"(y) : "d"(x + 2.0)); x = y; }
  long long t9 = clock64();
  for (int i = 0; i < n; ++i) { double y; asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x + 3.0)); x = y; }
  long long t10 = clock64();
  out[threadIdx.x] = x + xf + idx + c[0] + c[1] + c[2] + c[3];
  if (threadIdx.x == 0) {
    cyc[0] = (t1 - t0) / n; cyc[1] = (t2 - t1) / n; cyc[2] = (t3 - t2) / n;
    cyc[3] = (t4 - t3) / n; cyc[4] = (t5 - t4) / n; cyc[5] = (t6 - t5) / n; cyc[6] = (t7 - t6) / n;
    cyc[7] = (t8 - t7) / n; cyc[8] = (t9 - t8) / n; cyc[9] = (t10 - t9) / n;
  }
}

int main() {
  double* o; long long* c;
  cudaMalloc(&o, 64 * 8); cudaMallocManaged(&c, 16 * 8);
  lat<<<1, 32>>>(o, c, 1.0000001, 0.9999999, 1000);
  lat<<<1, 32>>>(o, c, 1.0000001, 0.9999999, 1000);
  cudaDeviceSynchronize();
  printf("cycles per dependent op: dfma %lld dadd %lld ffma %lld lds %lld shfl(f64) %lld dsqrt %lld ddiv %lld "
         "dmma16x8x4 %lld rsqrt.approx.f64 %lld rcp.approx.f64 %lld\n",
         c[0], c[1], c[2], c[3], c[4], c[5], c[6], c[7], c[8], c[9]);
  return 0;
}
