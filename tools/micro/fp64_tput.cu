// Single-warp fp64 issue throughput on the B200: independent DFMA streams,
// DMMA m16n8k4 streams, and LDS.64 broadcast loads (cycles per instruction).
#include <cstdio>
__global__ void k(double* out, long long* cyc, int iters) {
  __shared__ double s[64];
  if (threadIdx.x < 64) s[threadIdx.x] = threadIdx.x;
  __syncwarp();
  double a[8];
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x + i;
  const double m = 1.0000001, c = 1e-9;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = fma(a[i], m, c);
  }
  long long t1 = clock64();
  double acc[4] = {0, 0, 0, 0}, acc2[4] = {0, 0, 0, 0}, acc3[4] = {0, 0, 0, 0}, acc4[4] = {0, 0, 0, 0};
  for (int it = 0; it < iters; ++it) {
    asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                 : "+d"(acc[0]), "+d"(acc[1]), "+d"(acc[2]), "+d"(acc[3]) : "d"(a[0]), "d"(a[1]), "d"(a[2]));
    asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                 : "+d"(acc2[0]), "+d"(acc2[1]), "+d"(acc2[2]), "+d"(acc2[3]) : "d"(a[3]), "d"(a[1]), "d"(a[2]));
    asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                 : "+d"(acc3[0]), "+d"(acc3[1]), "+d"(acc3[2]), "+d"(acc3[3]) : "d"(a[4]), "d"(a[1]), "d"(a[2]));
    asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                 : "+d"(acc4[0]), "+d"(acc4[1]), "+d"(acc4[2]), "+d"(acc4[3]) : "d"(a[5]), "d"(a[1]), "d"(a[2]));
  }
  long long t2 = clock64();
  double l = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) l += s[(it + i) & 63];
  }
  long long t3 = clock64();
  double r = l;
  for (int i = 0; i < 8; ++i) r += a[i];
  for (int i = 0; i < 4; ++i) r += acc[i] + acc2[i] + acc3[i] + acc4[i];
  out[threadIdx.x] = r;
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; }
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 1024 * 8); cudaMalloc(&c, 64);
  for (int w : {32, 128}) {
    k<<<1, w>>>(o, c, 1000);
    long long h[3]; cudaMemcpy(h, c, 24, cudaMemcpyDeviceToHost);
    printf("threads %d: DFMA %.2f cyc/instr (8 streams), DMMA %.2f cyc/instr (4 streams), LDS+DADD %.2f cyc/elem\n", w,
           h[0] / 8000.0, h[1] / 4000.0, h[2] / 8000.0);
  }
  return 0;
}
