// Dependent-chain latencies (cycles) of FP64 ops and shuffles on one warp of sm_100a.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void lat(double* out, long long* cyc, double a, double b) {
  double x = a + threadIdx.x * 1e-9;
  long long t0, t1;
  // DFMA chain
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 1024; ++i) x = fma(x, b, a);
  t1 = clock64(); cyc[0] = t1 - t0;
  // DMUL chain
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 1024; ++i) x = x * b;
  t1 = clock64(); cyc[1] = t1 - t0;
  // sqrt chain
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 256; ++i) x = sqrt(x) + 1.0;
  t1 = clock64(); cyc[2] = t1 - t0;
  // div chain
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 256; ++i) x = 1.0 / x + 0.5;
  t1 = clock64(); cyc[3] = t1 - t0;
  // shfl chain (double)
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 1024; ++i) x = __shfl_sync(0xffffffff, x, (threadIdx.x + 1) & 31);
  t1 = clock64(); cyc[4] = t1 - t0;
  // rsqrt chain
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 256; ++i) x = rsqrt(x) + 1.0;
  t1 = clock64(); cyc[5] = t1 - t0;
  // fp32 FFMA chain for reference
  float y = (float)x;
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 1024; ++i) y = fmaf(y, 1.0001f, 0.5f);
  t1 = clock64(); cyc[6] = t1 - t0;
  // LDS chain
  __shared__ double s[64];
  s[threadIdx.x] = (double)(threadIdx.x ^ 1);
  __syncwarp();
  int idx = threadIdx.x;
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 1024; ++i) idx = (int)s[idx & 31];
  t1 = clock64(); cyc[7] = t1 - t0;
  // __syncthreads cost (1 warp)
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 1024; ++i) __syncthreads();
  t1 = clock64(); cyc[8] = t1 - t0;
  out[threadIdx.x] = x + y + idx;
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 4096); cudaMalloc(&c, 4096);
  lat<<<1, 32>>>(o, c, 1.0, 0.999999);
  lat<<<1, 32>>>(o, c, 1.0, 0.999999);
  long long h[16]; cudaMemcpy(h, c, sizeof(h), cudaMemcpyDeviceToHost);
  printf("DFMA  %.1f cyc\nDMUL  %.1f cyc\nsqrt+add %.1f cyc\n1/x+add %.1f cyc\nSHFL(double) %.1f cyc\nrsqrt+add %.1f cyc\nFFMA %.1f cyc\nLDS(dep) %.1f cyc\nBAR(1 warp) %.1f cyc\n",
         h[0] / 1024.0, h[1] / 1024.0, h[2] / 256.0, h[3] / 256.0, h[4] / 1024.0, h[5] / 256.0, h[6] / 1024.0, h[7] / 1024.0, h[8] / 1024.0);
  return 0;
}
