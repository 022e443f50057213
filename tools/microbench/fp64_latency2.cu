// Unrolled dependent chains: per-op latency without loop overhead.
#include <cstdio>
#include <cuda_runtime.h>
template <int N> __device__ __forceinline__ double chain_fma(double x, double a, double b) {
#pragma unroll
  for (int i = 0; i < N; ++i) x = fma(x, a, b);
  return x;
}
__global__ void lat(double* out, long long* cyc, double a, double b, float fa) {
  double x = a + threadIdx.x * 1e-9;
  long long t0, t1;
  t0 = clock64(); x = chain_fma<256>(x, b, a); t1 = clock64(); cyc[0] = t1 - t0;
  t0 = clock64();
#pragma unroll
  for (int i = 0; i < 256; ++i) x = x * b;
  t1 = clock64(); cyc[1] = t1 - t0;
  t0 = clock64();
#pragma unroll
  for (int i = 0; i < 64; ++i) x = __shfl_sync(0xffffffff, x, (threadIdx.x + 1) & 31);
  t1 = clock64(); cyc[2] = t1 - t0;
  t0 = clock64();
#pragma unroll
  for (int i = 0; i < 64; ++i) x = rsqrt(x);
  t1 = clock64(); cyc[3] = t1 - t0;
  t0 = clock64();
#pragma unroll
  for (int i = 0; i < 64; ++i) x = sqrt(x);
  t1 = clock64(); cyc[4] = t1 - t0;
  float y = fa;
  t0 = clock64();
#pragma unroll
  for (int i = 0; i < 256; ++i) y = fmaf(y, 1.0001f, 0.5f);
  t1 = clock64(); cyc[5] = t1 - t0;
  t0 = clock64();
#pragma unroll
  for (int i = 0; i < 64; ++i) { double r; asm volatile("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x)); x = r; }
  t1 = clock64(); cyc[6] = t1 - t0;
  t0 = clock64();
#pragma unroll
  for (int i = 0; i < 64; ++i) x = 1.0 / x;
  t1 = clock64(); cyc[7] = t1 - t0;
  // DMMA dependent chain
  double d0 = x, d1 = 0;
  t0 = clock64();
#pragma unroll
  for (int i = 0; i < 64; ++i) asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n" : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
  t1 = clock64(); cyc[8] = t1 - t0;
  out[threadIdx.x] = x + y + d0 + d1;
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 4096); cudaMalloc(&c, 4096);
  for (int r = 0; r < 2; ++r) lat<<<1, 32>>>(o, c, 1.0, 0.999999, 1.0f);
  long long h[16]; cudaMemcpy(h, c, sizeof(h), cudaMemcpyDeviceToHost);
  printf("DFMA %.1f DMUL %.1f SHFL.f64 %.1f rsqrt %.1f sqrt %.1f FFMA %.1f rsqrt.approx %.1f 1/x %.1f DMMA %.1f (cycles per dependent op)\n",
         h[0] / 256.0, h[1] / 256.0, h[2] / 64.0, h[3] / 64.0, h[4] / 64.0, h[5] / 256.0, h[6] / 64.0, h[7] / 64.0, h[8] / 64.0);
  return 0;
}
