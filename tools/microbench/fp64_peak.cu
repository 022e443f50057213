// FP64 throughput microbenchmark for sm_100a: DFMA register chains vs mma.sync f64 (DMMA).
// Decides the core of the update kernels (SURVEY §7 phase 3). Not part of the product path.
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

template <int NACC>
__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double acc[NACC];
#pragma unroll
  for (int i = 0; i < NACC; ++i) acc[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) acc[i] = fma(acc[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += acc[i];
  if (s == 123.456) out[threadIdx.x] = s;
}

template <int NACC>
__global__ void dmma884_kernel(double* out, int iters) {
  double c[NACC][2];
  double a = 1.0 + threadIdx.x * 1e-6, b = 0.999;
#pragma unroll
  for (int i = 0; i < NACC; ++i) { c[i][0] = 0; c[i][1] = i; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += c[i][0] + c[i][1];
  if (s == 123.456) out[threadIdx.x] = s;
}

template <int NACC>
__global__ void dmma16816_kernel(double* out, int iters) {
  double c[NACC][4];
  double a[8], b[4];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = 1.0 + threadIdx.x * 1e-6 + i;
#pragma unroll
  for (int i = 0; i < 4; ++i) b[i] = 0.999 - i * 1e-3;
#pragma unroll
  for (int i = 0; i < NACC; ++i) { c[i][0] = 0; c[i][1] = i; c[i][2] = 0; c[i][3] = 1; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                     "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  if (s == 123.456) out[threadIdx.x] = s;
}

int main() {
  int dev = 0; cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, dev));
  int clk_khz = 0; cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev);
  printf("device %s SMs %d clock(attr) %d MHz\n", p.name, p.multiProcessorCount, clk_khz / 1000);
  double* out; CK(cudaMalloc(&out, 1 << 20));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int sms = p.multiProcessorCount;
  for (int rep = 0; rep < 2; ++rep) {
    for (int tpb : {256, 512, 1024}) {
      int blocks = sms * (2048 / tpb);
      int iters = 20000;
      dfma_kernel<8><<<blocks, tpb>>>(out, 100, 1.0000001, 1e-9);
      cudaEventRecord(e0);
      dfma_kernel<8><<<blocks, tpb>>>(out, iters, 1.0000001, 1e-9);
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double flops = 2.0 * 8 * iters * (double)blocks * tpb;
      printf("DFMA  tpb=%4d blocks=%d: %.2f TFLOP/s (%.3f ms)\n", tpb, blocks, flops / ms / 1e9, ms);
    }
    for (int tpb : {128, 256, 512}) {
      int blocks = sms * (2048 / tpb);
      int iters = 20000;
      dmma884_kernel<8><<<blocks, tpb>>>(out, 100);
      cudaEventRecord(e0);
      dmma884_kernel<8><<<blocks, tpb>>>(out, iters);
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double flops = 2.0 * 256 * 8 * iters * (double)blocks * (tpb / 32);
      printf("DMMA884 tpb=%4d blocks=%d: %.2f TFLOP/s (%.3f ms)\n", tpb, blocks, flops / ms / 1e9, ms);
    }
    for (int tpb : {128, 256}) {
      int blocks = sms * (1024 / tpb);
      int iters = 4000;
      dmma16816_kernel<4><<<blocks, tpb>>>(out, 100);
      cudaEventRecord(e0);
      dmma16816_kernel<4><<<blocks, tpb>>>(out, iters);
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double flops = 2.0 * 16 * 8 * 16 * 4 * iters * (double)blocks * (tpb / 32);
      printf("DMMA16816 tpb=%4d blocks=%d: %.2f TFLOP/s (%.3f ms)\n", tpb, blocks, flops / ms / 1e9, ms);
    }
  }
  // sustained DFMA for ~3 s to see clocks under FP64 load
  {
    int tpb = 512, blocks = sms * 4, iters = 400000;
    cudaEventRecord(e0);
    for (int r = 0; r < 10; ++r) dfma_kernel<8><<<blocks, tpb>>>(out, iters, 1.0000001, 1e-9);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 10 * 2.0 * 8 * (double)iters * blocks * tpb;
    printf("DFMA sustained: %.2f TFLOP/s over %.1f ms\n", flops / ms / 1e9, ms);
  }
  {
    int tpb = 256, blocks = sms * 8, iters = 200000;
    cudaEventRecord(e0);
    for (int r = 0; r < 10; ++r) dmma884_kernel<8><<<blocks, tpb>>>(out, iters);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 10 * 2.0 * 256 * 8 * (double)iters * blocks * (tpb / 32);
    printf("DMMA884 sustained: %.2f TFLOP/s over %.1f ms\n", flops / ms / 1e9, ms);
  }
  return 0;
}
