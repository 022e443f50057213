// Does alternating dynamic-smem sizes between consecutive kernels cost time on B200?
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_small(int* p) { extern __shared__ double s[]; if (threadIdx.x == 0 && p[0] == 12345) s[0] = 1, p[1] = (int)s[0]; }
__global__ void k_big(int* p) { extern __shared__ double s[]; if (threadIdx.x == 0 && p[0] == 12345) s[0] = 1, p[1] = (int)s[0]; }
int main() {
  int* d; cudaMalloc(&d, 64); cudaMemset(d, 0, 64);
  cudaFuncSetAttribute(k_big, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(k_small, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  auto run = [&](const char* name, int s1, int s2, int grid) {
    for (int w = 0; w < 2; ++w) {
      cudaEventRecord(a);
      for (int i = 0; i < 500; ++i) { k_small<<<grid, 128, s1>>>(d); k_big<<<grid, 128, s2>>>(d); }
      cudaEventRecord(b); cudaEventSynchronize(b);
    }
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("%-40s grid %4d: %.2f us per launch\n", name, grid, ms * 1000 / 1000);
  };
  for (int grid : {1, 148, 1184}) {
    run("same smem 0/0", 0, 0, grid);
    run("same smem 32K/32K", 32 << 10, 32 << 10, grid);
    run("alternating 32K/132K", 32 << 10, 132 << 10, grid);
    run("alternating 0/132K", 0, 132 << 10, grid);
    run("same 132K/132K", 132 << 10, 132 << 10, grid);
  }
  // with carveout forced to max shared for both
  cudaFuncSetAttribute(k_big, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  cudaFuncSetAttribute(k_small, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  for (int grid : {1, 148}) {
    run("carveout100: alternating 32K/132K", 32 << 10, 132 << 10, grid);
    run("carveout100: alternating 0/132K", 0, 132 << 10, grid);
  }
  // graph version
  cudaStream_t s; cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  cudaGraph_t g; cudaGraphExec_t ge;
  cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
  for (int i = 0; i < 500; ++i) { k_small<<<148, 128, 32 << 10, s>>>(d); k_big<<<148, 128, 132 << 10, s>>>(d); }
  cudaStreamEndCapture(s, &g); cudaGraphInstantiate(&ge, g, 0);
  for (int w = 0; w < 2; ++w) { cudaEventRecord(a, s); cudaGraphLaunch(ge, s); cudaEventRecord(b, s); cudaEventSynchronize(b); }
  float ms; cudaEventElapsedTime(&ms, a, b);
  printf("graph alternating 32K/132K carveout100 grid 148: %.2f us per node\n", ms * 1000 / 1000);
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
