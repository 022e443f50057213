// Times the batched potf2 per size class: full kernel, memory phases only
// (BATCH_MODE 1) and factorization only (BATCH_MODE 2).
#include <cstdio>
#include <vector>
#include <cmath>
#ifndef RELAPACK_BATCH_MODE
#define RELAPACK_BATCH_MODE 0
#endif
#include "../../paper_1602_06763_b200/csrc/batched.cu"
using namespace relapack;
int main() {
  const int count = 32768;
  for (int n : {16, 32, 48, 64}) {
    std::vector<double> h((size_t)count * n * n);
    for (int b = 0; b < count; ++b)
      for (int j = 0; j < n; ++j) for (int i = 0; i < n; ++i)
        h[(size_t)b * n * n + i + j * n] = (i == j) ? n : 1.0 / (1 + i + j);
    double* d; cudaMalloc(&d, h.size() * 8);
    double* d0; cudaMalloc(&d0, h.size() * 8);
    cudaMemcpy(d0, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
    std::vector<double*> ptrs(count); std::vector<int> ns(count, n);
    for (int b = 0; b < count; ++b) ptrs[b] = d + (size_t)b * n * n;
    double** dp; int* dn; int* dinfo;
    cudaMalloc(&dp, count * 8); cudaMalloc(&dn, count * 4); cudaMalloc(&dinfo, count * 4);
    cudaMemcpy(dp, ptrs.data(), count * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(dn, ns.data(), count * 4, cudaMemcpyHostToDevice);
    cudaEvent_t a, e; cudaEventCreate(&a); cudaEventCreate(&e);
    float best = 1e9;
    for (int r = 0; r < 6; ++r) {
      cudaMemcpy(d, d0, h.size() * 8, cudaMemcpyDeviceToDevice);
      cudaDeviceSynchronize();
      cudaEventRecord(a);
      launch_potf2_batched(kLayoutN, count, dn, dp, dn, dinfo, 0);
      cudaEventRecord(e); cudaEventSynchronize(e);
      float ms; cudaEventElapsedTime(&ms, a, e); if (r > 0 && ms < best) best = ms;
    }
    double tri = 8.0 * n * (n + 1) * (double)count;
    printf("mode %d n=%2d count=%d: %.3f ms  %.0f GB/s (tri r+w)  %.2f us per matrix-slot (%s)\n", RELAPACK_BATCH_MODE, n, count, best,
           tri / best / 1e6, best * 1e3 / count, cudaGetErrorString(cudaGetLastError()));
    cudaFree(d); cudaFree(d0); cudaFree(dp); cudaFree(dn); cudaFree(dinfo);
  }
  return 0;
}
