// Times the getrf cluster panel kernel (k_getf2_cl) alone on an m x w panel
// and prints its per-phase cycles (CTA 0, thread 0, summed over the columns).
#include <cstdio>
#include <cstdlib>
#include <vector>
#define RELAPACK_GETF2_PROBE 1
#include "../../paper_1602_06763_b200/csrc/xkernels.cu"
using namespace relapack;
int main(int argc, char** argv) {
  const int m = argc > 1 ? atoi(argv[1]) : 16384, w = argc > 2 ? atoi(argv[2]) : 16;
  std::vector<double> h((size_t)m * w);
  srand(1);
  for (auto& x : h) x = 2.0 * rand() / RAND_MAX - 1.0;
  double *d, *d0; int *ipiv, *info;
  cudaMalloc(&d, h.size() * 8); cudaMalloc(&d0, h.size() * 8); cudaMalloc(&ipiv, w * 4); cudaMalloc(&info, 16);
  cudaMemcpy(d0, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
  cudaMemset(info, 0, 16);
  const int C = getf2_cluster_caps();
  const size_t cap = 0;
  XGetf2ClArgs a{};
  a.P = d; a.ld = m; a.m = m; a.w = w; a.rows_per_cta = (m + C - 1) / C; a.ipiv = ipiv; a.pivot_base = 1;
  a.getrf_info = info + 1; a.info_base = 0; a.d_info = info;
  printf("cluster %d, rows/CTA %d (%zu)\n", C, a.rows_per_cta, cap);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float best = 1e9;
  for (int rep = 0; rep < 5; ++rep) {
    cudaMemcpy(d, d0, h.size() * 8, cudaMemcpyDeviceToDevice);
    long long z[8] = {};
    cudaMemcpyToSymbol(g_gprobe, z, sizeof(z));
    cudaDeviceSynchronize();
    cudaEventRecord(e0);
    cudaError_t e = launch_getf2_cl(a, C, 0);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
    if (rep == 4) {
      long long p[8];
      cudaMemcpyFromSymbol(p, g_gprobe, sizeof(p));
      printf("m=%d w=%d: %.1f us (%s); per column cycles: max+publish %lld | cluster sync %lld | global pick + rows %lld | swap %lld | update %lld; load %lld, store %lld\n",
             m, w, best * 1e3, cudaGetErrorString(e), p[0] / w, p[1] / w, p[2] / w, p[4] / w, p[5] / w, p[6], p[7]);
    }
  }
  return 0;
}
