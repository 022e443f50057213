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
  const int C = getf2_cluster_caps();  // 0 unless RELAPACK_GETF2_CLUSTER is set
  const size_t cap = 0;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  if (C > 0) {
  XGetf2ClArgs a{};
  a.P = d; a.ld = m; a.m = m; a.w = w; a.rows_per_cta = (m + C - 1) / C; a.ipiv = ipiv; a.pivot_base = 1;
  a.getrf_info = info + 1; a.info_base = 0; a.d_info = info;
  printf("cluster %d, rows/CTA %d (%zu)\n", C, a.rows_per_cta, cap);
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
  }
  // the cooperative grid kernel (k_getf2) on the same panel, grid barrier (poll 0)
  // and epoch-stamped exchange (poll 1); the two must give identical results
  {
    const int rows_coop = argc > 3 ? atoi(argv[3]) : 32;
    const int G = (m + rows_coop - 1) / rows_coop;
    unsigned* bar; double* cand; int* cidx; void* pws; unsigned* rep;
    cudaMalloc(&bar, 4); cudaMalloc(&cand, (2 * G + 2 * G * kGetf2Max + 2 * kGetf2Max) * 8); cudaMalloc(&cidx, 2 * G * 4);
    const size_t pb = 2 * 160 * 16 + 2 * 160 * kGetf2Max * 16 + 2 * kGetf2Max * 16;
    cudaMalloc(&pws, pb); cudaMemset(pws, 0, pb); cudaMalloc(&rep, 4); cudaMemset(rep, 0, 4);
    std::vector<double> out[2];
    std::vector<int> piv[2];
    for (int poll = 0; poll < 2; ++poll) {
      XGetf2Args g{};
      g.P = d; g.ld = m; g.m = m; g.w = w; g.rows_per_cta = rows_coop; g.ipiv = ipiv; g.pivot_base = 1;
      g.getrf_info = info + 1; g.info_base = 0; g.bar = bar; g.cand_val = cand; g.cand_rows = cand + 2 * G;
      g.diag_row = cand + 2 * G + 2 * G * kGetf2Max; g.cand_idx = cidx; g.A0 = d; g.ncols = w; g.c0 = 0; g.d_info = info;
      g.poll = poll; g.epoch_base = 0; g.replay = rep; g.prec = pws; g.prow = (char*)pws + 2 * 160 * 16;
      g.pdiag = (char*)pws + 2 * 160 * 16 + 2 * 160 * kGetf2Max * 16;
      cudaFuncSetAttribute(k_getf2, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      float bestc = 1e9;
      for (int rep_i = 0; rep_i < 5; ++rep_i) {
        cudaMemcpy(d, d0, h.size() * 8, cudaMemcpyDeviceToDevice);
        cudaMemset(bar, 0, 4);
        unsigned rv = rep_i + 1 + 10 * poll;
        cudaMemcpy(rep, &rv, 4, cudaMemcpyHostToDevice);
        long long z[8] = {};
        cudaMemcpyToSymbol(g_gprobe, z, sizeof(z));
        cudaDeviceSynchronize();
        cudaEventRecord(e0);
        cudaError_t e = launch_getf2(g, G, 0);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        if (ms < bestc) bestc = ms;
        if (rep_i == 4) {
          long long p[8];
          cudaMemcpyFromSymbol(p, g_gprobe, sizeof(p));
          printf("coop poll=%d m=%d w=%d G=%d: %.1f us (%s); per column cycles: max+publish %lld | grid barrier %lld | global pick + rows %lld | swap %lld | update %lld\n",
                 poll, m, w, G, bestc * 1e3, cudaGetErrorString(e), p[0] / w, p[1] / w, p[2] / w, p[4] / w, p[5] / w);
          out[poll].resize(h.size());
          piv[poll].resize(w);
          cudaMemcpy(out[poll].data(), d, h.size() * 8, cudaMemcpyDeviceToHost);
          cudaMemcpy(piv[poll].data(), ipiv, w * 4, cudaMemcpyDeviceToHost);
        }
      }
    }
    int firstbad = -1;
    for (int j = 0; j < w && firstbad < 0; ++j) if (piv[0][j] != piv[1][j]) firstbad = j;
    size_t diff = 0;
    for (size_t i = 0; i < h.size(); ++i) diff += out[0][i] != out[1][i];
    printf("poll vs barrier: first differing pivot %d, differing entries %zu\n", firstbad, diff);
    if (firstbad >= 0) { for (int j = 0; j < w; ++j) printf("%d/%d ", piv[0][j], piv[1][j]); printf("\n"); }
  }
  return 0;
}
