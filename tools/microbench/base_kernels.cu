// Times the base-case kernels (K1 potf2, K5 trsm) in isolation, warm, with
// CUDA events around 200 back-to-back launches.  Includes the library sources.
#include <cstdio>
#include <vector>
#define RELAPACK_PROBE 1
#include "../../paper_1602_06763_b200/csrc/potf2.cu"
#include "../../paper_1602_06763_b200/csrc/trsm.cu"
#include "../../paper_1602_06763_b200/csrc/trsm_fused.cu"
namespace relapack {
thread_local TraceRec* g_launch_trace = nullptr;  // defined by driver.cu in the library
}
using namespace relapack;
int main() {
  const int n = 4096;
  std::vector<double> h((size_t)n * n);
  for (int j = 0; j < n; ++j) for (int i = 0; i < n; ++i) h[(size_t)i + (size_t)j * n] = (i == j) ? n : 1.0 / (1 + i + j);
  double* d; cudaMalloc(&d, h.size() * 8);
  int* info; cudaMalloc(&info, 4); cudaMemset(info, 0, 4);
  configure_potf2(); configure_trsm(); configure_trsm_fused();
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  auto time = [&](const char* name, auto fn) {
    for (int w = 0; w < 3; ++w) { cudaMemcpy(d, h.data(), h.size() * 8, cudaMemcpyHostToDevice); fn(); }
    cudaDeviceSynchronize();
    cudaEventRecord(a);
    for (int i = 0; i < 200; ++i) fn();
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    cudaMemset(info, 0, 4);
    printf("%-40s %8.2f us/launch  (%s)\n", name, ms * 1000 / 200, cudaGetErrorString(cudaGetLastError()));
  };
  for (int nb : {1, 8, 16, 32, 64, 96, 128}) {
    char nm[64]; snprintf(nm, 64, "potf2 n=%d layout N", nb);
    time(nm, [&] { launch_potf2(d, n, kLayoutN, nb, info, 0, 0); });
  }
  {
    long long pr[64];
    cudaMemcpyFromSymbol(pr, g_probe, sizeof(pr));
    launch_potf2(d, n, kLayoutN, 64, info, 0, 0);
    cudaDeviceSynchronize();
    cudaMemcpyFromSymbol(pr, g_probe, sizeof(pr));
    printf("potf2 n=64 phases (cycles from start): stage-in %lld |", pr[1] - pr[0]);
    for (int p = 0; p < 8; ++p) printf(" P%d %lld |", p, pr[2 + p] - pr[0]);
    printf(" factor-end %lld end %lld\n", pr[62] - pr[0], pr[63] - pr[0]);
    auto loops = [&](const char* what) {
      for (int p = 0; p < 7; ++p)
        printf("%s loop j0=%2d: warp0 strip_update %5lld factor_panel %5lld | warp1 trail %5lld | barrier end %5lld\n", what, 8 * p,
               pr[12 + p] - (p ? pr[1 + p] : pr[11]), pr[22 + p] - pr[12 + p], pr[32 + p] - (p ? pr[1 + p] : pr[11]),
               pr[2 + p] - (p ? pr[1 + p] : pr[11]));
    };
    loops("potf2 n=64");
    launch_potf2(d, n, kLayoutN, 128, info, 0, 0);
    cudaDeviceSynchronize();
    cudaMemcpyFromSymbol(pr, g_probe, sizeof(pr));
    printf("node128 phases (cycles): load %lld | potf2(A11) %lld | trsm %lld | syrk %lld | potf2(A22) %lld | store %lld\n",
           pr[51] - pr[50], pr[52] - pr[51], pr[53] - pr[52], pr[54] - pr[53], pr[55] - pr[54], pr[56] - pr[55]);
    printf("node128 potf2(A22): first panel %lld\n", pr[11] - pr[54]);
    loops("node128 A22");
    setenv("RELAPACK_NODE128", "0", 1);
    launch_potf2(d, n, kLayoutN, 128, info, 0, 0);
    cudaDeviceSynchronize();
    cudaMemcpyFromSymbol(pr, g_probe, sizeof(pr));
    printf("potf2 n=128 phases (cycles from start): stage-in %lld |", pr[1] - pr[0]);
    for (int p = 0; p < 16; ++p) printf(" P%d %lld |", p, pr[2 + p] - pr[0]);
    printf(" end %lld\n", pr[63] - pr[0]);
  }
  time("potf2 n=64 layout T", [&] { launch_potf2(d, n, kLayoutT, 64, info, 0, 0); });
  time("potf2 n=128 layout T", [&] { launch_potf2(d, n, kLayoutT, 128, info, 0, 0); });
  for (int m : {64, 512, 2048, 8192}) for (int t : {16, 64}) {
    char nm[64]; snprintf(nm, 64, "trsm m=%d t=%d layout N", m, t);
    time(nm, [&] { launch_trsm_base(d, n, d + 64, n, kLayoutN, m, t, info, 0); });
  }
  for (int m : {64, 256, 2048, 8192, 16384}) for (int t : {64, 128, 256}) {
    char nm[64]; snprintf(nm, 64, "trsm_fused m=%d t=%d layout N", m, t);
    time(nm, [&] { launch_trsm_fused(d, n, d + 256, n, kLayoutN, m, t, info, 0); });
  }
  for (int lay : {kLayoutN, kLayoutT})
  for (int m : {128, 8192}) {
    launch_trsm_fused(d, n, d + 256 * (lay == kLayoutN ? 1 : n), n, lay, m, 128, info, 0);
    cudaDeviceSynchronize();
    long long pr[64];
    cudaMemcpyFromSymbol(pr, g_tprobe, sizeof(pr));
    printf("trsm_reg layout %c m=%d load: L issue %lld, slab loads issued %lld, L landed + rinv %lld\n",
           lay == kLayoutN ? 'N' : 'T', m, pr[6] - pr[0], pr[7] - pr[6], pr[1] - pr[7]);
    printf("trsm_reg layout %c m=%d t=128 phases (cycles, CTA 0 thread 0): slab+L %lld | cb0 solve %lld | cb1 update %lld | cb1 solve %lld | store %lld | total %lld\n",
           lay == kLayoutN ? 'N' : 'T', m, pr[1] - pr[0], pr[2] - pr[1], pr[3] - pr[2], pr[4] - pr[3], pr[5] - pr[4], pr[5] - pr[0]);
  }
  for (int m : {2048, 8192}) {
    char nm[64]; snprintf(nm, 64, "trsm_fused m=%d t=128 layout T", m);
    time(nm, [&] { launch_trsm_fused(d, n, d + 256 * n, n, kLayoutT, m, 128, info, 0); });
  }
  time("trsm m=2048 t=64 layout T", [&] { launch_trsm_base(d, n, d + 64 * n, n, kLayoutT, 2048, 64, info, 0); });
  return 0;
}
