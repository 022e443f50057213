// Times the 128-node and 256-node base-case kernels alone (200 back-to-back
// launches, CUDA events) and prints the 256-node's phases (clock64 probes of
// CTA 0 thread 0).  Includes the library sources.
#include <cstdio>
#include <vector>
#define RELAPACK_PROBE 1
#include "../../paper_1602_06763_b200/csrc/potf2.cu"
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
  configure_potf2();
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
  for (int layout : {kLayoutN, kLayoutT}) {
    for (int nb : {128, 192, 256}) {
      char nm[64]; snprintf(nm, 64, "potf2 n=%d layout %c", nb, layout ? 'T' : 'N');
      time(nm, [&] { launch_potf2(d, n, layout, nb, info, 0, 0); });
    }
    long long pr[64];
    launch_potf2(d, n, layout, 256, info, 0, 0);
    cudaDeviceSynchronize();
    cudaMemcpyFromSymbol(pr, g_probe, sizeof(pr));
    printf("node256 layout %c phases (cycles): load %lld | node(A11) %lld | L11 store + A21 load %lld | trsm %lld | "
           "L21 store + syrk %lld | apply %lld | node(A22) %lld | store %lld | total %lld\n", layout ? 'T' : 'N',
           pr[51] - pr[50], pr[62] - pr[51], pr[57] - pr[62], pr[58] - pr[57], pr[59] - pr[58], pr[60] - pr[59],
           pr[55] - pr[60], pr[61] - pr[55], pr[61] - pr[50]);
    printf("node256 A22 node: potf2(A11') %lld | trsm %lld | syrk %lld | potf2(A22') %lld\n", pr[52] - pr[60],
           pr[53] - pr[52], pr[54] - pr[53], pr[55] - pr[54]);
  }
  return 0;
}
