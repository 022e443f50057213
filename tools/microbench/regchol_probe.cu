// Cycles per register-resident factorization (chol_regs.cuh) vs warps per SM.
#include <cstdio>
#include "../../paper_1602_06763_b200/csrc/chol_regs.cuh"
using namespace relapack;
template <int TN>
__global__ void k_probe(double* out, long long* cyc, int reps) {
  using T = RegTri<TN>;
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  double v[T::NT][2];
  long long total = 0;
  int fails = 0;
  for (int rep = 0; rep < reps; ++rep) {
#pragma unroll
    for (int i = 0; i < TN; ++i)
#pragma unroll
      for (int k = 0; k <= i; ++k)
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          const int r = 8 * i + g, c = 8 * k + 2 * t + q;
          v[T::id(i, k)][q] = (r == c) ? 8.0 * TN + rep : 1.0 / (1 + r + c);
        }
    __syncwarp();
    const long long c0 = clock64();
    fails += reg_potrf<TN>(v, lane);
    __syncwarp();
    total += clock64() - c0;
  }
  double s = fails;
#pragma unroll
  for (int i = 0; i < T::NT; ++i) s += v[i][0] + v[i][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (lane == 0) cyc[blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32] = total / reps;
}
template <int TN>
void run(int wpsm) {
  const int blocks = 148, threads = 32 * wpsm, reps = 50;
  double* out; long long* cyc;
  cudaMalloc(&out, blocks * threads * 8); cudaMalloc(&cyc, blocks * wpsm * 8);
  k_probe<TN><<<blocks, threads>>>(out, cyc, 2);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  k_probe<TN><<<blocks, threads>>>(out, cyc, reps);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  long long h[8]; cudaMemcpy(h, cyc, 8 * 8 < blocks * wpsm * 8 ? 64 : blocks * wpsm * 8, cudaMemcpyDeviceToHost);
  cudaFuncAttributes fa; cudaFuncGetAttributes(&fa, k_probe<TN>);
  printf("n=%2d warps/SM=%2d: %7lld cycles per factorization (warp 0), %.2f us per factorization per warp, regs %d (%s)\n", 8 * TN, wpsm, h[0],
         ms * 1e3 / reps, fa.numRegs, cudaGetErrorString(cudaGetLastError()));
  cudaFree(out); cudaFree(cyc);
}
int main() {
  for (int w : {1, 4, 8}) { run<2>(w); run<4>(w); run<6>(w); run<8>(w); }
  return 0;
}
