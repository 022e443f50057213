// Per-column timing of the potf2 register panel (warp 0 only), n = 64.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ double rsqrt_nr(double d) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(d));
  const double h = 0.5 * d;
#pragma unroll
  for (int it = 0; it < 2; ++it) { const double e = fma(-h * y, y, 0.5); y = fma(y, e, y); }
  return y;
}
template <int VARIANT>
__global__ void panel(double* out, long long* cyc, int n, int j0) {
  __shared__ double s[64 * 65];
  const int lane = threadIdx.x & 31;
  for (int e = lane; e < 64 * 65; e += 32) s[e] = (e % 66 == 0) ? 64.0 : 0.01 * (e % 7);
  __syncwarp();
  const int w = 8;
  double x[2][8];
  long long t0 = clock64();
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    const int i = lane + 32 * r;
#pragma unroll
    for (int c = 0; c < 8; ++c) x[r][c] = (i < n && c < w && i >= j0 + c) ? s[i + (j0 + c) * 65] : 0.0;
  }
  long long tl = clock64();
  long long tc[8];
  int fail = 0;
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    if (VARIANT == 0 ? (c < w && !fail) : true) {
      const int j = j0 + c;
      const double own = (j >> 5) == 1 ? x[1][c] : x[0][c];
      const double d = __shfl_sync(0xffffffffu, own, j & 31);
      if (VARIANT == 0 && !(d > 0.0)) {
        fail = j + 1;
      } else {
        const double rinv = VARIANT == 2 ? 0.125 : rsqrt_nr(d);
        x[0][c] *= rinv;
        x[1][c] *= rinv;
#pragma unroll
        for (int c2 = c + 1; c2 < 8; ++c2) {
          const int jj = j0 + c2;
          const double src = (jj >> 5) == 1 ? x[1][c] : x[0][c];
          const double l = __shfl_sync(0xffffffffu, src, jj & 31);
          x[0][c2] -= x[0][c] * l;
          x[1][c2] -= x[1][c] * l;
        }
      }
    }
    tc[c] = clock64();
  }
  long long te = clock64();
  double acc = 0;
  for (int r = 0; r < 2; ++r) for (int c = 0; c < 8; ++c) acc += x[r][c];
  out[lane] = acc + fail;
  if (lane == 0) {
    cyc[0] = tl - t0;
    for (int c = 0; c < 8; ++c) cyc[1 + c] = tc[c] - (c ? tc[c - 1] : tl);
    cyc[9] = te - t0;
  }
}
__global__ void panel_new(double* out, long long* cyc, int n, int j0) {
  __shared__ double s[64 * 65];
  const int lane = threadIdx.x & 31;
  for (int e = lane; e < 64 * 65; e += 32) s[e] = (e % 66 == 0) ? 64.0 : 0.01 * (e % 7);
  __syncwarp();
  constexpr int R = 2, kPanel = 8;
  const int w = 8;
  double x[R][8];
  long long t0 = clock64();
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int i = lane + 32 * r;
#pragma unroll
    for (int c = 0; c < 8; ++c) x[r][c] = (i < n && c < w && i >= j0 + c) ? s[i + (j0 + c) * 65] : 0.0;
  }
  long long tl = clock64();
  long long tc[8];
  double dpiv[kPanel], rpiv[kPanel];
  double dnext;
  {
    double own = x[0][0];
    for (int r = 1; r < R; ++r) if ((j0 >> 5) == r) own = x[r][0];
    dnext = own;
  }
#pragma unroll
  for (int c = 0; c < kPanel; ++c) {
    const int j = j0 + c;
    const double d = __shfl_sync(0xffffffffu, dnext, j & 31);
    dpiv[c] = d;
    const double rinv = rsqrt_nr(d);
    rpiv[c] = rinv;
#pragma unroll
    for (int r = 0; r < R; ++r) x[r][c] *= rinv;
    if (c + 1 < kPanel) {
      const int jn = j + 1;
      double xn = x[0][c], an = x[0][c + 1];
#pragma unroll
      for (int r = 1; r < R; ++r) if ((jn >> 5) == r) { xn = x[r][c]; an = x[r][c + 1]; }
      dnext = an - xn * xn;
#pragma unroll
      for (int c2 = c + 1; c2 < kPanel; ++c2) {
        const int jj = j0 + c2;
        double src = x[0][c];
#pragma unroll
        for (int r = 1; r < R; ++r) if ((jj >> 5) == r) src = x[r][c];
        const double l = __shfl_sync(0xffffffffu, src, jj & 31);
#pragma unroll
        for (int r = 0; r < R; ++r) x[r][c2] -= x[r][c] * l;
      }
    }
    tc[c] = clock64();
  }
  long long te = clock64();
  double acc = 0;
  for (int r = 0; r < R; ++r) for (int c = 0; c < 8; ++c) acc += x[r][c] + dpiv[c] + rpiv[c];
  out[lane] = acc;
  if (lane == 0) {
    cyc[0] = tl - t0;
    for (int c = 0; c < 8; ++c) cyc[1 + c] = tc[c] - (c ? tc[c - 1] : tl);
    cyc[9] = te - t0;
  }
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 4096); cudaMalloc(&c, 4096);
  long long h[16];
  const char* names[3] = {"as-in-kernel", "no fail branch", "no rsqrt"};
  for (int v = 0; v < 3; ++v) {
    for (int rep = 0; rep < 2; ++rep) {
      if (v == 0) panel<0><<<1, 32>>>(o, c, 64, 0);
      if (v == 1) panel<1><<<1, 32>>>(o, c, 64, 0);
      if (v == 2) panel<2><<<1, 32>>>(o, c, 64, 0);
    }
    cudaMemcpy(h, c, sizeof(h), cudaMemcpyDeviceToHost);
    printf("%-16s load %lld | cols", names[v], h[0]);
    for (int k = 1; k <= 8; ++k) printf(" %lld", h[k]);
    printf(" | total %lld\n", h[9]);
  }
  for (int rep = 0; rep < 2; ++rep) panel_new<<<1, 32>>>(o, c, 64, 0);
  cudaMemcpy(h, c, sizeof(h), cudaMemcpyDeviceToHost);
  printf("%-16s load %lld | cols", "new chain", h[0]);
  for (int k = 1; k <= 8; ++k) printf(" %lld", h[k]);
  printf(" | total %lld\n", h[9]);
  return 0;
}
