// potf2.cu — K1 (base case of the recursion) and K2 (batched small
// factorizations): Cholesky of a block of order n <= 64 held entirely in one
// SM's shared memory (north_star subsystem (2); P:301-307 crossover to the
// unblocked kernel; "the unblocked kernel is slightly faster ...
// within the processor's L1 cache" -> on the GPU: within shared memory).
//
// Arithmetic per column j (S:219-227 post-condition, right-looking):
//   d = a_jj; stop with info = j+1 if !(d > 0)
//   l_jj = sqrt(d), l_ij = a_ij * rsqrt(d)            i > j
//   a_ik -= l_ij * l_kj                               j < k <= i
// Organisation (latency-bound: the critical path is one dependent chain per
// column): panels of 8 columns are factored by warp 0 entirely in registers
// (lane l holds rows l and l+32 of the panel; pivots and l_kj are broadcast
// with warp shuffles; rsqrt keeps the per-column chain at shuffle + rsqrt +
// multiply-add), then all 4 warps apply the rank-8 trailing update of the
// shared-memory block on the FP64 tensor cores (DMMA.8x8x4, 8x8 tiles, lower
// triangle only).  Two __syncthreads per panel.
#include "common.cuh"
#include "kernels.h"

namespace relapack {

namespace {

constexpr int kNW = 4;               // warps per CTA
constexpr int kP2Threads = kNW * 32;
constexpr int kLds = kPotf2Max + 1;  // 65: odd column stride
constexpr int kPanel = 8;

// Factor the n x n lower triangle of s (column-major, s[i + j*kLds]) in place.
// Returns 0 or the 1-based local column of the first non-positive pivot.
__device__ int potf2_smem(double* s, int n, int* fail_flag) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  for (int j0 = 0; j0 < n; j0 += kPanel) {
    const int w = min(kPanel, n - j0);
    if (warp == 0) {
      // ---- panel factorization in registers (rows i_r = lane + 32 r)
      double x[2][kPanel];
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        const int i = lane + 32 * r;
#pragma unroll
        for (int c = 0; c < kPanel; ++c) x[r][c] = (i < n && c < w && i >= j0 + c) ? s[i + (j0 + c) * kLds] : 0.0;
      }
      int fail = 0;
#pragma unroll
      for (int c = 0; c < kPanel; ++c) {
        if (c < w && !fail) {
          const int j = j0 + c;
          const int jl = j & 31;
          const bool jh = j >= 32;
          const double d = __shfl_sync(0xffffffffu, jh ? x[1][c] : x[0][c], jl);
          if (!(d > 0.0)) {  // catches d <= 0, -0.0 and NaN (uniform across the warp)
            fail = j + 1;
          } else {
            const double rinv = rsqrt(d);
            const double ljj = sqrt(d);
#pragma unroll
            for (int r = 0; r < 2; ++r) {
              const int i = lane + 32 * r;
              x[r][c] = (i == j) ? ljj : x[r][c] * rinv;
            }
#pragma unroll
            for (int c2 = c + 1; c2 < kPanel; ++c2) {
              const int jj = j0 + c2;
              const double l = __shfl_sync(0xffffffffu, jj >= 32 ? x[1][c] : x[0][c], jj & 31);  // l_{jj, j}
#pragma unroll
              for (int r = 0; r < 2; ++r) {
                const int i = lane + 32 * r;
                if (i >= jj) x[r][c2] -= x[r][c] * l;
              }
            }
          }
        }
      }
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        const int i = lane + 32 * r;
#pragma unroll
        for (int c = 0; c < kPanel; ++c)
          if (i < n && c < w && i >= j0 + c) s[i + (j0 + c) * kLds] = x[r][c];
      }
      if (lane == 0 && fail) *fail_flag = fail;
    }
    __syncthreads();
    if (*fail_flag) return *fail_flag;
    // ---- trailing update: A22 -= P2 P2^T on 8x8 tiles (lower triangle), K = 8
    const int r0 = j0 + kPanel;
    if (r0 < n) {
      const int T = (n - r0 + 7) / 8;
      const int ntiles = T * (T + 1) / 2;
      for (int tile = warp; tile < ntiles; tile += kNW) {
        int ti = 0;
        while ((ti + 1) * (ti + 2) / 2 <= tile) ++ti;
        const int tk = tile - ti * (ti + 1) / 2;
        const int i0 = r0 + 8 * ti, k0 = r0 + 8 * tk;
        double c0 = s[(i0 + g) + (k0 + 2 * t) * kLds];
        double c1 = s[(i0 + g) + (k0 + 2 * t + 1) * kLds];
#pragma unroll
        for (int ks = 0; ks < 2; ++ks) {
          const double a = -s[(i0 + g) + (j0 + 4 * ks + t) * kLds];
          const double b = s[(k0 + g) + (j0 + 4 * ks + t) * kLds];
          dmma_884(c0, c1, a, b);
        }
        s[(i0 + g) + (k0 + 2 * t) * kLds] = c0;
        s[(i0 + g) + (k0 + 2 * t + 1) * kLds] = c1;
      }
    }
    __syncthreads();
  }
  return 0;
}

// Copy of the lower triangle of the L-view block between global memory and
// shared memory, coalesced along the contiguous index (layout N: rows; layout
// T: columns of L), every load of a thread in flight at once.
template <bool TO_SMEM>
__device__ __forceinline__ void copy_lower(double* s, double* __restrict__ A, int64_t ld, int layout, int n) {
  constexpr int kPer = (kPotf2Max * kPotf2Max) / kP2Threads;  // 32
  double v[kPer];
#pragma unroll
  for (int u = 0; u < kPer; ++u) {
    const int e = threadIdx.x + u * kP2Threads;
    const int a = e & (kPotf2Max - 1), b = e >> 6;  // a: contiguous index
    const int i = layout == kLayoutN ? a : b, j = layout == kLayoutN ? b : a;
    const bool ok = i < n && j < n && i >= j;
    if (TO_SMEM)
      v[u] = ok ? A[lv_off(layout, i, j, ld)] : 0.0;
    else
      v[u] = s[i + j * kLds];
  }
#pragma unroll
  for (int u = 0; u < kPer; ++u) {
    const int e = threadIdx.x + u * kP2Threads;
    const int a = e & (kPotf2Max - 1), b = e >> 6;
    const int i = layout == kLayoutN ? a : b, j = layout == kLayoutN ? b : a;
    const bool ok = i < n && j < n && i >= j;
    if (TO_SMEM)
      s[i + j * kLds] = v[u];
    else if (ok)
      A[lv_off(layout, i, j, ld)] = v[u];
  }
}

constexpr size_t kSmemBytes = sizeof(double) * kPotf2Max * kLds;

__global__ void __launch_bounds__(kP2Threads) k_potf2_base(double* A, int64_t ld, int layout, int n, int* d_info,
                                                         int info_base) {
  if (ld_info(d_info) != 0) return;
  extern __shared__ double s[];
  __shared__ int fail_flag;
  if (threadIdx.x == 0) fail_flag = 0;
  copy_lower<true>(s, A, ld, layout, n);
  __syncthreads();
  const int fail = potf2_smem(s, n, &fail_flag);
  copy_lower<false>(s, A, ld, layout, n);
  if (fail && threadIdx.x == 0) *d_info = info_base + fail;
}

__global__ void __launch_bounds__(kP2Threads) k_potf2_batched(int layout, int batch, const int* d_n,
                                                            double* const* d_A, const int* d_lda, int* d_info) {
  const int b = blockIdx.x;
  if (b >= batch) return;
  const int n = d_n[b];
  const int lda = d_lda[b];
  if (n < 0 || n > RELAPACK_BATCH_NMAX_) {
    if (threadIdx.x == 0) d_info[b] = -2;
    return;
  }
  if (lda < (n > 1 ? n : 1)) {
    if (threadIdx.x == 0) d_info[b] = -4;
    return;
  }
  extern __shared__ double s[];
  __shared__ int fail_flag;
  if (threadIdx.x == 0) fail_flag = 0;
  double* A = d_A[b];
  int fail = 0;
  if (n > 0) {
    copy_lower<true>(s, A, lda, layout, n);
    __syncthreads();
    fail = potf2_smem(s, n, &fail_flag);
    copy_lower<false>(s, A, lda, layout, n);
  }
  if (threadIdx.x == 0) d_info[b] = fail;
}

}  // namespace

cudaError_t configure_potf2() {
  cudaError_t e = cudaFuncSetAttribute(k_potf2_base, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemBytes);
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(k_potf2_batched, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemBytes);
}

cudaError_t launch_potf2(double* A, int64_t ld, int layout, int n, int* d_info, int info_base, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  if (n > kPotf2Max) return cudaErrorInvalidValue;
  k_potf2_base<<<1, kP2Threads, kSmemBytes, st>>>(A, ld, layout, n, d_info, info_base);
  return cudaGetLastError();
}

cudaError_t launch_potf2_batched(int layout, int batch, const int* d_n, double* const* d_A, const int* d_lda,
                                 int* d_info, cudaStream_t st) {
  if (batch <= 0) return cudaSuccess;
  k_potf2_batched<<<batch, kP2Threads, kSmemBytes, st>>>(layout, batch, d_n, d_A, d_lda, d_info);
  return cudaGetLastError();
}

}  // namespace relapack
