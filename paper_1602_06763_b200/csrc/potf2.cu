// potf2.cu — K1 (base case of the recursion) and K2 (batched small
// factorizations): unblocked Cholesky of a block held entirely in shared
// memory (north_star subsystem (2); P:301-307 crossover to the unblocked
// kernel, "the unblocked kernel is slightly faster ... within the processor's
// L1 cache" P:342-344 -> on the GPU: within one SM's shared memory).
//
// Per column j (right-looking, S:219-227 post-condition):
//   l_jj = sqrt(a_jj)  (stop with info = j+1 if !(a_jj > 0))
//   l_ij = a_ij / l_jj                      i > j
//   a_ik -= l_ij * l_kj                     j < k <= i
// Only one __syncthreads per column: the warp that owns column j+1 of the
// trailing update also finalises it (pivot test, sqrt, scale) right after
// updating it, with warp shuffles broadcasting the pivot.
#include "common.cuh"
#include "kernels.h"

namespace relapack {

namespace {

// Factor the n x n lower triangle of s (column-major, leading dimension lds,
// element (i,j) at s[i + j*lds]) in place; n <= kPotf2Max = 64, 4 warps.
// Returns 0 or the 1-based local column of the first non-positive pivot
// (uniform across the CTA).
//
// Work split: thread (warp w, lane l) owns rows {l, l+32} x columns
// {w, w+4, ..., w+60} of the trailing matrix, so every step's 32 updates per
// thread are independent (loads, then FMAs, then stores).  Column j+1 is
// finalised (pivot test, sqrt, scale by the reciprocal) by its owner warp
// right after its update, so there is one __syncthreads per column.
constexpr int kNW = 4;
constexpr int kCols = kPotf2Max / kNW;  // 16 columns per warp

__device__ __forceinline__ void finalize_column(double* s, int lds, int n, int k, int lane, volatile int* fail_flag) {
  __syncwarp();
  const double d = s[k + k * lds];
  if (!(d > 0.0)) {  // catches d <= 0, -0.0 and NaN
    if (lane == 0) *fail_flag = k + 1;
    return;
  }
  const double r = sqrt(d);
  const double rinv = 1.0 / r;
  const int i0 = k + 1 + lane, i1 = i0 + 32;
  double v0 = 0.0, v1 = 0.0;
  if (i0 < n) v0 = s[i0 + k * lds];
  if (i1 < n) v1 = s[i1 + k * lds];
  if (i0 < n) s[i0 + k * lds] = v0 * rinv;
  if (i1 < n) s[i1 + k * lds] = v1 * rinv;
  __syncwarp();
  if (lane == 0) s[k + k * lds] = r;
}

__device__ int potf2_smem(double* s, int lds, int n, volatile int* fail_flag) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int i0 = lane, i1 = lane + 32;
  if (warp == 0) finalize_column(s, lds, n, 0, lane, fail_flag);
  __syncthreads();
  for (int j = 0; j < n - 1; ++j) {
    if (*fail_flag) return *fail_flag;  // uniform: read after the barrier
    const double* lj = s + j * lds;
    const double li0 = i0 < n ? lj[i0] : 0.0;
    const double li1 = i1 < n ? lj[i1] : 0.0;
    double lk[kCols], a0[kCols], a1[kCols];
#pragma unroll
    for (int c = 0; c < kCols; ++c) {
      const int k = warp + kNW * c;
      const bool colok = k > j && k < n;  // warp-uniform
      lk[c] = colok ? lj[k] : 0.0;
      a0[c] = (colok && i0 >= k && i0 < n) ? s[i0 + k * lds] : 0.0;
      a1[c] = (colok && i1 >= k && i1 < n) ? s[i1 + k * lds] : 0.0;
    }
#pragma unroll
    for (int c = 0; c < kCols; ++c) {
      const int k = warp + kNW * c;
      if (k > j && k < n) {
        if (i0 >= k && i0 < n) s[i0 + k * lds] = a0[c] - li0 * lk[c];
        if (i1 >= k && i1 < n) s[i1 + k * lds] = a1[c] - li1 * lk[c];
      }
    }
    if (warp == (j + 1) % kNW) finalize_column(s, lds, n, j + 1, lane, fail_flag);
    __syncthreads();
  }
  return *fail_flag;
}

// Coalesced copy of the lower triangle of the L-view block between global
// memory and shared memory (layout N: columns contiguous in memory; layout T:
// rows of L contiguous), 8 independent global accesses in flight per thread.
template <bool TO_SMEM>
__device__ void copy_lower(double* s, int lds, double* __restrict__ A, int64_t ld, int layout, int n) {
  const int nth = blockDim.x;
  const int total = n * n;
  for (int e0 = threadIdx.x; e0 < total; e0 += 8 * nth) {
    double v[8];
    int idx[8];
    int64_t goff[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int e = e0 + u * nth;
      const int a = e % n, b = e / n;  // a: contiguous index
      const int i = layout == kLayoutN ? a : b, j = layout == kLayoutN ? b : a;
      const bool ok = e < total && i >= j;
      idx[u] = ok ? i + j * lds : -1;
      goff[u] = lv_off(layout, i, j, ld);
      if (TO_SMEM) v[u] = ok ? A[goff[u]] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      if (idx[u] < 0) continue;
      if (TO_SMEM)
        s[idx[u]] = v[u];
      else
        A[goff[u]] = s[idx[u]];
    }
  }
}

constexpr int kBaseThreads = kNW * 32;

__global__ void __launch_bounds__(kBaseThreads) k_potf2_base(double* A, int64_t ld, int layout, int n, int* d_info,
                                                             int info_base) {
  if (ld_info(d_info) != 0) return;
  extern __shared__ double s[];
  __shared__ int fail_flag;
  const int lds = n | 1;  // odd stride
  if (threadIdx.x == 0) fail_flag = 0;
  copy_lower<true>(s, lds, A, ld, layout, n);
  __syncthreads();
  const int fail = potf2_smem(s, lds, n, &fail_flag);
  copy_lower<false>(s, lds, A, ld, layout, n);
  if (fail && threadIdx.x == 0) *d_info = info_base + fail;
}

constexpr int kBatchThreads = kNW * 32;

__global__ void __launch_bounds__(kBatchThreads) k_potf2_batched(int layout, int batch, const int* d_n,
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
  const int lds = n | 1;
  if (n > 0) {
    copy_lower<true>(s, lds, A, lda, layout, n);
    __syncthreads();
    potf2_smem(s, lds, n, &fail_flag);
    copy_lower<false>(s, lds, A, lda, layout, n);
  }
  if (threadIdx.x == 0) d_info[b] = fail_flag;
}

}  // namespace

cudaError_t configure_potf2() {
  return cudaFuncSetAttribute(k_potf2_base, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (kPotf2Max | 1) * kPotf2Max * (int)sizeof(double));
}

cudaError_t launch_potf2(double* A, int64_t ld, int layout, int n, int* d_info, int info_base, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  if (n > kPotf2Max) return cudaErrorInvalidValue;
  const size_t smem = (size_t)(n | 1) * n * sizeof(double);
  k_potf2_base<<<1, kBaseThreads, smem, st>>>(A, ld, layout, n, d_info, info_base);
  return cudaGetLastError();
}

cudaError_t launch_potf2_batched(int layout, int batch, const int* d_n, double* const* d_A, const int* d_lda,
                                 int* d_info, cudaStream_t st) {
  if (batch <= 0) return cudaSuccess;
  const size_t smem = (size_t)(RELAPACK_BATCH_NMAX_ | 1) * RELAPACK_BATCH_NMAX_ * sizeof(double);
  k_potf2_batched<<<batch, kBatchThreads, smem, st>>>(layout, batch, d_n, d_A, d_lda, d_info);
  return cudaGetLastError();
}

}  // namespace relapack
