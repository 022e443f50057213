// trsm.cu — K5: the base case of the recursive TRSM (north_star subsystem (3);
// P:292-295; SPEC trsm Right/Lower/Trans/NonUnit):
//     B (m x t) := B * L^{-T},  L a t x t lower-triangular diagonal block,
// i.e. every row x of the result solves x L^T = b by forward substitution
//     x_j = (b_j - sum_{k<j} x_k L_jk) / L_jj.
//
// Rows are independent.  A warp solves R (1..8) rows at once with its 32
// lanes owning the columns (lane l: columns l and l+32), right-looking: at step
// j the lane owning column j broadcasts x_j (one shuffle per row) and every
// lane updates its columns k > j with x_j * L_kj.  The dependent chain is one
// shuffle + one multiply-add per column; the loop body stays small (no
// I-cache-bound full unroll).  L, 1/L_jj and the CTA's row block are staged
// through shared memory with coalesced, batched loads for both layouts.
#include "common.cuh"
#include "kernels.h"

namespace relapack {

namespace {

constexpr int kWarps = 4;
constexpr int kThreads = kWarps * 32;
constexpr int kLd = kTrsmMax + 1;  // 65: odd stride

template <int R>
constexpr size_t smem_bytes() {
  return sizeof(double) * ((size_t)kTrsmMax * kLd + (size_t)kWarps * R * kLd + kTrsmMax);
}

// One half (HI = columns 32..63 or LO = 0..31) of the substitution steps.
template <int R, bool HI>
__device__ __forceinline__ void solve_steps(double (&x0)[R], double (&x1)[R], const double* sL, const double* sRinv,
                                            int jbeg, int jend, int lane) {
  for (int j = jbeg; j < jend; ++j) {
    const double l0 = sL[lane + j * kLd];       // L(lane, j)
    const double l1 = sL[lane + 32 + j * kLd];  // L(lane+32, j)
    const double rj = sRinv[j];
    const int src = j & 31;
    const bool own = lane == src;
    const bool upd0 = !HI && lane > j;
    const bool upd1 = lane + 32 > j;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const double xj = __shfl_sync(0xffffffffu, HI ? x1[r] : x0[r], src) * rj;
      if (own) {
        if (HI)
          x1[r] = xj;
        else
          x0[r] = xj;
      }
      if (upd0) x0[r] -= xj * l0;
      if (upd1) x1[r] -= xj * l1;
    }
  }
}

template <int R>
__global__ void __launch_bounds__(kThreads) k_trsm_base(const double* __restrict__ L, int64_t ldl,
                                                        double* __restrict__ B, int64_t ldb, int layout, int m, int t,
                                                        const int* d_info) {
  if (ld_info(d_info) != 0) return;
  extern __shared__ double smem_d[];
  double* sL = smem_d;                // sL[k + j*kLd] = L(k, j), zero above the diagonal / beyond t
  double* sB = sL + kTrsmMax * kLd;   // sB[r*kLd + j] = B(r0 + r, j)
  constexpr int kRows = kWarps * R;  // rows per CTA
  double* sRinv = sB + kRows * kLd;   // 1 / L(j, j)
  const int r0 = blockIdx.x * kRows;
  const int rows = min(kRows, m - r0);
  const int tid = threadIdx.x;

  // ---- stage L (lower triangle) : coalesced along the contiguous index
  {
    const int total = kTrsmMax * kTrsmMax;
#pragma unroll 4
    for (int e = tid; e < total; e += kThreads) {
      const int a = e & (kTrsmMax - 1), b = e >> 6;  // a fast, b slow
      const int i = layout == kLayoutN ? a : b, j = layout == kLayoutN ? b : a;
      double v = 0.0;
      if (i < t && j < t && i >= j) v = L[lv_off(layout, i, j, ldl)];
      sL[i + j * kLd] = v;
    }
  }
  // ---- stage the row block of B
  {
    const int total = kRows * kTrsmMax;
#pragma unroll 4
    for (int e = tid; e < total; e += kThreads) {
      int r, j;
      if (layout == kLayoutN) {
        r = e % kRows;
        j = e / kRows;
      } else {
        j = e & (kTrsmMax - 1);
        r = e >> 6;
      }
      double v = 0.0;
      if (r < rows && j < t) v = B[lv_off(layout, r0 + r, j, ldb)];
      sB[r * kLd + j] = v;
    }
  }
  __syncthreads();
  if (tid < t) sRinv[tid] = 1.0 / sL[tid + tid * kLd];
  __syncthreads();

  // ---- solve: warp w owns rows w*R .. w*R+R-1, lane owns columns lane, lane+32
  const int warp = tid >> 5, lane = tid & 31;
  double x0[R], x1[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    x0[r] = sB[(warp * R + r) * kLd + lane];
    x1[r] = sB[(warp * R + r) * kLd + lane + 32];
  }
  solve_steps<R, false>(x0, x1, sL, sRinv, 0, min(t, 32), lane);
  solve_steps<R, true>(x0, x1, sL, sRinv, 32, t, lane);
#pragma unroll
  for (int r = 0; r < R; ++r) {
    sB[(warp * R + r) * kLd + lane] = x0[r];
    sB[(warp * R + r) * kLd + lane + 32] = x1[r];
  }
  __syncthreads();
  {
    const int total = kRows * kTrsmMax;
#pragma unroll 4
    for (int e = tid; e < total; e += kThreads) {
      int r, j;
      if (layout == kLayoutN) {
        r = e % kRows;
        j = e / kRows;
      } else {
        j = e & (kTrsmMax - 1);
        r = e >> 6;
      }
      if (r < rows && j < t) B[lv_off(layout, r0 + r, j, ldb)] = sB[r * kLd + j];
    }
  }
}

template <int R>
cudaError_t launch_r(const double* L, int64_t ldl, double* B, int64_t ldb, int layout, int m, int t, const int* d_info,
                     cudaStream_t st) {
  const int grid = (m + kWarps * R - 1) / (kWarps * R);
  k_trsm_base<R><<<grid, kThreads, smem_bytes<R>(), st>>>(L, ldl, B, ldb, layout, m, t, d_info);
  return cudaGetLastError();
}

}  // namespace

cudaError_t configure_trsm() {
  cudaError_t e;
  if ((e = cudaFuncSetAttribute(k_trsm_base<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_bytes<1>())) != cudaSuccess) return e;
  if ((e = cudaFuncSetAttribute(k_trsm_base<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_bytes<2>())) != cudaSuccess) return e;
  if ((e = cudaFuncSetAttribute(k_trsm_base<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_bytes<4>())) != cudaSuccess) return e;
  return cudaFuncSetAttribute(k_trsm_base<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_bytes<8>());
}

cudaError_t launch_trsm_base(const double* L, int64_t ldl, double* B, int64_t ldb, int layout, int m, int t,
                             const int* d_info, cudaStream_t st) {
  if (m <= 0 || t <= 0) return cudaSuccess;
  if (t > kTrsmMax) return cudaErrorInvalidValue;
  // rows per warp: enough warps to cover the SMs ~8 deep before batching rows
  const int warps_wanted = 148 * 8;
  if (m >= warps_wanted * 8) return launch_r<8>(L, ldl, B, ldb, layout, m, t, d_info, st);
  if (m >= warps_wanted * 4) return launch_r<4>(L, ldl, B, ldb, layout, m, t, d_info, st);
  if (m >= warps_wanted * 2) return launch_r<2>(L, ldl, B, ldb, layout, m, t, d_info, st);
  return launch_r<1>(L, ldl, B, ldb, layout, m, t, d_info, st);
}

}  // namespace relapack
