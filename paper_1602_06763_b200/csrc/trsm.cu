// trsm.cu — K5: the base case of the recursive TRSM (north_star subsystem (3);
// P:292-295; SPEC trsm Right/Lower/Trans/NonUnit):
//     B (m x t) := B * L^{-T},  L a t x t lower-triangular diagonal block,
// i.e. every row x of the result solves x L^T = b by forward substitution
//     x_j = (b_j - sum_{k<j} x_k L_jk) / L_jj        (x_j = (...) * (1/L_jj)).
//
// Rows are independent.  A warp solves R (1..8) rows at once with its 32 lanes
// owning the columns (lane l: columns l and l+32), right-looking: at step j the
// lane owning column j broadcasts x_j (one shuffle per row) and every lane
// updates its columns with x_j * L_kj, where the staged L is zero on and above
// the diagonal so no per-lane predicates are needed.  The dependent chain per
// column is shuffle -> multiply -> multiply-add.  L, 1/L_jj and the CTA's row
// block are staged through shared memory with every global load of a thread in
// flight at once, coalesced along the contiguous index for both layouts.
#include "common.cuh"
#include "kernels.h"

namespace relapack {

namespace {

constexpr int kWarps = 4;
constexpr int kTsThreads = kWarps * 32;
constexpr int kLd = kTrsmMax + 1;  // 65: odd stride

template <int R>
constexpr size_t smem_bytes() {
  return sizeof(double) * ((size_t)kTrsmMax * kLd + (size_t)kWarps * R * kLd + kTrsmMax);
}

// One half (HI = columns 32..63 or LO = 0..31) of the substitution steps.
template <int R, bool HI>
__device__ __forceinline__ void solve_steps(double (&x0)[R], double (&x1)[R], const double* sL, const double* sRinv,
                                            int jbeg, int jend, int lane) {
#pragma unroll 4
  for (int j = jbeg; j < jend; ++j) {
    const double l0 = sL[lane + j * kLd];       // L(lane, j), 0 unless lane > j
    const double l1 = sL[lane + 32 + j * kLd];  // L(lane+32, j), 0 unless lane+32 > j
    const double rj = sRinv[j];
    const int src = j & 31;
    const bool own = lane == src;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const double xj = __shfl_sync(0xffffffffu, HI ? x1[r] : x0[r], src) * rj;
      if (!HI) x0[r] -= xj * l0;
      x1[r] -= xj * l1;
      if (own) {
        if (HI)
          x1[r] = xj;
        else
          x0[r] = xj;
      }
    }
  }
}

template <int R>
__global__ void __launch_bounds__(kTsThreads) k_trsm_base(const double* __restrict__ L, int64_t ldl,
                                                        double* __restrict__ B, int64_t ldb, int layout, int m, int t,
                                                        const int* d_info, TraceRec* tr) {
  {
    const KState ks = ld_state(d_info);
    if (ks.info != 0) return;
    L = rebase(L, ks.base);
    B = rebase(B, ks.base);
  }
  trace_begin(tr);
  constexpr int kRows = kWarps * R;  // rows per CTA
  extern __shared__ double smem_d[];
  double* sL = smem_d;                // sL[k + j*kLd] = L(k, j) for k > j, else 0
  double* sB = sL + kTrsmMax * kLd;   // sB[r*kLd + j] = B(r0 + r, j)
  double* sRinv = sB + kRows * kLd;   // 1 / L(j, j)
  const int r0 = blockIdx.x * kRows;
  const int rows = min(kRows, m - r0);
  const int tid = threadIdx.x;

  // ---- stage L (strict lower triangle) and the row block of B: all loads first
  constexpr int kPerL = kTrsmMax * kTrsmMax / kTsThreads;  // 32
  constexpr int kPerB = kRows * kTrsmMax / kTsThreads;     // 2R
  double vl[kPerL], vb[kPerB];
#pragma unroll
  for (int u = 0; u < kPerL; ++u) {
    const int e = tid + u * kTsThreads;
    const int a = e & (kTrsmMax - 1), b = e >> 6;  // a: contiguous index
    const int i = layout == kLayoutN ? a : b, j = layout == kLayoutN ? b : a;
    vl[u] = (i < t && j < t && i >= j) ? L[lv_off(layout, i, j, ldl)] : 0.0;
  }
#pragma unroll
  for (int u = 0; u < kPerB; ++u) {
    const int e = tid + u * kTsThreads;
    int r, j;
    if (layout == kLayoutN) {
      r = e % kRows;
      j = e / kRows;
    } else {
      j = e & (kTrsmMax - 1);
      r = e >> 6;
    }
    vb[u] = (r < rows && j < t) ? B[lv_off(layout, r0 + r, j, ldb)] : 0.0;
  }
#pragma unroll
  for (int u = 0; u < kPerL; ++u) {
    const int e = tid + u * kTsThreads;
    const int a = e & (kTrsmMax - 1), b = e >> 6;
    const int i = layout == kLayoutN ? a : b, j = layout == kLayoutN ? b : a;
    if (i == j && i < t) sRinv[i] = 1.0 / vl[u];
    sL[i + j * kLd] = (i > j) ? vl[u] : 0.0;
  }
#pragma unroll
  for (int u = 0; u < kPerB; ++u) {
    const int e = tid + u * kTsThreads;
    int r, j;
    if (layout == kLayoutN) {
      r = e % kRows;
      j = e / kRows;
    } else {
      j = e & (kTrsmMax - 1);
      r = e >> 6;
    }
    sB[r * kLd + j] = vb[u];
  }
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
#pragma unroll
  for (int u = 0; u < kPerB; ++u) {
    const int e = tid + u * kTsThreads;
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
  trace_end(tr);
}

template <int R>
cudaError_t launch_r(const double* L, int64_t ldl, double* B, int64_t ldb, int layout, int m, int t, const int* d_info,
                     cudaStream_t st) {
  const int grid = (m + kWarps * R - 1) / (kWarps * R);
  k_trsm_base<R><<<grid, kTsThreads, smem_bytes<R>(), st>>>(L, ldl, B, ldb, layout, m, t, d_info, g_launch_trace);
  return cudaGetLastError();
}

}  // namespace

cudaError_t configure_trsm() {
  cudaError_t e;
  const auto attr = cudaFuncAttributeMaxDynamicSharedMemorySize;
  if ((e = cudaFuncSetAttribute(k_trsm_base<1>, attr, (int)smem_bytes<1>())) != cudaSuccess) return e;
  if ((e = cudaFuncSetAttribute(k_trsm_base<2>, attr, (int)smem_bytes<2>())) != cudaSuccess) return e;
  if ((e = cudaFuncSetAttribute(k_trsm_base<4>, attr, (int)smem_bytes<4>())) != cudaSuccess) return e;
  return cudaFuncSetAttribute(k_trsm_base<8>, attr, (int)smem_bytes<8>());
}

cudaError_t launch_trsm_base(const double* L, int64_t ldl, double* B, int64_t ldb, int layout, int m, int t,
                             const int* d_info, cudaStream_t st) {
  if (m <= 0 || t <= 0) return cudaSuccess;
  if (t > kTrsmMax) return cudaErrorInvalidValue;
  // The per-warp time is the length-t dependent chain whatever R is, so batch
  // R rows per warp as long as the grid still spreads over the 148 SMs.
  const int ctas_per_r1 = (m + kWarps - 1) / kWarps;
  if (ctas_per_r1 >= 148 * 8) return launch_r<8>(L, ldl, B, ldb, layout, m, t, d_info, st);
  if (ctas_per_r1 >= 148 * 4) return launch_r<4>(L, ldl, B, ldb, layout, m, t, d_info, st);
  if (ctas_per_r1 >= 148 * 2) return launch_r<2>(L, ldl, B, ldb, layout, m, t, d_info, st);
  return launch_r<1>(L, ldl, B, ldb, layout, m, t, d_info, st);
}

}  // namespace relapack
