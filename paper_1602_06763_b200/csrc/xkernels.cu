// xkernels.cu — base-case kernels of the other recursive operations of the
// paper (N1 trtri, N2 blocked variants, N3 lauum / potri /
// potrs, N4 getrf).  Their BLAS-3 bulk runs on the update kernel of update.cu
// (mixed operand layouts); these kernels are the recursion's leaves:
//
//   k_tri_rows   every row x of a block B (m x t, t <= 64) against a t x t
//                lower-triangular block T of the L-view (P:292-295 / S:183-191
//                and their transposed forms): x := x T^{-T} (forward solve),
//                x := x T^{-1} (backward solve), x := alpha x T, x := alpha x T^T,
//                unit or non-unit diagonal.  Left-side operations run on the
//                transposed view of B, so one kernel serves every TRSM / TRMM
//                variant the recursions issue.
//   k_trti2      in-place inverse of a t x t lower-triangular block (t <= 64;
//                the paper's "unblocked dtrti2")
//   k_lauu2      in-place L^T L of a t x t lower-triangular block (t <= 64)
//   k_diag_check first zero diagonal entry of the L-view (dtrtri's info)
//   k_getf2      LU with partial pivoting of an m x w panel (w <= 32), one
//                cooperative grid, one grid barrier per column
//   k_laswp      row interchanges ipiv[k0..k1) on a range of columns
//
// Operand X (rows x cols) of layout 0 has element (r, c) at X[r + c*ld],
// layout 1 at X[c + r*ld] (common.cuh lv_off).
#include <cuda_runtime.h>

#include <cstdlib>

#include "chol_regs.cuh"
#include "common.cuh"
#include "kernels.h"
#include "xkernels.h"

#include <cooperative_groups.h>
namespace cg = cooperative_groups;

namespace relapack {

namespace {

constexpr int kTriRows = 128;            // rows (threads) per CTA of k_tri_rows
constexpr int kTriLd = kTriMax + 1;      // odd smem stride: row r's column c at r * kTriLd + c

__device__ __forceinline__ double at(const double* X, int layout, int64_t ld, int r, int c) {
  return X[lv_off(layout, r, c, ld)];
}

// Global -> shared staging with B loads of a thread in flight at once (a
// plain loop waits for every load before the next one: ~0.5 us each).
// idx(e, &src_offset, &dst_offset) -> false if element e is skipped.
template <int B, class Idx>
__device__ __forceinline__ void stage_in(double* dst, const double* src, int total, Idx idx) {
  for (int e0 = threadIdx.x; e0 < total; e0 += blockDim.x * B) {
    double v[B];
    int64_t so[B];
    int dof[B];
    bool ok[B];
#pragma unroll
    for (int u = 0; u < B; ++u) {
      const int e = e0 + u * (int)blockDim.x;
      ok[u] = e < total && idx(e, so[u], dof[u]);
      v[u] = ok[u] ? src[so[u]] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < B; ++u)
      if (ok[u]) dst[dof[u]] = v[u];
  }
}

}  // namespace

// One thread per row of B; the CTA's rows are staged through shared memory
// both ways (global accesses along B's contiguous index; row stride 65, so the
// threads' accesses to one column hit distinct banks).  T is staged once per
// CTA as the strictly triangular part the mode reads — Tm[j][k] = T(j, k) for
// k < j (row sweeps) or Tu[j][k] = T(k, j) for k > j (column sweeps), zero
// elsewhere — plus its diagonal (1 for a unit diagonal), so every dot product
// runs over whole groups of 8 with no bounds: inner loops unrolled by 8 into
// four interleaved partial sums (a quarter of the dependent-FMA chain), T read
// by broadcast.  Solves divide by the diagonal (true division, as the oracle).
template <int MODE>
__global__ void __launch_bounds__(kTriRows) k_tri_rows(XTriArgs a) {
  if (ld_info(a.d_info) != 0) return;
  constexpr int W = kTriMax;                       // 64
  constexpr bool kRows = MODE == kTriSolveLT || MODE == kTriMulLT;  // reads T by rows (else by columns)
  extern __shared__ double sm[];
  double* sT = sm;                                 // W x W masked copy (see above)
  double* sD = sm + W * W;                         // W diagonal entries
  double* sB = sD + W;                             // kTriRows x (W + 1)
  const int t = a.t;
  const int row0 = blockIdx.x * kTriRows;
  const int rows = min(kTriRows, a.m - row0);
  for (int e = threadIdx.x; e < W * W; e += blockDim.x) sT[e] = 0.0;
  for (int j = threadIdx.x; j < W; j += blockDim.x)
    sD[j] = (a.unit || j >= t) ? 1.0 : at(a.T, a.lt, a.ldt, j, j);
  __syncthreads();
  // T(i, j), i > j, i < t, read in the contiguous order of T's layout
  stage_in<8>(sT, a.T, t * t, [&](int e, int64_t& so, int& dof) {
    int i, j;
    if (a.lt == 0) { i = e % t; j = e / t; } else { j = e % t; i = e / t; }
    so = lv_off(a.lt, i, j, a.ldt);
    dof = kRows ? i * W + j : j * W + i;  // Tm[i][j] = T(i, j) (j < i), or Tu[j][i] = T(i, j) (i > j)
    return i > j;
  });
  stage_in<16>(sB, a.B, rows * t, [&](int e, int64_t& so, int& dof) {
    int r, c;
    if (a.lb == 0) { r = e % rows; c = e / rows; } else { c = e % t; r = e / t; }
    so = lv_off(a.lb, row0 + r, c, a.ldb);
    dof = r * (W + 1) + c;
    return true;
  });
  __syncthreads();
  const int r = threadIdx.x;
  if (r < rows) {
    double* x = sB + r * (W + 1);
    for (int c = t; c < W; ++c) x[c] = 0.0;  // padding columns (never stored)
    const double alpha = a.alpha;
    constexpr bool kAsc = MODE == kTriSolveLT || MODE == kTriMulL;  // block order
    constexpr bool kSolve = MODE == kTriSolveLT || MODE == kTriSolveL;
    // 8-column blocks J: the off-diagonal part off[jj] = sum over the blocks K
    // the mode reads (K < J for row sweeps, K > J for column sweeps) of
    // x_K . S[8J + jj][8K .. 8K+7] — eight independent FMA chains, x_K loaded
    // once per block pair, S by 16-byte broadcast loads — then the 8 x 8
    // diagonal block (sequential for the solves).
    for (int bi = 0; bi < W / 8; ++bi) {
      const int J = kAsc ? bi : W / 8 - 1 - bi;
      const int K0 = kRows ? 0 : J + 1, K1 = kRows ? J : W / 8;
      double off[8];
#pragma unroll
      for (int jj = 0; jj < 8; ++jj) off[jj] = 0.0;
      for (int K = K0; K < K1; ++K) {
        double xk[8];
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) xk[kk] = x[8 * K + kk];
#pragma unroll
        for (int jj = 0; jj < 8; ++jj) {
          const double2* srow = reinterpret_cast<const double2*>(sT + (8 * J + jj) * W + 8 * K);
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const double2 sv = srow[q];
            off[jj] = fma(xk[2 * q], sv.x, off[jj]);
            off[jj] = fma(xk[2 * q + 1], sv.y, off[jj]);
          }
        }
      }
      double xj[8], y[8];
#pragma unroll
      for (int jj = 0; jj < 8; ++jj) xj[jj] = x[8 * J + jj];
      if (kSolve) {
        // y_jj = (alpha x_jj - off_jj - sum_{kk before jj} y_kk S[jj][kk]) / D_jj
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int jj = kAsc ? i : 7 - i;
          double acc = fma(alpha, xj[jj], -off[jj]);
#pragma unroll
          for (int kk = 0; kk < 8; ++kk)
            if (kAsc ? kk < jj : kk > jj) acc = fma(-y[kk], sT[(8 * J + jj) * W + 8 * J + kk], acc);
          y[jj] = acc / sD[8 * J + jj];
        }
      } else {
        // y_jj = alpha (x_jj D_jj + sum_{kk in the block's part} x_kk S[jj][kk] + off_jj)
#pragma unroll
        for (int jj = 0; jj < 8; ++jj) {
          double acc = fma(xj[jj], sD[8 * J + jj], off[jj]);
#pragma unroll
          for (int kk = 0; kk < 8; ++kk)
            if (kRows ? kk < jj : kk > jj) acc = fma(xj[kk], sT[(8 * J + jj) * W + 8 * J + kk], acc);
          y[jj] = alpha * acc;
        }
      }
#pragma unroll
      for (int jj = 0; jj < 8; ++jj) x[8 * J + jj] = y[jj];
    }
  }
  __syncthreads();
  for (int e = threadIdx.x; e < rows * t; e += blockDim.x) {
    int rr, c;
    if (a.lb == 0) { rr = e % rows; c = e / rows; } else { c = e % t; rr = e / t; }
    a.B[lv_off(a.lb, row0 + rr, c, a.ldb)] = sB[rr * (W + 1) + c];
  }
}

// ---- DMMA form of the triangular-rows leaf (the same four operations)
// A warp owns 8 rows of B, all t <= 64 columns in registers as eight 8 x 8
// DMMA accumulator tiles (lane (g, q4) holds x(g, 8J + 2 q4 + e)); T sits in
// shared memory as a dense 64 x 64 lower block (zero above the diagonal, 1 on
// a unit diagonal, identity beyond t).  With 8-column blocks J:
//   MulL   x := alpha x T      out_J = sum_{K >= J} x_K T_KJ         (DMMA)
//   MulLT  x := alpha x T^T    out_J = sum_{K <= J} x_K T_JK^T       (DMMA)
//   SolveLT x T^T = b (fwd)    per J ascending: the in-block substitution
//                              (quad shuffles, x_c = y_c * (1 / T_cc)), then
//                              y_J' -= x_J T_J'J^T for J' > J        (DMMA)
//   SolveL  x T = b (bwd)      per J descending: in-block substitution, then
//                              y_J' -= x_J T_JJ' for J' < J          (DMMA)
// (the factorization's register TRSM applied to the other operations: the
// row-per-thread kernel above runs one dependent FMA chain per row).
constexpr int kTriMmaWarps = 8;
constexpr int kTriMmaRows = 8 * kTriMmaWarps;
constexpr int kTriMmaLd = kTriMax + 4;  // column stride: fragment reads at most 2-way conflicted

// BSRC 1 (trti2): B is the identity and the result X^T = T^{-T} (i.e. X =
// T^{-1}, lower) is written over T's strictly lower part (and its diagonal
// unless unit): T X = I solved as rows of X^T T^T = I.
// BSRC 2 (lauu2): B is the transposed view of T (row r = column r of L, only
// its entries c >= r read), MulL gives L^T L, stored as its lower part.
template <int MODE, int UNIT, int BSRC = 0>
__global__ void __launch_bounds__(32 * kTriMmaWarps) k_tri_mma(XTriArgs a) {
  if (ld_info(a.d_info) != 0) return;
  constexpr int W = kTriMax, LD = kTriMmaLd, NB = W / 8;
  extern __shared__ double sm[];
  double* sT = sm;              // T(i, j) at sT[i + j * LD]
  double* sR = sm + W * LD;     // 1 / T(i, i)
  const int t = a.t;
  for (int e = threadIdx.x; e < W * LD; e += blockDim.x) {
    const int i = e % LD, j = e / LD;
    sT[e] = (i == j && (UNIT || j >= t)) ? 1.0 : 0.0;
  }
  __syncthreads();
  stage_in<8>(sT, a.T, t * t, [&](int e, int64_t& so, int& dof) {
    int i, j;
    if (a.lt == 0) { i = e % t; j = e / t; } else { j = e % t; i = e / t; }
    so = lv_off(a.lt, i, j, a.ldt);
    dof = i + j * LD;
    return i > j || (i == j && !UNIT);
  });
  __syncthreads();
  if (MODE == kTriSolveLT || MODE == kTriSolveL)
    for (int i = threadIdx.x; i < W; i += blockDim.x) sR[i] = 1.0 / sT[i + i * LD];
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, q4 = lane & 3;
  const int row = blockIdx.x * kTriMmaRows + 8 * warp + g;
  if (blockIdx.x * kTriMmaRows + 8 * warp >= a.m) return;  // whole warp past the end
  const bool rok = row < a.m;
  double v[NB][2];
#pragma unroll
  for (int J = 0; J < NB; ++J)
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int c = 8 * J + 2 * q4 + e;
      if (BSRC == 1)
        v[J][e] = (rok && c < t && c == row) ? 1.0 : 0.0;
      else
        v[J][e] = (rok && c < t && (BSRC == 0 || c >= row)) ? a.B[lv_off(a.lb, row, c, a.ldb)] : 0.0;
    }
  const int nb = (t + 7) / 8;  // blocks holding columns < t (the rest stay 0)
  if (MODE == kTriMulL || MODE == kTriMulLT) {
    double fr[NB][2];
#pragma unroll
    for (int K = 0; K < NB; ++K) {
      fr[K][0] = tile_frag(v[K][0], v[K][1], 0, g, q4);
      fr[K][1] = tile_frag(v[K][0], v[K][1], 1, g, q4);
    }
#pragma unroll
    for (int J = 0; J < NB; ++J) {
      if (J >= nb) break;
      double o0 = 0.0, o1 = 0.0;
#pragma unroll
      for (int K = 0; K < NB; ++K) {
        if (MODE == kTriMulL ? (K < J || K >= nb) : K > J) continue;
#pragma unroll
        for (int ks = 0; ks < 2; ++ks) {
          // B(kk, n): (T_KJ)(4ks + kk, n) for MulL, (T_JK^T)(4ks + kk, n) = T(8J + n, 8K + 4ks + kk) for MulLT
          const double b = MODE == kTriMulL ? sT[(8 * K + 4 * ks + q4) + (8 * J + g) * LD]
                                            : sT[(8 * J + g) + (8 * K + 4 * ks + q4) * LD];
          dmma_884(o0, o1, fr[K][ks], b);
        }
      }
      v[J][0] = a.alpha * o0;
      v[J][1] = a.alpha * o1;
    }
  } else {
    constexpr bool kFwd = MODE == kTriSolveLT;
#pragma unroll
    for (int i = 0; i < NB; ++i) {
      const int J = kFwd ? i : NB - 1 - i;
      if (J >= nb) continue;
      // in-block substitution: column c of block J final at its owner lane
      // (q4 == c / 2), broadcast in the quad, applied to the lane's columns
      // still to come (c2 = 2 q4 + e after c in the sweep order)
      double tc[8][2];  // T(8J + c2, 8J + c) (fwd: T^T(c, c2)) or T(8J + c, 8J + c2) (bwd)
#pragma unroll
      for (int c = 0; c < 8; ++c)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int c2 = 2 * q4 + e;
          tc[c][e] = kFwd ? sT[(8 * J + c2) + (8 * J + c) * LD] : sT[(8 * J + c) + (8 * J + c2) * LD];
        }
#pragma unroll
      for (int s = 0; s < 8; ++s) {
        const int c = kFwd ? s : 7 - s;
        const int co = c >> 1, ce = c & 1;
        double own = ce ? v[J][1] : v[J][0];
        if (!UNIT) own *= sR[8 * J + c];
        if (q4 == co) {
          if (ce)
            v[J][1] = own;
          else
            v[J][0] = own;
        }
        const double xc = __shfl_sync(0xffffffffu, own, (lane & ~3) | co);
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int c2 = 2 * q4 + e;
          const double nv = fma(-xc, tc[c][e], v[J][e]);
          v[J][e] = (kFwd ? c2 > c : c2 < c) ? nv : v[J][e];
        }
      }
      // the other blocks still to solve: y_J' -= x_J * (T_J'J^T | T_JJ')
      double fr0 = tile_frag(v[J][0], v[J][1], 0, g, q4), fr1 = tile_frag(v[J][0], v[J][1], 1, g, q4);
#pragma unroll
      for (int i2 = i + 1; i2 < NB; ++i2) {
        const int J2 = kFwd ? i2 : NB - 1 - i2;
        if (J2 >= nb) continue;
#pragma unroll
        for (int ks = 0; ks < 2; ++ks) {
          // fwd: B(kk, n) = T^T(8J + 4ks + kk, 8J2 + n) = T(8J2 + n, 8J + 4ks + kk); bwd: T(8J + 4ks + kk, 8J2 + n)
          const double b = kFwd ? sT[(8 * J2 + g) + (8 * J + 4 * ks + q4) * LD]
                                : sT[(8 * J + 4 * ks + q4) + (8 * J2 + g) * LD];
          dmma_884(v[J2][0], v[J2][1], -(ks ? fr1 : fr0), b);
        }
      }
    }
  }
#pragma unroll
  for (int J = 0; J < NB; ++J)
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int c = 8 * J + 2 * q4 + e;
      const bool keep = BSRC == 0 || c > row || (c == row && !UNIT);  // X(c, row) / C(c, row): lower part only
      if (rok && c < t && keep) a.B[lv_off(a.lb, row, c, a.ldb)] = v[J][e];
    }
}

// Inverse of the t x t lower-triangular block in place.  Column j of X = T^{-1}
// is owned by thread j; rows are produced in ascending order, every thread
// reading the same T(i, k) (broadcast) and its own column of X:
//   x_jj = 1 / t_jj;  x_ij = (0 - sum_{k=j}^{i-1} t_ik x_kj) / t_ii.
// diag unit: t_ii = 1 and the diagonal is left untouched.
__global__ void __launch_bounds__(kTriMax) k_trti2(XBlockArgs a) {
  if (ld_info(a.d_info) != 0) return;
  extern __shared__ double sm[];
  double* sT = sm;
  double* sX = sm + kTriMax * kTriLd;  // sX[i * kTriLd + j] = X(i, j)
  const int t = a.n;
  stage_in<16>(sT, a.A, t * t, [&](int e, int64_t& so, int& dof) {
    int i, j;
    if (a.layout == 0) { i = e % t; j = e / t; } else { j = e % t; i = e / t; }
    so = lv_off(a.layout, i, j, a.ld);
    dof = i * kTriLd + j;
    return i >= j;
  });
  __syncthreads();
  const int j = threadIdx.x;
  if (j < t) {
    for (int i = j; i < t; ++i) {
      double s = i == j ? 1.0 : 0.0;
      for (int k = j; k < i; ++k) s -= sT[i * kTriLd + k] * sX[k * kTriLd + j];
      sX[i * kTriLd + j] = a.unit ? s : s / sT[i * kTriLd + i];
    }
  }
  __syncthreads();
  for (int e = threadIdx.x; e < t * t; e += blockDim.x) {
    int i, jj;
    if (a.layout == 0) { i = e % t; jj = e / t; } else { jj = e % t; i = e / t; }
    if (i > jj || (i == jj && !a.unit)) a.A[lv_off(a.layout, i, jj, a.ld)] = sX[i * kTriLd + jj];
  }
}

// L^T L of the t x t lower-triangular block, lower triangle in place:
// c_ij = sum_{k=i}^{t-1} l_ki l_kj (i >= j), ascending k.
__global__ void __launch_bounds__(256) k_lauu2(XBlockArgs a) {
  if (ld_info(a.d_info) != 0) return;
  __shared__ double sT[kTriMax * kTriLd];
  const int t = a.n;
  stage_in<8>(sT, a.A, t * t, [&](int e, int64_t& so, int& dof) {
    int i, j;
    if (a.layout == 0) { i = e % t; j = e / t; } else { j = e % t; i = e / t; }
    so = lv_off(a.layout, i, j, a.ld);
    dof = i * kTriLd + j;
    return i >= j;
  });
  __syncthreads();
  for (int e = threadIdx.x; e < t * t; e += blockDim.x) {
    int i, j;
    if (a.layout == 0) { i = e % t; j = e / t; } else { j = e % t; i = e / t; }
    if (i < j) continue;
    double s = 0.0;
    for (int k = i; k < t; ++k) s += sT[k * kTriLd + i] * sT[k * kTriLd + j];
    a.A[lv_off(a.layout, i, j, a.ld)] = s;
  }
}

// info = 1 + first k with T(k, k) == 0 (0 if none): LAPACK dtrtri's
// singularity check, before anything is modified.
__global__ void k_diag_check(const double* A, int64_t ld, int layout, int n, int* d_info) {
  __shared__ int first;
  if (threadIdx.x == 0) first = 0x7fffffff;
  __syncthreads();
  for (int k = threadIdx.x; k < n; k += blockDim.x)
    if (A[lv_off(layout, k, k, ld)] == 0.0) atomicMin(&first, k);
  __syncthreads();
  if (threadIdx.x == 0) *d_info = first == 0x7fffffff ? 0 : first + 1;
}

// ------------------------------------------------------------------ getrf panel
namespace {

__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// One 16-byte access each, memory-model strong (relaxed.gpu): a record and its
// epoch are read or written whole, and a spin on it is not hoisted (a weak
// load in a loop is; __ldcg on a longlong2 may also be split in two).
__device__ __forceinline__ longlong2 ld16_cg(const longlong2* p) {
  longlong2 v;
  asm volatile(
      "{\n .reg .b128 t;\n ld.relaxed.gpu.global.b128 t, [%2];\n mov.b128 {%0, %1}, t;\n}\n"
      : "=l"(v.x), "=l"(v.y)
      : "l"(p)
      : "memory");
  return v;
}
__device__ __forceinline__ void st16_cg(longlong2* p, longlong2 v) {
  asm volatile("{\n .reg .b128 t;\n mov.b128 t, {%1, %2};\n st.relaxed.gpu.global.b128 [%0], t;\n}\n" ::"l"(p), "l"(v.x),
               "l"(v.y)
               : "memory");
}

// Barrier of the panel warps only (named barrier 1, kGetf2RowThreads threads):
// the interchange warps run decoupled (k_getf2).
__device__ __forceinline__ void panel_sync() {
  asm volatile("bar.sync 1, %0;" ::"n"(kGetf2RowThreads) : "memory");
}

// Grid-wide barrier of the panel warps (all CTAs co-resident: cooperative
// launch); the counter is zeroed before the launch, `phase` counts the
// barriers passed so far.
__device__ __forceinline__ void grid_sync(unsigned* bar, unsigned& phase) {
  panel_sync();
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned target = (phase + 1) * gridDim.x;
    atomicAdd(bar, 1u);
    while (ld_acquire_u32(bar) < target) __nanosleep(32);
    __threadfence();
  }
  ++phase;
  panel_sync();
}

}  // namespace

// LU with partial pivoting of the m x w panel P (layout 0, ld), w <= kGetf2Max,
// rows [0, m); pivots written to ipiv[0..w) as panel-relative row indices plus
// `pivot_base` (the panel's global first row).  CTA g owns rows [g R, g R + R)
// in shared memory.  The panel warps (threads < kGetf2RowThreads), per column
// j: local first-maximum candidate -> published with its whole row (and, by
// the owner, row j) -> grid barrier -> every CTA picks the global first
// maximum, applies the interchange to its rows, divides its multipliers by the
// pivot and updates its rows' trailing columns.  A zero pivot records info
// (min over the launch, atomicMin on getrf_info) and skips the division
// (LAPACK continues).  Candidate slots are double-buffered by column parity (a
// CTA can be at most one barrier ahead of another).  The other warps apply
// each interchange to this CTA's slice of every column outside the panel (the
// recursion's laswp calls, folded in), following the pivots through a
// shared-memory list at their own pace, off the panel's chain.
#ifdef RELAPACK_GETF2_PROBE  // tools/microbench/getf2_probe.cu only: phase cycles accumulated in registers
__device__ long long g_gprobe[8];
#define GPROBE(k)                    \
  {                                  \
    const long long now = clock64(); \
    pacc[k] += now - t_last;         \
    t_last = now;                    \
  }
#else
#define GPROBE(k)
#endif

__global__ void __launch_bounds__(kGetf2Threads) k_getf2(XGetf2Args a) {
  if (ld_info(a.d_info) != 0) return;
#ifdef RELAPACK_GETF2_PROBE
  long long t_last = clock64(), pacc[8] = {};
#endif
  extern __shared__ double sm[];
  const int w = a.w, R = a.rows_per_cta;
  const int g = blockIdx.x, G = gridDim.x;
  const int r0 = g * R;
  const int rows = max(0, min(R, a.m - r0));
  double* sP = sm;                          // rows x w, row-major with stride w + 1
  const int sld = kGetf2Max + 1;
  double* sPiv = sP + (size_t)R * sld;      // the pivot row (w)
  double* sDiag = sPiv + kGetf2Max;         // the old row j (w)
  constexpr int NPW = kGetf2RowThreads / 32;  // panel warps
  __shared__ double red_v[NPW];
  __shared__ int red_i[NPW];
  __shared__ int s_p;
  __shared__ int s_pivots[kGetf2Max];       // panel-relative pivot row of each column (interchange warps)
  __shared__ volatile int s_ready;          // columns whose pivot is in s_pivots
  if (threadIdx.x == 0) s_ready = 0;
  for (int e = threadIdx.x; e < rows * w; e += blockDim.x) {
    const int r = e % rows, c = e / rows;
    sP[r * sld + c] = a.P[(int64_t)(r0 + r) + (int64_t)c * a.ld];
  }
  __syncthreads();
  const int jmax = min(a.m, w);  // pivots exist for the first min(m, w) columns
  if (threadIdx.x >= kGetf2RowThreads) {
    // ---- interchange warps: every column of the matrix outside the panel
    const int total = a.ncols - w;
    const int lo = (int)((int64_t)total * g / G), hi = (int)((int64_t)total * (g + 1) / G);
    const int tid = threadIdx.x - kGetf2RowThreads, nt = blockDim.x - kGetf2RowThreads;
    for (int j = 0; j < jmax; ++j) {
      while (s_ready <= j) __nanosleep(64);
      const int p = s_pivots[j];
      if (p == j) continue;
      for (int x = lo + tid; x < hi; x += nt) {
        double* col = a.A0 + (int64_t)(x < a.c0 ? x : x + w) * a.ld;
        const double u = col[j], v = col[p];
        col[j] = v;
        col[p] = u;
      }
    }
  } else {
    // ---- panel warps
    unsigned phase = 0;
    const unsigned epoch = a.poll ? ((*a.replay) << 16) + a.epoch_base : 0u;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int j = 0; j < jmax; ++j) {
      // (a) local first maximum of |a(i, j)| over owned rows i >= j
      double bv = -1.0;
      int bi = 0x7fffffff;
      for (int r = threadIdx.x; r < rows; r += kGetf2RowThreads) {
        const int gi = r0 + r;
        if (gi < j) continue;
        const double v = fabs(sP[r * sld + j]);
        if (v > bv || (v == bv && gi < bi)) { bv = v; bi = gi; }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
      }
      if (lane == 0) { red_v[warp] = bv; red_i[warp] = bi; }
      panel_sync();
      if (warp == 0) {
        bv = lane < NPW ? red_v[lane] : -1.0;
        bi = lane < NPW ? red_i[lane] : 0x7fffffff;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
          const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
          if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
        }
      }
      // (b) publish: value, index and the candidate row; the owner of row j publishes it too
      const int buf = j & 1;
      if (a.poll) {
        // epoch-stamped 16-byte records, one store each: a reader takes a
        // record once its epoch is this column's (old or new, never torn)
        const unsigned E = epoch + (unsigned)j + 1u;
        longlong2* rec = reinterpret_cast<longlong2*>(a.prec);
        longlong2* rrow = reinterpret_cast<longlong2*>(a.prow);
        longlong2* rdiag = reinterpret_cast<longlong2*>(a.pdiag);
        if (warp == 0) {
          const bool ok = bi != 0x7fffffff;
          for (int c = lane; c < w; c += 32)
            st16_cg(rrow + ((int64_t)buf * G + g) * kGetf2Max + c,
                   make_longlong2(__double_as_longlong(ok ? sP[(bi - r0) * sld + c] : 0.0), (long long)E));
          if (lane == 0)
            st16_cg(rec + buf * G + g, make_longlong2(__double_as_longlong(bv),
                                                     (long long)(((unsigned long long)E << 32) | (unsigned)bi)));
        } else if (warp == 1 && j >= r0 && j < r0 + rows) {
          for (int c = lane; c < w; c += 32)
            st16_cg(rdiag + buf * kGetf2Max + c, make_longlong2(__double_as_longlong(sP[(j - r0) * sld + c]), (long long)E));
        }
        GPROBE(0);
        GPROBE(1);
        if (warp == 0) {
          double v = -1.0;
          int i = 0x7fffffff, who = -1;
          for (int q = lane; q < G; q += 32) {
            longlong2 x;
            do {
              x = ld16_cg(rec + buf * G + q);
            } while ((unsigned)((unsigned long long)x.y >> 32) != E);
            const double qv = __longlong_as_double(x.x);
            const int qi = (int)(unsigned)(x.y & 0xffffffffull);
            if (qi != 0x7fffffff && (qv > v || (qv == v && qi < i))) { v = qv; i = qi; who = q; }
          }
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) {
            const double ov = __shfl_xor_sync(0xffffffffu, v, o);
            const int oi = __shfl_xor_sync(0xffffffffu, i, o);
            const int ow = __shfl_xor_sync(0xffffffffu, who, o);
            if (ov > v || (ov == v && oi < i)) { v = ov; i = oi; who = ow; }
          }
          if (who < 0) i = j;  // no comparable candidate (a NaN column): row j stays, no interchange
          if (lane == 0) {
            s_p = i;
            s_pivots[j] = i;
            __threadfence_block();
            s_ready = j + 1;  // the interchange warps may apply it
          }
          for (int c = lane; c < w; c += 32) {
            longlong2 x;
            do {
              x = ld16_cg(rdiag + buf * kGetf2Max + c);
            } while ((unsigned)x.y != E);
            sDiag[c] = __longlong_as_double(x.x);
            if (who >= 0) {
              do {
                x = ld16_cg(rrow + ((int64_t)buf * G + who) * kGetf2Max + c);
              } while ((unsigned)x.y != E);
            }
            sPiv[c] = __longlong_as_double(x.x);
          }
        }
      } else {
      double* slot_row = a.cand_rows + ((int64_t)buf * G + g) * kGetf2Max;
      if (threadIdx.x == 0) {
        a.cand_val[buf * G + g] = bv;
        a.cand_idx[buf * G + g] = bi;
      }
      if (warp == 0 && bi != 0x7fffffff) {
        const int cand_local = bi - r0;
        for (int c = lane; c < w; c += 32) slot_row[c] = sP[cand_local * sld + c];
      }
      if (j >= r0 && j < r0 + rows)
        for (int c = threadIdx.x; c < w; c += kGetf2RowThreads) a.diag_row[buf * kGetf2Max + c] = sP[(j - r0) * sld + c];
      GPROBE(0);
      // (c) barrier
      grid_sync(a.bar, phase);
      GPROBE(1);
      // (d) global first maximum
      if (warp == 0) {
        double v = -1.0;
        int i = 0x7fffffff, who = -1;
        for (int q = lane; q < G; q += 32) {
          const double qv = __ldcg(a.cand_val + buf * G + q);
          const int qi = __ldcg(a.cand_idx + buf * G + q);
          if (qi != 0x7fffffff && (qv > v || (qv == v && qi < i))) { v = qv; i = qi; who = q; }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          const double ov = __shfl_xor_sync(0xffffffffu, v, o);
          const int oi = __shfl_xor_sync(0xffffffffu, i, o);
          const int ow = __shfl_xor_sync(0xffffffffu, who, o);
          if (ov > v || (ov == v && oi < i)) { v = ov; i = oi; who = ow; }
        }
        if (lane == 0) {
          s_p = i;
          s_pivots[j] = i;
          __threadfence_block();
          s_ready = j + 1;  // the interchange warps may apply it
        }
        const double* wr = a.cand_rows + ((int64_t)buf * G + who) * kGetf2Max;
        for (int c = lane; c < w; c += 32) {
          sPiv[c] = __ldcg(wr + c);
          sDiag[c] = __ldcg(a.diag_row + buf * kGetf2Max + c);
        }
      }
      }  // !poll
      panel_sync();
      const int p = s_p;
      GPROBE(2);
      // (e) interchange rows j and p among the owned rows
      if (p != j) {
        if (j >= r0 && j < r0 + rows)
          for (int c = threadIdx.x; c < w; c += kGetf2RowThreads) sP[(j - r0) * sld + c] = sPiv[c];
        if (p >= r0 && p < r0 + rows)
          for (int c = threadIdx.x; c < w; c += kGetf2RowThreads) sP[(p - r0) * sld + c] = sDiag[c];
      }
      if (g == 0 && threadIdx.x == 0) {
        a.ipiv[j] = a.pivot_base + p;
        if (sPiv[j] == 0.0) atomicMin(a.getrf_info, a.info_base + j + 1);
      }
      panel_sync();
      GPROBE(4);
      // (f) multipliers and the rank-1 update of the owned rows below row j
      const double piv = sPiv[j];
      for (int r = threadIdx.x; r < rows; r += kGetf2RowThreads) {
        const int gi = r0 + r;
        if (gi <= j) continue;
        double l = sP[r * sld + j];
        if (piv != 0.0) l = l / piv;
        sP[r * sld + j] = l;
        for (int c = j + 1; c < w; ++c) sP[r * sld + c] -= l * sPiv[c];
      }
      panel_sync();
      GPROBE(5);
    }
  }
  __syncthreads();
  for (int e = threadIdx.x; e < rows * w; e += blockDim.x) {
    const int r = e % rows, c = e / rows;
    a.P[(int64_t)(r0 + r) + (int64_t)c * a.ld] = sP[r * sld + c];
  }
#ifdef RELAPACK_GETF2_PROBE
  if (threadIdx.x == 0 && blockIdx.x == 0)
    for (int k = 0; k < 8; ++k) g_gprobe[k] = pacc[k];
#endif
}

// ---- cluster panel
// LU with partial pivoting of the m x w panel by one cluster of C CTAs, the
// panel held in REGISTERS: CTA g owns rows [g R, g R + R), thread t its rows
// t + T s (s < S), all W columns (W, S, T compile-time: every register index
// static, runtime column j by predicates).  Per column j (the same
// arithmetic as k_getf2):
//   (a) the first maximum |a(i, j)|, i >= j, of the thread's rows — tracked
//       while column j was updated (step f of column j-1) — reduced over the
//       warp (shuffles) and the CTA;
//   (b) published with the whole candidate row in this CTA's shared memory;
//       the owner of row j publishes row j too (slots by column parity: a CTA
//       is at most one barrier ahead);
//   (c) cluster barrier (barrier.cluster arrive.release / wait.acquire);
//   (d) every CTA reads the C candidates through DSMEM, picks the global first
//       maximum p and reads the pivot row and row j from their publishers;
//   (e) the owners of rows j and p interchange them in their registers;
//   (f) multipliers l = a(i, j) / a(p, j) (true division, as the oracle) and
//       the rank-1 update of the rows below j (a zero pivot records info and
//       skips the division).
// No global-memory round trip and no shared-memory traffic proportional to
// the panel inside the column loop.

template <int T, int S, int W>
__global__ void __launch_bounds__(T) k_getf2_clr(XGetf2ClArgs a) {
  cg::cluster_group cl = cg::this_cluster();
  if (ld_info(a.d_info) != 0) return;  // the same flag for every CTA of the cluster
#ifdef RELAPACK_GETF2_PROBE
  long long t_last = clock64(), pacc[8] = {};
#endif
  constexpr int NW = T / 32;
  const int rank = (int)cl.block_rank(), C = (int)cl.num_blocks();
  const int w = a.w, R = a.rows_per_cta, m = a.m;
  const int r0 = rank * R;
  const int rows = max(0, min(R, m - r0));
  __shared__ double pub[2][2][W];  // [parity][candidate row | row j]
  __shared__ double cand_v[2];
  __shared__ int cand_i[2];
  __shared__ double sPiv[W], sDiag[W];
  __shared__ double red_v[NW];
  __shared__ int red_i[NW];
  __shared__ int s_bi, s_p;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double x[S][W];
#pragma unroll
  for (int s = 0; s < S; ++s) {
    const int r = tid + T * s;
#pragma unroll
    for (int c = 0; c < W; ++c) x[s][c] = (r < rows && c < w) ? a.P[(int64_t)(r0 + r) + (int64_t)c * a.ld] : 0.0;
  }
  // column 0's candidates
  double bv = -1.0;
  int bi = 0x7fffffff;
#pragma unroll
  for (int s = 0; s < S; ++s)
    if (tid + T * s < rows && fabs(x[s][0]) > bv) {  // rows ascend: the first maximum wins ties
      bv = fabs(x[s][0]);
      bi = r0 + tid + T * s;
    }
  cl.sync();
  GPROBE(6);
  const int jmax = min(m, w);
  for (int j = 0; j < jmax; ++j) {
    const int buf = j & 1;
    // (a)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ov > bv || (ov == bv && oi < bi)) {
        bv = ov;
        bi = oi;
      }
    }
    if (lane == 0) {
      red_v[warp] = bv;
      red_i[warp] = bi;
    }
    __syncthreads();
    if (warp == 0) {
      bv = lane < NW ? red_v[lane] : -1.0;
      bi = lane < NW ? red_i[lane] : 0x7fffffff;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ov > bv || (ov == bv && oi < bi)) {
          bv = ov;
          bi = oi;
        }
      }
      if (lane == 0) {
        cand_v[buf] = bv;
        cand_i[buf] = bi;
        s_bi = bi;
      }
    }
    __syncthreads();
    // (b) the owners of the candidate row and of row j publish them
    {
      const int cr = s_bi - r0, jr = j - r0;
#pragma unroll
      for (int s = 0; s < S; ++s) {
        if (cr == tid + T * s)
#pragma unroll
          for (int c = 0; c < W; ++c) pub[buf][0][c] = x[s][c];
        if (jr == tid + T * s)
#pragma unroll
          for (int c = 0; c < W; ++c) pub[buf][1][c] = x[s][c];
      }
    }
    GPROBE(0);
    // (c)
    cl.sync();
    GPROBE(1);
    // (d)
    if (warp == 0) {
      double v = -1.0;
      int i = 0x7fffffff, who = 0;
      if (lane < C) {
        v = *cl.map_shared_rank(&cand_v[buf], lane);
        i = *cl.map_shared_rank(&cand_i[buf], lane);
        who = lane;
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, v, o);
        const int oi = __shfl_xor_sync(0xffffffffu, i, o);
        const int ow = __shfl_xor_sync(0xffffffffu, who, o);
        if (ov > v || (ov == v && oi < i)) {
          v = ov;
          i = oi;
          who = ow;
        }
      }
      if (lane == 0) s_p = i;
      if (lane < W) {
        sPiv[lane] = cl.map_shared_rank(&pub[buf][0][0], who)[lane];
        sDiag[lane] = cl.map_shared_rank(&pub[buf][1][0], j / R)[lane];
      }
    }
    __syncthreads();
    GPROBE(2);
    // (e)
    const int p = s_p;
    if (p != j) {
      const int jr = j - r0, pr = p - r0;
#pragma unroll
      for (int s = 0; s < S; ++s) {
        if (jr == tid + T * s)
#pragma unroll
          for (int c = 0; c < W; ++c) x[s][c] = sPiv[c];
        if (pr == tid + T * s)
#pragma unroll
          for (int c = 0; c < W; ++c) x[s][c] = sDiag[c];
      }
    }
    if (rank == 0 && tid == 0) {
      a.ipiv[j] = a.pivot_base + p;
      if (sPiv[j] == 0.0) atomicMin(a.getrf_info, a.info_base + j + 1);
    }
    GPROBE(4);
    // (f) rows below j; the next column's candidates on the way.  Column j
    // and j + 1 are picked by select chains, so the division and the compare
    // appear once in the code, not once per column.
    const double piv = sPiv[j];
    double pv[W];
#pragma unroll
    for (int c = 0; c < W; ++c) pv[c] = sPiv[c];
    bv = -1.0;
    bi = 0x7fffffff;
#pragma unroll
    for (int s = 0; s < S; ++s) {
      const int r = tid + T * s;
      if (r < rows && r0 + r > j) {
        double xj = x[s][0];
#pragma unroll
        for (int c = 1; c < W; ++c) xj = c == j ? x[s][c] : xj;
        const double l = piv != 0.0 ? xj / piv : xj;
        double xn = 0.0;
        // branch-free per column (selects, not W reconvergence regions)
#pragma unroll
        for (int c = 0; c < W; ++c) {
          const double nv = fma(-l, pv[c], x[s][c]);
          x[s][c] = c == j ? l : ((c > j && c < w) ? nv : x[s][c]);
          xn = c == j + 1 ? x[s][c] : xn;
        }
        if (j + 1 < w && fabs(xn) > bv) {
          bv = fabs(xn);
          bi = r0 + r;
        }
      }
    }
    GPROBE(5);
  }
#pragma unroll
  for (int s = 0; s < S; ++s) {
    const int r = tid + T * s;
#pragma unroll
    for (int c = 0; c < W; ++c)
      if (r < rows && c < w) a.P[(int64_t)(r0 + r) + (int64_t)c * a.ld] = x[s][c];
  }
  cl.sync();  // no CTA leaves while another may still read its published slots
  GPROBE(7);
#ifdef RELAPACK_GETF2_PROBE
  if (threadIdx.x == 0 && cl.block_rank() == 0)
    for (int k = 0; k < 8; ++k) g_gprobe[k] = pacc[k];
#endif
}

// The interchanges of up to 32 consecutive pivots (row k <-> p_k, k ascending,
// p_k >= k, rows relative to the first pivot's row) as one permutation,
// composed by one warp: lane l tracks row l < npiv (cont_lo: the row whose
// value ends there) and extra slot l a pivot row >= npiv.  The moved rows go
// to s_row / s_src (compacted); returns their count (all lanes).
__device__ __forceinline__ int compose_pivots(const int* ipiv, int npiv, int base, int* s_row, int* s_src) {
  const int lane = threadIdx.x & 31;
  int cont_lo = lane, xrow = -1, xcont = -1, ne = 0;
  const int mypiv = lane < npiv ? ipiv[lane] - base : lane;  // all pivots in one load
  for (int k = 0; k < npiv; ++k) {
    const int p = __shfl_sync(0xffffffffu, mypiv, k);
    if (p == k) continue;
    const int ck = __shfl_sync(0xffffffffu, cont_lo, k);
    if (p < npiv) {
      const int cp = __shfl_sync(0xffffffffu, cont_lo, p);
      if (lane == k) cont_lo = cp;
      if (lane == p) cont_lo = ck;
    } else {
      const unsigned mk = __ballot_sync(0xffffffffu, xrow == p);
      int slot;
      if (mk) {
        slot = __ffs(mk) - 1;
      } else {
        slot = ne++;
        if (lane == slot) {
          xrow = p;
          xcont = p;
        }
      }
      const int cp = __shfl_sync(0xffffffffu, xcont, slot);
      if (lane == k) cont_lo = cp;
      if (lane == slot) xcont = ck;
    }
  }
  const bool mv_lo = lane < npiv && cont_lo != lane, mv_x = xrow >= 0 && xcont != xrow;
  const unsigned b_lo = __ballot_sync(0xffffffffu, mv_lo), b_x = __ballot_sync(0xffffffffu, mv_x);
  const int n_lo = __popc(b_lo);
  if (mv_lo) {
    const int at = __popc(b_lo & ((1u << lane) - 1));
    s_row[at] = lane;
    s_src[at] = cont_lo;
  }
  if (mv_x) {
    const int at = n_lo + __popc(b_x & ((1u << lane) - 1));
    s_row[at] = xrow;
    s_src[at] = xcont;
  }
  return n_lo + __popc(b_x);
}

// One panel's interchanges as a permutation: warp 0 composes them
// (compose_pivots), then every warp moves whole columns.
__global__ void __launch_bounds__(256) k_permute(XPermArgs a) {
  if (ld_info(a.d_info) != 0) return;
  __shared__ int s_row[2 * kGetf2Max], s_src[2 * kGetf2Max];
  __shared__ int s_cnt;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (warp == 0) {
    const int cnt = compose_pivots(a.ipiv + a.k0, a.npiv, a.base, s_row, s_src);
    if (lane == 0) s_cnt = cnt;
  }
  __syncthreads();
  const int cnt = s_cnt;
  if (cnt == 0) return;
  const int r0 = lane < cnt ? s_row[lane] : 0, q0 = lane < cnt ? s_src[lane] : 0;
  const int r1 = lane + 32 < cnt ? s_row[lane + 32] : 0, q1 = lane + 32 < cnt ? s_src[lane + 32] : 0;
  const int wpb = blockDim.x >> 5;
  for (int col = blockIdx.x * wpb + warp; col < a.ncols; col += gridDim.x * wpb) {
    double* c = a.A + (int64_t)col * a.ld;
    const double v0 = lane < cnt ? c[q0] : 0.0, v1 = lane + 32 < cnt ? c[q1] : 0.0;
    __syncwarp();
    if (lane < cnt) c[r0] = v0;
    if (lane + 32 < cnt) c[r1] = v1;
  }
}

// Row interchanges: for k = k0 .. k1-1 (in order) swap rows k and ipiv[k] - base
// of the columns [0, ncols) of A (layout 0).  The pivots in chunks of 32, each
// composed into one permutation (compose_pivots, warp 0 of every CTA; the next
// chunk's composition overlaps the moves of the current one: two buffers);
// one warp per column moves the chunk's rows (two loads in flight per lane).
__global__ void __launch_bounds__(256) k_laswp(XLaswpArgs a) {
  if (ld_info(a.d_info) != 0) return;
  __shared__ int s_row[2][2 * kGetf2Max], s_src[2][2 * kGetf2Max];
  __shared__ int s_cnt[2];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nchunks = (a.k1 - a.k0 + 31) / 32;
  if (warp == 0 && nchunks > 0) {
    const int cnt = compose_pivots(a.ipiv + a.k0, min(32, a.k1 - a.k0), a.base + a.k0, s_row[0], s_src[0]);
    if (lane == 0) s_cnt[0] = cnt;
  }
  __syncthreads();
  const int wpb = blockDim.x >> 5;
  for (int ch = 0; ch < nchunks; ++ch) {
    const int cur = ch & 1, k = a.k0 + 32 * ch;
    if (warp == 0 && ch + 1 < nchunks) {  // compose the next chunk into the other buffer
      const int kn = k + 32;
      const int cnt = compose_pivots(a.ipiv + kn, min(32, a.k1 - kn), a.base + kn, s_row[cur ^ 1], s_src[cur ^ 1]);
      if (lane == 0) s_cnt[cur ^ 1] = cnt;
    }
    const int cnt = s_cnt[cur];
    if (cnt > 0) {
      const int r0 = lane < cnt ? k + s_row[cur][lane] : 0, q0 = lane < cnt ? k + s_src[cur][lane] : 0;
      const int r1 = lane + 32 < cnt ? k + s_row[cur][lane + 32] : 0;
      const int q1 = lane + 32 < cnt ? k + s_src[cur][lane + 32] : 0;
      for (int col = blockIdx.x * wpb + warp; col < a.ncols; col += gridDim.x * wpb) {
        double* c = a.A + (int64_t)col * a.ld;
        const double v0 = lane < cnt ? c[q0] : 0.0, v1 = lane + 32 < cnt ? c[q1] : 0.0;
        __syncwarp();
        if (lane < cnt) c[r0] = v0;
        if (lane + 32 < cnt) c[r1] = v1;
      }
    }
    __syncthreads();  // moves of this chunk done (column order), next composition visible
  }
}

// ------------------------------------------------------------------ launchers
constexpr size_t kTriSmem = sizeof(double) * ((size_t)kTriMax * kTriMax + kTriMax + (size_t)kTriRows * (kTriMax + 1));

template <int MODE>
cudaError_t launch_tri_mode(const XTriArgs& a, cudaStream_t st) {
  k_tri_rows<MODE><<<(a.m + kTriRows - 1) / kTriRows, kTriRows, kTriSmem, st>>>(a);
  return cudaGetLastError();
}

template <int MODE>
cudaError_t configure_tri_mode() {
  return cudaFuncSetAttribute(k_tri_rows<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kTriSmem);
}

constexpr size_t kTriMmaSmem = sizeof(double) * ((size_t)kTriMax * kTriMmaLd + kTriMax);

template <int MODE, int UNIT>
cudaError_t launch_tri_mma(const XTriArgs& a, cudaStream_t st) {
  k_tri_mma<MODE, UNIT><<<(a.m + kTriMmaRows - 1) / kTriMmaRows, 32 * kTriMmaWarps, kTriMmaSmem, st>>>(a);
  return cudaGetLastError();
}

template <int MODE>
cudaError_t configure_tri_mma() {
  cudaError_t e = cudaFuncSetAttribute(k_tri_mma<MODE, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kTriMmaSmem);
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(k_tri_mma<MODE, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kTriMmaSmem);
}

// RELAPACK_TRI_MMA=0: the row-per-thread kernel instead of the DMMA one
static bool tri_mma() {
  static const bool v = [] {
    const char* e = getenv("RELAPACK_TRI_MMA");
    return !(e && e[0] == '0');
  }();
  return v;
}

cudaError_t launch_tri_rows(const XTriArgs& a, cudaStream_t st) {
  if (a.m <= 0 || a.t <= 0) return cudaSuccess;
  if (a.t > kTriMax) return cudaErrorInvalidValue;
  if (tri_mma()) {
    const bool u = a.unit != 0;
    switch (a.mode) {
      case kTriSolveLT: return u ? launch_tri_mma<kTriSolveLT, 1>(a, st) : launch_tri_mma<kTriSolveLT, 0>(a, st);
      case kTriSolveL: return u ? launch_tri_mma<kTriSolveL, 1>(a, st) : launch_tri_mma<kTriSolveL, 0>(a, st);
      case kTriMulL: return u ? launch_tri_mma<kTriMulL, 1>(a, st) : launch_tri_mma<kTriMulL, 0>(a, st);
      default: return u ? launch_tri_mma<kTriMulLT, 1>(a, st) : launch_tri_mma<kTriMulLT, 0>(a, st);
    }
  }
  switch (a.mode) {
    case kTriSolveLT: return launch_tri_mode<kTriSolveLT>(a, st);
    case kTriSolveL: return launch_tri_mode<kTriSolveL>(a, st);
    case kTriMulL: return launch_tri_mode<kTriMulL>(a, st);
    default: return launch_tri_mode<kTriMulLT>(a, st);
  }
}

cudaError_t launch_trti2(const XBlockArgs& a, cudaStream_t st) {
  if (a.n <= 0) return cudaSuccess;
  if (a.n > kTriMax) return cudaErrorInvalidValue;
  if (tri_mma()) {
    // T^{-1} as the rows of X^T T^T = I (the DMMA triangular kernel on the
    // identity), written back through the transposed view of T's storage
    XTriArgs t{a.A, a.ld, a.layout, a.A, a.ld, a.layout ^ 1, a.n, a.n, kTriSolveLT, a.unit, 1.0, a.d_info};
    if (a.unit)
      k_tri_mma<kTriSolveLT, 1, 1><<<1, 32 * kTriMmaWarps, kTriMmaSmem, st>>>(t);
    else
      k_tri_mma<kTriSolveLT, 0, 1><<<1, 32 * kTriMmaWarps, kTriMmaSmem, st>>>(t);
    return cudaGetLastError();
  }
  k_trti2<<<1, kTriMax, 2 * sizeof(double) * kTriMax * kTriLd, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_lauu2(const XBlockArgs& a, cudaStream_t st) {
  if (a.n <= 0) return cudaSuccess;
  if (a.n > kTriMax) return cudaErrorInvalidValue;
  if (tri_mma()) {
    // L^T L = (rows of L^T) times L: MulL on the transposed view of the block
    XTriArgs t{a.A, a.ld, a.layout, a.A, a.ld, a.layout ^ 1, a.n, a.n, kTriMulL, 0, 1.0, a.d_info};
    k_tri_mma<kTriMulL, 0, 2><<<1, 32 * kTriMmaWarps, kTriMmaSmem, st>>>(t);
    return cudaGetLastError();
  }
  k_lauu2<<<1, 256, 0, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_diag_check(const double* A, int64_t ld, int layout, int n, int* d_info, cudaStream_t st) {
  k_diag_check<<<1, 256, 0, st>>>(A, ld, layout, n, d_info);
  return cudaGetLastError();
}

size_t getf2_smem(int rows_per_cta) {
  return sizeof(double) * ((size_t)rows_per_cta * (kGetf2Max + 1) + 2 * kGetf2Max);
}

cudaError_t launch_getf2(const XGetf2Args& a, int grid, cudaStream_t st) {
  if (a.m <= 0 || a.w <= 0) return cudaSuccess;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kGetf2Threads);
  cfg.dynamicSmemBytes = getf2_smem(a.rows_per_cta);
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k_getf2, a);
}

cudaError_t launch_laswp(const XLaswpArgs& a, cudaStream_t st) {
  if (a.ncols <= 0 || a.k1 <= a.k0) return cudaSuccess;
  int grid = (a.ncols + 7) / 8;
  if (grid > 148 * 8) grid = 148 * 8;
  k_laswp<<<grid, 256, 0, st>>>(a);
  return cudaGetLastError();
}

// (threads, rows per thread, width) of the register panel for a CTA row count
template <class F>
cudaError_t getf2_clr_dispatch(int rows_per_cta, F&& f) {
  if (rows_per_cta <= kGetf2ClRows32) return f(k_getf2_clr<256, 2, 32>, 256);
  if (rows_per_cta <= kGetf2ClRows16) return f(k_getf2_clr<512, 2, 16>, 512);
  if (rows_per_cta <= kGetf2ClRows8) return f(k_getf2_clr<512, 4, 8>, 512);
  return cudaErrorInvalidValue;
}

// Largest supported cluster size <= want (16 non-portable, 8), 0 if none.
int getf2_cluster_size(int want) {
  static int ok[kMaxDevices][2] = {}, done[kMaxDevices] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= kMaxDevices) return 0;
  if (!done[dev]) {
    done[dev] = 1;
    for (auto k : {k_getf2_clr<256, 2, 32>, k_getf2_clr<512, 2, 16>, k_getf2_clr<512, 4, 8>})
      cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    for (int i = 0; i < 2; ++i) {
      const int c = i == 0 ? 16 : 8;
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(c);
      cfg.blockDim = dim3(512);
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeClusterDimension;
      attr[0].val.clusterDim.x = c;
      attr[0].val.clusterDim.y = 1;
      attr[0].val.clusterDim.z = 1;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      int nc = 0;
      ok[dev][i] = cudaOccupancyMaxActiveClusters(&nc, k_getf2_clr<512, 2, 16>, &cfg) == cudaSuccess && nc > 0;
      cudaGetLastError();
    }
  }
  if (want >= 16 && ok[dev][0]) return 16;
  if (want >= 8 && ok[dev][1]) return 8;
  return 0;
}

int getf2_cluster_caps() {
  // opt-in (RELAPACK_GETF2_CLUSTER=16|8) for the plain recursion: measured
  // slower end to end than the cooperative grid kernel at n = 16384 (225 vs
  // 208 ms, tools/experiments r3q); the lookahead plan uses it by default
  const char* v = getenv("RELAPACK_GETF2_CLUSTER");
  return getf2_cluster_size(v ? atoi(v) : 0);
}

cudaError_t launch_getf2_cl(const XGetf2ClArgs& a, int csize, cudaStream_t st) {
  if (a.m <= 0 || a.w <= 0) return cudaSuccess;
  return getf2_clr_dispatch(a.rows_per_cta, [&](auto kern, int threads) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(csize);
    cfg.blockDim = dim3(threads);
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = csize;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, a);
  });
}

cudaError_t launch_permute(const XPermArgs& a, cudaStream_t st) {
  if (a.ncols <= 0 || a.npiv <= 0) return cudaSuccess;
  int grid = (a.ncols + 7) / 8;
  if (grid > 148 * 8) grid = 148 * 8;
  k_permute<<<grid, 256, 0, st>>>(a);
  return cudaGetLastError();
}

cudaError_t configure_xkernels() {
  cudaError_t e;
  if ((e = configure_tri_mode<kTriSolveLT>()) != cudaSuccess) return e;
  if ((e = configure_tri_mode<kTriSolveL>()) != cudaSuccess) return e;
  if ((e = configure_tri_mode<kTriMulL>()) != cudaSuccess) return e;
  if ((e = configure_tri_mode<kTriMulLT>()) != cudaSuccess) return e;
  if ((e = configure_tri_mma<kTriSolveLT>()) != cudaSuccess) return e;
  if ((e = configure_tri_mma<kTriSolveL>()) != cudaSuccess) return e;
  if ((e = configure_tri_mma<kTriMulL>()) != cudaSuccess) return e;
  if ((e = configure_tri_mma<kTriMulLT>()) != cudaSuccess) return e;
  for (auto k : {k_tri_mma<kTriSolveLT, 0, 1>, k_tri_mma<kTriSolveLT, 1, 1>, k_tri_mma<kTriMulL, 0, 2>})
    if ((e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kTriMmaSmem)) != cudaSuccess)
      return e;
  e = cudaFuncSetAttribute(k_trti2, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)(2 * sizeof(double) * kTriMax * kTriLd));
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(k_getf2, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
}

}  // namespace relapack
