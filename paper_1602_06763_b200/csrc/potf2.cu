// potf2.cu — K1 (base case of the recursion, order n <= 128): Cholesky of a
// block held entirely in one SM's shared memory (north_star subsystem (2); P:301-307 crossover to the
// unblocked kernel; "the unblocked kernel is slightly faster ...
// within the processor's L1 cache" -> on the GPU: within shared memory).
//
// Arithmetic per column j (S:219-227 post-condition, right-looking):
//   d = a_jj; stop with info = j+1 if !(d > 0)
//   l_jj = sqrt(d), l_ij = a_ij * (1/sqrt(d))         i > j
//   a_ik -= l_ij * l_kj                               j < k <= i
// Organisation (latency-bound: the critical path is one dependent chain per
// column): panels of 8 columns are factored by warp 0 in registers (lane l
// holds rows l, l+32, ... of the panel; the pivot and l_kj are broadcast with
// warp shuffles).  The per-column chain is shuffle -> rsqrt (MUFU.RSQ64H + two
// branch-free Newton steps) -> multiply-add on the lane of the next row ->
// shuffle; l_jj = sqrt(d) is formed off the chain from the same rsqrt.
// The rank-8 trailing updates of the shared-memory block run on the FP64
// tensor cores (DMMA.8x8x4 on 8x8 tiles, lower triangle only) with a one-panel
// lookahead: warp 0 updates and factors the next panel while the other warps
// update the rest.  One __syncthreads per panel.
#include "common.cuh"
#include "kernels.h"

namespace relapack {

namespace {

constexpr int kPanel = 8;

#ifdef RELAPACK_PROBE  // phase timestamps for tools/microbench/base_kernels.cu only
__device__ long long g_probe[64];
#define PROBE(k) \
  if (threadIdx.x == 0 && blockIdx.x == 0) g_probe[k] = clock64();
#else
#define PROBE(k)
#endif

template <int NMAX>
struct P2 {
  static constexpr int NW = NMAX / 16;         // 4 warps (64) / 8 warps (128)
  static constexpr int THREADS = NW * 32;
  static constexpr int LDS = NMAX + 1;         // odd column stride
  static constexpr int RPL = NMAX / 32;        // panel rows per lane
  static constexpr size_t SMEM = sizeof(double) * NMAX * LDS;
};

// Apply the rank-8 update of panel columns [j0, j0+8) to the 8x8 tiles
// (ti, tk), tile index range [t_beg, t_end) of the lower-triangular tile grid
// whose first row/column is r0; tiles with tk < tk_min are skipped.  Two tiles
// are in flight per warp (DMMA.8x8x4, K = 8 -> 2 dependent DMMA per tile).
template <int LDS>
__device__ __forceinline__ void trail_tiles(double* s, int j0, int r0, int tile_beg, int tile_end, int tile_step,
                                            int g, int t) {
  for (int base = tile_beg; base < tile_end; base += 2 * tile_step) {
    double c0[2], c1[2];
    int ii[2], kk[2];
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int tile = base + q * tile_step;
      int ti = 0;
      while ((ti + 1) * (ti + 2) / 2 <= tile) ++ti;
      const int tk = tile - ti * (ti + 1) / 2;
      ii[q] = r0 + 8 * ti;
      kk[q] = r0 + 8 * tk;
      const bool ok = tile < tile_end;
      c0[q] = ok ? s[(ii[q] + g) + (kk[q] + 2 * t) * LDS] : 0.0;
      c1[q] = ok ? s[(ii[q] + g) + (kk[q] + 2 * t + 1) * LDS] : 0.0;
    }
#pragma unroll
    for (int ks = 0; ks < 2; ++ks) {
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        if (base + q * tile_step < tile_end) {
          const double a = -s[(ii[q] + g) + (j0 + 4 * ks + t) * LDS];
          const double b = s[(kk[q] + g) + (j0 + 4 * ks + t) * LDS];
          dmma_884(c0[q], c1[q], a, b);
        }
      }
    }
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      if (base + q * tile_step < tile_end) {
        s[(ii[q] + g) + (kk[q] + 2 * t) * LDS] = c0[q];
        s[(ii[q] + g) + (kk[q] + 2 * t + 1) * LDS] = c1[q];
      }
    }
  }
}

// Update the 8-column strip [r0, r0+8) (rows >= r0) with panel [j0, j0+8):
// the tiles (ti, 0) of the trailing grid, all in flight at once (warp 0).
template <int NMAX, int LDS>
__device__ __forceinline__ void strip_update(double* s, int n, int j0, int r0, int g, int t) {
  constexpr int TMAX = NMAX / 8, QB = TMAX < 8 ? TMAX : 8;  // tiles in flight (register budget)
  const int T = (n - r0 + 7) / 8;
#pragma unroll 1
  for (int q0 = 0; q0 < T; q0 += QB) {
    double c0[QB], c1[QB];
#pragma unroll
    for (int q = 0; q < QB; ++q) {
      if (q0 + q < T) {
        c0[q] = s[(r0 + 8 * (q0 + q) + g) + (r0 + 2 * t) * LDS];
        c1[q] = s[(r0 + 8 * (q0 + q) + g) + (r0 + 2 * t + 1) * LDS];
      }
    }
#pragma unroll
    for (int ks = 0; ks < 2; ++ks) {
      const double b = s[(r0 + g) + (j0 + 4 * ks + t) * LDS];
#pragma unroll
      for (int q = 0; q < QB; ++q) {
        if (q0 + q < T) {
          const double a = -s[(r0 + 8 * (q0 + q) + g) + (j0 + 4 * ks + t) * LDS];
          dmma_884(c0[q], c1[q], a, b);
        }
      }
    }
#pragma unroll
    for (int q = 0; q < QB; ++q) {
      if (q0 + q < T) {
        s[(r0 + 8 * (q0 + q) + g) + (r0 + 2 * t) * LDS] = c0[q];
        s[(r0 + 8 * (q0 + q) + g) + (r0 + 2 * t + 1) * LDS] = c1[q];
      }
    }
  }
}

// Factor panel [j0, j0 + 8) (rows j0..n-1, already fully updated) in warp 0's
// registers and store it.  Returns the 1-based failing column or 0.
template <int NMAX>
__device__ __forceinline__ int factor_panel(double* s, int n, int j0, int lane) {
  using C = P2<NMAX>;
  constexpr int LDS = C::LDS, R = C::RPL;
  const int w = min(kPanel, n - j0);
  double x[R][kPanel];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int i = lane + 32 * r;
#pragma unroll
    for (int c = 0; c < kPanel; ++c) x[r][c] = (i < n && c < w && i >= j0 + c) ? s[i + (j0 + c) * LDS] : 0.0;
  }
  // Updates go to every row of the panel (rows above a column's diagonal hold
  // don't-care values that are never stored): no predicates on the chain.  The
  // critical path per column is: shuffle the pivot d_j -> rsqrt -> (lane of
  // row j+1) l = a*rinv, d_{j+1} = a' - l*l -> shuffle.  A non-positive pivot
  // turns the rest of the panel into NaN/garbage; it is detected once per
  // panel from the saved pivots (first failing column).
  double dpiv[kPanel], rpiv[kPanel];
  double dnext;
  {
    double own = x[0][0];
#pragma unroll
    for (int r = 1; r < R; ++r)
      if ((j0 >> 5) == r) own = x[r][0];
    dnext = own;  // lane (j0 & 31) holds a_{j0,j0}
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
      // the lane holding row j+1 forms the next pivot from its own registers
      const int jn = j + 1;
      double xn = x[0][c], an = x[0][c + 1];
#pragma unroll
      for (int r = 1; r < R; ++r)
        if ((jn >> 5) == r) {
          xn = x[r][c];
          an = x[r][c + 1];
        }
      dnext = an - xn * xn;
#pragma unroll
      for (int c2 = c + 1; c2 < kPanel; ++c2) {
        const int jj = j0 + c2;
        double src = x[0][c];
#pragma unroll
        for (int r = 1; r < R; ++r)
          if ((jj >> 5) == r) src = x[r][c];
        const double l = __shfl_sync(0xffffffffu, src, jj & 31);  // l_{jj, j}
#pragma unroll
        for (int r = 0; r < R; ++r) x[r][c2] -= x[r][c] * l;
      }
    }
  }
  int fail = 0;
#pragma unroll
  for (int c = kPanel - 1; c >= 0; --c)
    if (c < w && !(dpiv[c] > 0.0)) fail = j0 + c + 1;  // catches d <= 0, -0.0 and NaN
  // diagonal entries l_jj = sqrt(d), off the critical path
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int i = lane + 32 * r;
#pragma unroll
    for (int c = 0; c < kPanel; ++c) {
      if (i == j0 + c) x[r][c] = sqrt_from_rsqrt(dpiv[c], rpiv[c]);
      if (i < n && c < w && i >= j0 + c) s[i + (j0 + c) * LDS] = x[r][c];
    }
  }
  return fail;
}

// Factor the n x n lower triangle of s (column-major, s[i + j*LDS]) in place.
// Returns 0 or the 1-based local column of the first non-positive pivot.
// Lookahead: while warp 0 updates the next panel's strip and factors it,
// the other warps apply the current panel to the rest of the trailing
// matrix, so one __syncthreads per panel and the bulk update is off the
// critical path.
template <int NMAX>
__device__ int potf2_smem(double* s, int n, int* fail_flag) {
  using C = P2<NMAX>;
  constexpr int LDS = C::LDS;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  if (warp == 0) {
    const int f = factor_panel<NMAX>(s, n, 0, lane);
    if (lane == 0 && f) *fail_flag = f;
  }
  __syncthreads();
  for (int j0 = 0; j0 < n; j0 += kPanel) {
    if (*fail_flag) return *fail_flag;  // uniform: read after the barrier
    const int r0 = j0 + kPanel;
    if (r0 >= n) break;
    if (warp == 0) {
      strip_update<NMAX, LDS>(s, n, j0, r0, g, t);
      __syncwarp();
      const int f = factor_panel<NMAX>(s, n, r0, lane);
      if (lane == 0 && f) *fail_flag = f;
    } else {
      // tiles of the trailing grid with tk >= 1 (columns >= r0 + 8)
      const int T = (n - r0 + 7) / 8;
      const int ntiles = T * (T + 1) / 2;
      // enumerate tiles with tk >= 1: tile index over the grid starting at r0+8
      if (T > 1) {
        const int T2 = T - 1;
        const int nt2 = T2 * (T2 + 1) / 2;  // lower tiles of the grid rooted at (r0+8, r0+8)
        trail_tiles<LDS>(s, j0, r0 + 8, warp - 1, nt2, C::NW - 1, g, t);
      }
      (void)ntiles;
    }
    PROBE(2 + (j0 / kPanel) % 60);
    __syncthreads();
  }
  return *fail_flag;
}

// Copy of the lower triangle of the L-view block between global memory and
// shared memory, coalesced along the contiguous index (layout N: rows; layout
// T: columns of L), 32 loads of a thread in flight at once.
template <int NMAX, bool TO_SMEM>
__device__ __forceinline__ void copy_lower(double* s, double* __restrict__ A, int64_t ld, int layout, int n) {
  using C = P2<NMAX>;
  constexpr int kBatch = 16;
  constexpr int kPer = NMAX * NMAX / C::THREADS;  // 32 (64) or 64 (128)
  // NMAX = 128: not unrolled, so the index math is recomputed per batch
  // instead of being kept live (spilled) across the kernel for the copy back
#pragma unroll(NMAX <= 64 ? kPer / kBatch : 1)
  for (int u0 = 0; u0 < kPer; u0 += kBatch) {
    double v[kBatch];
#pragma unroll
    for (int u = 0; u < kBatch; ++u) {
      const int e = threadIdx.x + (u0 + u) * C::THREADS;
      const int a = e % NMAX, b = e / NMAX;  // a: contiguous index
      const int i = layout == kLayoutN ? a : b, j = layout == kLayoutN ? b : a;
      const bool ok = i < n && j < n && i >= j;
      if (TO_SMEM)
        v[u] = ok ? A[lv_off(layout, i, j, ld)] : 0.0;
      else
        v[u] = s[i + j * C::LDS];
    }
#pragma unroll
    for (int u = 0; u < kBatch; ++u) {
      const int e = threadIdx.x + (u0 + u) * C::THREADS;
      const int a = e % NMAX, b = e / NMAX;
      const int i = layout == kLayoutN ? a : b, j = layout == kLayoutN ? b : a;
      const bool ok = i < n && j < n && i >= j;
      if (TO_SMEM)
        s[i + j * C::LDS] = v[u];
      else if (ok)
        A[lv_off(layout, i, j, ld)] = v[u];
    }
  }
}

constexpr int kBaseMax = kPotf2Max;  // 128

__global__ void __launch_bounds__(P2<kBaseMax>::THREADS) k_potf2_base(double* A, int64_t ld, int layout, int n,
                                                                       int* d_info, int info_base) {
  PROBE(0);
  if (ld_info(d_info) != 0) return;
  extern __shared__ double s[];
  __shared__ int fail_flag;
  if (threadIdx.x == 0) fail_flag = 0;
  copy_lower<kBaseMax, true>(s, A, ld, layout, n);
  __syncthreads();
  PROBE(1);
  const int fail = potf2_smem<kBaseMax>(s, n, &fail_flag);
  copy_lower<kBaseMax, false>(s, A, ld, layout, n);
  if (fail && threadIdx.x == 0) *d_info = info_base + fail;
  PROBE(63);
}

// Same kernel sized for n <= 64 (4 warps, 33 KB): used when the block is small.
__global__ void __launch_bounds__(P2<64>::THREADS) k_potf2_base64(double* A, int64_t ld, int layout, int n,
                                                                  int* d_info, int info_base) {
  if (ld_info(d_info) != 0) return;
  extern __shared__ double s[];
  __shared__ int fail_flag;
  if (threadIdx.x == 0) fail_flag = 0;
  copy_lower<64, true>(s, A, ld, layout, n);
  __syncthreads();
  const int fail = potf2_smem<64>(s, n, &fail_flag);
  copy_lower<64, false>(s, A, ld, layout, n);
  if (fail && threadIdx.x == 0) *d_info = info_base + fail;
}

}  // namespace

cudaError_t configure_potf2() {
  const auto attr = cudaFuncAttributeMaxDynamicSharedMemorySize;
  cudaError_t e = cudaFuncSetAttribute(k_potf2_base, attr, (int)P2<kBaseMax>::SMEM);
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(k_potf2_base64, attr, (int)P2<64>::SMEM);
}

cudaError_t launch_potf2(double* A, int64_t ld, int layout, int n, int* d_info, int info_base, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  if (n > kPotf2Max) return cudaErrorInvalidValue;
  if (n <= 64)
    k_potf2_base64<<<1, P2<64>::THREADS, P2<64>::SMEM, st>>>(A, ld, layout, n, d_info, info_base);
  else
    k_potf2_base<<<1, P2<kBaseMax>::THREADS, P2<kBaseMax>::SMEM, st>>>(A, ld, layout, n, d_info, info_base);
  return cudaGetLastError();
}

}  // namespace relapack
