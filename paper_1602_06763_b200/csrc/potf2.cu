// potf2.cu — K1 (base case of the recursion, order n <= 128; the opt-in
// 256-node kernel for 128 < n <= 256): Cholesky of a block held entirely in
// one SM's shared memory (north_star subsystem (2); P:301-307 crossover to the
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
#include <cstdlib>

#include "chol_regs.cuh"
#include "common.cuh"
#include "kernels.h"
#include "trsm_regs.cuh"

namespace relapack {

namespace {

constexpr int kPanel = 8;

#ifndef RELAPACK_PANEL_RB
#define RELAPACK_PANEL_RB 1
#endif
#ifndef RELAPACK_NODE_EARLY_STORE
#define RELAPACK_NODE_EARLY_STORE 0
#endif
#ifndef RELAPACK_POTF2_SPARE
#define RELAPACK_POTF2_SPARE 1
#endif

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
  static constexpr int LDS = NMAX + 4;         // column stride == 4 (mod 16 doubles): every DMMA fragment access at most 2-way bank-conflicted
  static constexpr int RPL = NMAX / 32;        // panel rows per lane
  static constexpr size_t SMEM = sizeof(double) * NMAX * LDS;
};

// Apply the rank-8 update of panel columns [j0, j0+8) to the 8x8 tiles
// (ti, tk), tile index range [t_beg, t_end) (stride tile_step) of the
// lower-triangular tile grid whose first row/column is r0.  Four tiles are in
// flight per warp (DMMA.8x8x4, K = 8 -> 2 dependent DMMA per tile).
template <int LDS>
__device__ __forceinline__ void trail_tiles(double* s, int j0, int r0, int tile_beg, int tile_end, int tile_step,
                                            int g, int t) {
  constexpr int QB = 4;
  for (int base = tile_beg; base < tile_end; base += QB * tile_step) {
    double c0[QB], c1[QB], a[QB][2], b[QB][2];
    int ii[QB], kk[QB];
#pragma unroll
    for (int q = 0; q < QB; ++q) {
      const int tile = base + q * tile_step;
      int ti = (int)((sqrtf(8.0f * (float)tile + 1.0f) - 1.0f) * 0.5f);
      ti += ((ti + 1) * (ti + 2) / 2 <= tile);
      ti -= (ti * (ti + 1) / 2 > tile);
      const int tk = tile - ti * (ti + 1) / 2;
      ii[q] = r0 + 8 * ti;
      kk[q] = r0 + 8 * tk;
      const bool ok = tile < tile_end;
      if (!ok) ii[q] = kk[q] = r0;  // in-range addresses, results discarded
      c0[q] = s[(ii[q] + g) + (kk[q] + 2 * t) * LDS];
      c1[q] = s[(ii[q] + g) + (kk[q] + 2 * t + 1) * LDS];
#pragma unroll
      for (int ks = 0; ks < 2; ++ks) {
        a[q][ks] = -s[(ii[q] + g) + (j0 + 4 * ks + t) * LDS];
        b[q][ks] = s[(kk[q] + g) + (j0 + 4 * ks + t) * LDS];
      }
    }
#pragma unroll
    for (int ks = 0; ks < 2; ++ks)
#pragma unroll
      for (int q = 0; q < QB; ++q) dmma_884(c0[q], c1[q], a[q][ks], b[q][ks]);
#pragma unroll
    for (int q = 0; q < QB; ++q) {
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
template <int NMAX, int LDS, int RB = 0>
__device__ __forceinline__ int factor_panel(double* s, int n, int j0, int lane) {
  // RB: row blocks of 32 above j0 skipped (rows < 32 RB hold nothing of this panel)
  constexpr int R = P2<NMAX>::RPL - RB;
  const int w = min(kPanel, n - j0);
  double x[R][kPanel];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int i = lane + 32 * (r + RB);
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
  double dsh;  // the next pivot, already broadcast
  {
    double own = x[0][0];
#pragma unroll
    for (int r = 1; r < R; ++r)
      if ((j0 >> 5) - RB == r) own = x[r][0];
    dsh = __shfl_sync(0xffffffffu, own, j0 & 31);  // lane (j0 & 31) holds a_{j0,j0}
  }
  // Column c's update of column c+1 is done at once (it feeds the next
  // pivot); its updates of columns c+2.. are deferred into iteration c+1,
  // where they are issued behind that column's rsqrt chain instead of in
  // front of it (in-order issue).
  auto row_val = [&](int c, int row) -> double {  // x[row][c] as held by lane row & 31
    double v = x[0][c];
#pragma unroll
    for (int r = 1; r < R; ++r)
      if ((row >> 5) - RB == r) v = x[r][c];
    return v;
  };
#pragma unroll
  for (int c = 0; c < kPanel; ++c) {
    const int j = j0 + c;
    const double d = dsh;
    dpiv[c] = d;
    const double rinv = rsqrt_nr(d);
    rpiv[c] = rinv;
    if (c >= 1) {
#pragma unroll
      for (int c2 = c + 1; c2 < kPanel; ++c2) {
        const int jj = j0 + c2;
        const double l = __shfl_sync(0xffffffffu, row_val(c - 1, jj), jj & 31);  // l_{jj, j-1}
#pragma unroll
        for (int r = 0; r < R; ++r) x[r][c2] -= x[r][c - 1] * l;
      }
    }
#pragma unroll
    for (int r = 0; r < R; ++r) x[r][c] *= rinv;
    if (c + 1 < kPanel) {
      // the lane holding row j+1 forms the next pivot from its own registers
      const int jn = j + 1;
      const double xn = row_val(c, jn), an = row_val(c + 1, jn);
      dsh = __shfl_sync(0xffffffffu, an - xn * xn, jn & 31);
      const double l = __shfl_sync(0xffffffffu, xn, jn & 31);  // l_{j+1, j}
#pragma unroll
      for (int r = 0; r < R; ++r) x[r][c + 1] -= x[r][c] * l;
    }
  }
  int fail = 0;
#pragma unroll
  for (int c = kPanel - 1; c >= 0; --c)
    if (c < w && !(dpiv[c] >= kMinPivot)) fail = j0 + c + 1;  // d <= 0, -0.0, NaN and flushed (subnormal) d
  // diagonal entries l_jj = sqrt(d), off the critical path
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int i = lane + 32 * (r + RB);
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
template <int NMAX, int LDS, int NW>
__device__ int potf2_smem(double* s, int n, int* fail_flag) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  if (warp == 0) {
    const int f = factor_panel<NMAX, LDS>(s, n, 0, lane);
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
      const int f = (RELAPACK_PANEL_RB && NMAX == 64 && r0 >= 32) ? factor_panel<NMAX, LDS, NMAX == 64 ? 1 : 0>(s, n, r0, lane)
                                                                   : factor_panel<NMAX, LDS>(s, n, r0, lane);
      if (lane == 0 && f) *fail_flag = f;
    } else {
      // tiles of the trailing grid with tk >= 1 (columns >= r0 + 8)
      const int T = (n - r0 + 7) / 8;
      const int ntiles = T * (T + 1) / 2;
      // enumerate tiles with tk >= 1: tile index over the grid starting at r0+8
      if (T > 1) {
        const int T2 = T - 1;
        const int nt2 = T2 * (T2 + 1) / 2;  // lower tiles of the grid rooted at (r0+8, r0+8)
        // with 8 warps, warp 4 shares warp 0's SMSP: it stays idle so the
        // panel chain does not compete for issue slots and the DMMA pipe
        constexpr bool kSpare = NW == 8 && RELAPACK_POTF2_SPARE;
        const int hw = kSpare ? warp - 1 - (warp > 4) : warp - 1;
        if (!(kSpare && warp == 4)) trail_tiles<LDS>(s, j0, r0 + 8, hw, nt2, kSpare ? NW - 2 : NW - 1, g, t);
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

constexpr int kBaseMax = 128;  // the square of the 128-node kernels

__global__ void __launch_bounds__(P2<kBaseMax>::THREADS) k_potf2_base(double* A, int64_t ld, int layout, int n,
                                                                       int* d_info, int info_base, TraceRec* tr) {
  PROBE(0);
  {
    const KState ks = ld_state(d_info);
    if (ks.info != 0) return;
    A = rebase(A, ks.base);
  }
  trace_begin(tr);
  extern __shared__ double s[];
  __shared__ int fail_flag;
  if (threadIdx.x == 0) fail_flag = 0;
  copy_lower<kBaseMax, true>(s, A, ld, layout, n);
  __syncthreads();
  PROBE(1);
  const int fail = potf2_smem<kBaseMax, P2<kBaseMax>::LDS, P2<kBaseMax>::NW>(s, n, &fail_flag);
  pdl_trigger();
  copy_lower<kBaseMax, false>(s, A, ld, layout, n);
  if (fail && threadIdx.x == 0) *untag(d_info) = info_base + fail;
  PROBE(63);
  trace_end(tr);
}

// Same kernel sized for n <= 64 (4 warps, 33 KB): used when the block is small.
__global__ void __launch_bounds__(P2<64>::THREADS) k_potf2_base64(double* A, int64_t ld, int layout, int n,
                                                                  int* d_info, int info_base, TraceRec* tr) {
  PROBE(0);
  {
    const KState ks = ld_state(d_info);
    if (ks.info != 0) return;
    A = rebase(A, ks.base);
  }
  trace_begin(tr);
  extern __shared__ double s[];
  __shared__ int fail_flag;
  if (threadIdx.x == 0) fail_flag = 0;
  copy_lower<64, true>(s, A, ld, layout, n);
  __syncthreads();
  PROBE(1);
  const int fail = potf2_smem<64, P2<64>::LDS, P2<64>::NW>(s, n, &fail_flag);
  PROBE(62);
  pdl_trigger();
  copy_lower<64, false>(s, A, ld, layout, n);
  PROBE(63);
  if (fail && threadIdx.x == 0) *untag(d_info) = info_base + fail;
  trace_end(tr);
}

// Copy the lower-triangle part (i >= j, i < n) of the L-view rectangle rows
// [r0, r0+R) x cols [c0, c0+C) between global and shared memory (stride LDS),
// coalesced along the contiguous index.  MODE 0: synchronous load (zero
// outside), 1: asynchronous load (cp.async; wait with cp.async.wait_all),
// 2: store.
// copy_rect for layout N with ld even and A 16-byte aligned: rows i, i+1 of
// a column are adjacent in global and in shared memory (LDS even, r0 even),
// so each thread moves 16-byte pairs (half the load/store instructions; the
// copies of the 128-node are bound by LSU issue, not bandwidth).
template <int R, int C, int LDS, int THREADS, int MODE>
__device__ __forceinline__ void copy_rect_pairs(double* s, double* __restrict__ A, int64_t ld, int n, int r0,
                                                int c0) {
  constexpr int R2 = R / 2, kTot = R2 * C, kPer = (kTot + THREADS - 1) / THREADS, kBatch = 8;
#pragma unroll 1
  for (int u0 = 0; u0 < kPer; u0 += kBatch) {
    double2 v[kBatch];
#pragma unroll
    for (int u = 0; u < kBatch; ++u) {
      const int e = threadIdx.x + (u0 + u) * THREADS;
      const int i = r0 + 2 * (e % R2), j = c0 + e / R2;
      const bool in = u0 + u < kPer && e < kTot;
      const bool lo0 = in && i < n && i >= j, lo1 = in && i + 1 < n && i + 1 >= j;
      double* g = A + i + (int64_t)j * ld;
      double* sp = s + i + j * LDS;
      if (MODE == 0)
        v[u] = (lo0 && lo1) ? *reinterpret_cast<const double2*>(g) : make_double2(lo0 ? g[0] : 0.0, lo1 ? g[1] : 0.0);
      if (MODE == 1 && in) {
        if (lo0 && lo1) {
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(sp)), "l"(g) : "memory");
        } else {
          if (lo0)
            asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(smem_u32(sp)), "l"(g) : "memory");
          else
            sp[0] = 0.0;
          if (lo1)
            asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(smem_u32(sp + 1)), "l"(g + 1) : "memory");
          else
            sp[1] = 0.0;
        }
      }
      if (MODE == 2 && (lo0 || lo1)) v[u] = *reinterpret_cast<const double2*>(sp);
    }
#pragma unroll
    for (int u = 0; u < kBatch; ++u) {
      const int e = threadIdx.x + (u0 + u) * THREADS;
      const int i = r0 + 2 * (e % R2), j = c0 + e / R2;
      const bool in = u0 + u < kPer && e < kTot;
      const bool lo0 = in && i < n && i >= j, lo1 = in && i + 1 < n && i + 1 >= j;
      double* g = A + i + (int64_t)j * ld;
      if (MODE == 0 && in) *reinterpret_cast<double2*>(s + i + j * LDS) = v[u];
      if (MODE == 2) {
        if (lo0 && lo1) {
          *reinterpret_cast<double2*>(g) = v[u];
        } else {
          if (lo0) g[0] = v[u].x;
          if (lo1) g[1] = v[u].y;
        }
      }
    }
  }
}

// copy_rect for layout T (uplo U) with ld even and A 16-byte aligned: the L
// view's (i, j) and (i, j + 1) are adjacent in global memory, so a warp moves
// an 8-row x 8-column patch as 16-byte global accesses (4 column pairs x 8
// rows) and 8-byte shared-memory accesses at i + j*LDS, which with LDS = 4
// mod 16 hit every bank pair exactly twice (the element-wise copy runs 32
// consecutive columns per warp: 8-way conflicted).
template <int R, int C, int LDS, int THREADS, int MODE>
__device__ __forceinline__ void copy_rect_pairsT(double* s, double* __restrict__ A, int64_t ld, int n, int r0,
                                                 int c0) {
  static_assert(R % 8 == 0 && C % 8 == 0, "8x8 patches");
  constexpr int NW = THREADS / 32, PATCHES = (R / 8) * (C / 8), kPer = (PATCHES + NW - 1) / NW;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int jp = lane & 3, il = lane >> 2;
  constexpr int kBatch = 4;
#pragma unroll 1
  for (int u0 = 0; u0 < kPer; u0 += kBatch) {
    double2 v[kBatch];
#pragma unroll
    for (int u = 0; u < kBatch; ++u) {
      const int p = warp + (u0 + u) * NW;
      const bool in = u0 + u < kPer && p < PATCHES;
      const int i = r0 + 8 * (p / (C / 8)) + il, j = c0 + 8 * (p % (C / 8)) + 2 * jp;
      const bool lo0 = in && i < n && i >= j, lo1 = in && i < n && i >= j + 1;
      double* g = A + j + (int64_t)i * ld;
      if (MODE == 0)
        v[u] = (lo0 && lo1) ? *reinterpret_cast<const double2*>(g) : make_double2(lo0 ? g[0] : 0.0, lo1 ? g[1] : 0.0);
      if (MODE == 1 && in) {
        double* sp = s + i + j * LDS;
        if (lo0)
          asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(smem_u32(sp)), "l"(g) : "memory");
        else
          sp[0] = 0.0;
        if (lo1)
          asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(smem_u32(sp + LDS)), "l"(g + 1) : "memory");
        else
          sp[LDS] = 0.0;
      }
      if (MODE == 2 && (lo0 || lo1)) v[u] = make_double2(s[i + j * LDS], s[i + (j + 1) * LDS]);
    }
#pragma unroll
    for (int u = 0; u < kBatch; ++u) {
      const int p = warp + (u0 + u) * NW;
      const bool in = u0 + u < kPer && p < PATCHES;
      const int i = r0 + 8 * (p / (C / 8)) + il, j = c0 + 8 * (p % (C / 8)) + 2 * jp;
      const bool lo0 = in && i < n && i >= j, lo1 = in && i < n && i >= j + 1;
      double* g = A + j + (int64_t)i * ld;
      if (MODE == 0 && in) {
        s[i + j * LDS] = v[u].x;
        s[i + (j + 1) * LDS] = v[u].y;
      }
      if (MODE == 2) {
        if (lo0 && lo1) {
          *reinterpret_cast<double2*>(g) = v[u];
        } else {
          if (lo0) g[0] = v[u].x;
          if (lo1) g[1] = v[u].y;
        }
      }
    }
  }
}

template <int R, int C, int LDS, int THREADS, int MODE>
__device__ __forceinline__ void copy_rect(double* s, double* __restrict__ A, int64_t ld, int layout, int n, int r0,
                                          int c0, bool pairs) {
  if (pairs && layout == kLayoutN && (ld & 1) == 0 && (reinterpret_cast<uintptr_t>(A) & 15) == 0) {
    copy_rect_pairs<R, C, LDS, THREADS, MODE>(s, A, ld, n, r0, c0);
    return;
  }
  if (pairs && layout == kLayoutT && (ld & 1) == 0 && (reinterpret_cast<uintptr_t>(A) & 15) == 0) {
    copy_rect_pairsT<R, C, LDS, THREADS, MODE>(s, A, ld, n, r0, c0);
    return;
  }
  constexpr int kTot = R * C, kPer = (kTot + THREADS - 1) / THREADS, kBatch = 16;
#pragma unroll 1
  for (int u0 = 0; u0 < kPer; u0 += kBatch) {
    double v[kBatch];
#pragma unroll
    for (int u = 0; u < kBatch; ++u) {
      const int e = threadIdx.x + (u0 + u) * THREADS;
      const int a = layout == kLayoutN ? e % R : e % C, b = layout == kLayoutN ? e / R : e / C;
      const int i = r0 + (layout == kLayoutN ? a : b), j = c0 + (layout == kLayoutN ? b : a);
      const bool in = u0 + u < kPer && e < kTot;
      const bool ok = in && i < n && i >= j;
      if (MODE == 0) v[u] = ok ? A[lv_off(layout, i, j, ld)] : 0.0;
      if (MODE == 1 && in) {
        if (ok)
          asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(smem_u32(s + i + j * LDS)),
                       "l"(A + lv_off(layout, i, j, ld))
                       : "memory");
        else
          s[i + j * LDS] = 0.0;
      }
      if (MODE == 2 && ok) v[u] = s[i + j * LDS];
    }
#pragma unroll
    for (int u = 0; u < kBatch; ++u) {
      const int e = threadIdx.x + (u0 + u) * THREADS;
      const int a = layout == kLayoutN ? e % R : e % C, b = layout == kLayoutN ? e / R : e / C;
      const int i = r0 + (layout == kLayoutN ? a : b), j = c0 + (layout == kLayoutN ? b : a);
      const bool in = u0 + u < kPer && e < kTot;
      const bool ok = in && i < n && i >= j;
      if (MODE == 0 && in) s[i + j * LDS] = v[u];
      if (MODE == 2 && ok) A[lv_off(layout, i, j, ld)] = v[u];
    }
  }
}

// ---- K1' base case for 64 < n <= 128: the recursion's 128-node in ONE CTA.
// The block is split at 64 exactly as a recursion node: factor
// A11 (potf2_smem), A21 := A21 L11^{-T} (substitution, quad shuffles + DMMA
// between 8-column sub-blocks), A22 -= A21 A21^T (DMMA, lower tiles), factor
// A22 — four phases in shared memory instead of four kernel launches.
constexpr int kN1 = 64;

// A21 (rows kN1 .. kN1+n2) := A21 L11^{-T}; warp w owns rows kN1 + 8w .. +7.
template <int LDS>
__device__ __forceinline__ void trsm_in_smem(double* s, const double* rinv, int n2) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, tq = lane & 3;
  if (8 * warp >= n2) return;
  double* X = s + kN1 + 8 * warp;  // X(r, c) = X[r + c * LDS]
  double xs[8][2];
#pragma unroll
  for (int sb = 0; sb < 8; ++sb) {
    xs[sb][0] = X[g + (8 * sb + 2 * tq) * LDS];
    xs[sb][1] = X[g + (8 * sb + 2 * tq + 1) * LDS];
  }
#pragma unroll
  for (int sb = 0; sb < 8; ++sb) {
    double l0[8], l1[8], rc[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const int col = 8 * sb + c, r0 = 8 * sb + 2 * tq;
      // the upper half of the diagonal tiles holds don't-care values: mask
      l0[c] = (2 * tq > c) ? s[r0 + col * LDS] : 0.0;
      l1[c] = (2 * tq + 1 > c) ? s[r0 + 1 + col * LDS] : 0.0;
      rc[c] = rinv[col];
    }
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const double xj = __shfl_sync(0xffffffffu, (c & 1) ? xs[sb][1] : xs[sb][0], (lane & ~3) | (c >> 1)) * rc[c];
      xs[sb][0] -= xj * l0[c];
      xs[sb][1] -= xj * l1[c];
      if (tq == (c >> 1)) {
        if (c & 1)
          xs[sb][1] = xj;
        else
          xs[sb][0] = xj;
      }
    }
#pragma unroll
    for (int ks = 0; ks < 2; ++ks) {
      const int src = (lane & ~3) | (2 * ks + (tq >> 1));
      const double e0 = __shfl_sync(0xffffffffu, xs[sb][0], src);
      const double e1 = __shfl_sync(0xffffffffu, xs[sb][1], src);
      const double a = -((tq & 1) ? e1 : e0);  // -X_sb[g][4ks + tq]
#pragma unroll
      for (int s2 = sb + 1; s2 < 8; ++s2)
        dmma_884(xs[s2][0], xs[s2][1], a, s[(8 * s2 + g) + (8 * sb + 4 * ks + tq) * LDS]);
    }
  }
#pragma unroll
  for (int sb = 0; sb < 8; ++sb) {
    X[g + (8 * sb + 2 * tq) * LDS] = xs[sb][0];
    X[g + (8 * sb + 2 * tq + 1) * LDS] = xs[sb][1];
  }
}

// A22 -= A21 A21^T on the lower 8x8 tiles of the n2 x n2 block (K = 64); each
// warp keeps all its tiles' DMMA chains in flight.
template <int LDS, int NW>
__device__ __forceinline__ void syrk_in_smem(double* s, int n2) {
  constexpr int kMaxPer = (36 + NW - 1) / NW;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, tq = lane & 3;
  const int T = (n2 + 7) / 8, ntiles = T * (T + 1) / 2;
  double* L21 = s + kN1;             // L21(r, k) = L21[r + k * LDS]
  double* C = s + kN1 + kN1 * LDS;   // A22(r, c) = C[r + c * LDS]
  int ti[kMaxPer], tk[kMaxPer];
  double acc[kMaxPer][2];
#pragma unroll
  for (int q = 0; q < kMaxPer; ++q) {
    const int x = warp + q * NW;
    int r = 0;
    while ((r + 1) * (r + 2) / 2 <= x) ++r;
    ti[q] = r;
    tk[q] = x - r * (r + 1) / 2;
    const bool ok = x < ntiles;
    acc[q][0] = ok ? C[(8 * ti[q] + g) + (8 * tk[q] + 2 * tq) * LDS] : 0.0;
    acc[q][1] = ok ? C[(8 * ti[q] + g) + (8 * tk[q] + 2 * tq + 1) * LDS] : 0.0;
  }
#pragma unroll 4
  for (int k0 = 0; k0 < kN1; k0 += 4) {
#pragma unroll
    for (int q = 0; q < kMaxPer; ++q) {
      if (warp + q * NW < ntiles) {
        const double a = -L21[(8 * ti[q] + g) + (k0 + tq) * LDS];
        const double b = L21[(8 * tk[q] + g) + (k0 + tq) * LDS];
        dmma_884(acc[q][0], acc[q][1], a, b);
      }
    }
  }
#pragma unroll
  for (int q = 0; q < kMaxPer; ++q) {
    if (warp + q * NW < ntiles) {
      C[(8 * ti[q] + g) + (8 * tk[q] + 2 * tq) * LDS] = acc[q][0];
      C[(8 * ti[q] + g) + (8 * tk[q] + 2 * tq + 1) * LDS] = acc[q][1];
    }
  }
}

// The 128-node's four phases on the block already in shared memory (A11's
// 64 x 64 block loaded, the rest possibly still in flight by cp.async): factor
// A11, A21 := A21 L11^{-T}, A22 -= A21 A21^T, factor A22.  n <= 128; for
// n <= 64 only the first factorization runs.  Returns 0 or the 1-based local
// column of the first failed pivot (the block then holds the factor up to it).
template <int LDS, int NW>
__device__ __forceinline__ int node128_factor(double* s, int n, int* fail_flag, double* rinv) {
  int fail = potf2_smem<kN1, LDS, NW>(s, n < kN1 ? n : kN1, fail_flag);
  PROBE(52);
  if (fail == 0 && n > kN1) {
    const int n2 = n - kN1;
    if (threadIdx.x < kN1) rinv[threadIdx.x] = 1.0 / s[threadIdx.x * (LDS + 1)];
    asm volatile("cp.async.wait_all;\n" ::: "memory");
    __syncthreads();
    trsm_in_smem<LDS>(s, rinv, n2);
    __syncthreads();
    PROBE(53);
    syrk_in_smem<LDS, NW>(s, n2);
    __syncthreads();
    PROBE(54);
    fail = potf2_smem<kN1, LDS, NW>(s + kN1 + kN1 * LDS, n2, fail_flag);
    if (fail) fail += kN1;
  } else {
    asm volatile("cp.async.wait_all;\n" ::: "memory");
  }
  PROBE(55);
  return fail;
}

// Store the factored 128-node (the lower triangle of its n x n block) from
// shared memory; after a failure in the first 64 columns only A11's block.
template <int LDS, int TH>
__device__ __forceinline__ void node128_store(double* s, double* A, int64_t ld, int layout, int n, int fail,
                                              bool pairs) {
  if (fail == 0 || fail > kN1) {
    copy_rect<kBaseMax, kN1, LDS, TH, 2>(s, A, ld, layout, n, 0, 0, pairs);
    copy_rect<kBaseMax - kN1, kBaseMax - kN1, LDS, TH, 2>(s, A, ld, layout, n, kN1, kN1, pairs);
  } else {
    copy_rect<kN1, kN1, LDS, TH, 2>(s, A, ld, layout, n, 0, 0, pairs);
  }
}

__global__ void __launch_bounds__(P2<kBaseMax>::THREADS) k_potf2_node128(double* A, int64_t ld, int layout, int n,
                                                                          int* d_info, int info_base, TraceRec* tr) {
  const bool pairs = (layout & 0x100) != 0;  // 16-byte copies (host knob RELAPACK_COPY_PAIRS)
  layout &= 0xff;
  constexpr int LDS = P2<kBaseMax>::LDS, NW = P2<kBaseMax>::NW;
  PROBE(50);
  {
    const KState ks = ld_state(d_info);
    if (ks.info != 0) return;
    A = rebase(A, ks.base);
  }
  trace_begin(tr);
  extern __shared__ double s[];
  __shared__ int fail_flag;
  __shared__ double rinv[kN1];
  if (threadIdx.x == 0) fail_flag = 0;
  constexpr int TH = P2<kBaseMax>::THREADS;
  // A11 now; A21 and A22 stream in (cp.async) while A11 is factored
  copy_rect<kN1, kN1, LDS, TH, 0>(s, A, ld, layout, n, 0, 0, pairs);
  copy_rect<kBaseMax - kN1, kBaseMax, LDS, TH, 1>(s, A, ld, layout, n, kN1, 0, pairs);
  __syncthreads();
  PROBE(51);
  const int fail = node128_factor<LDS, NW>(s, n, &fail_flag, rinv);
  pdl_trigger();
  node128_store<LDS, TH>(s, A, ld, layout, n, fail, pairs);
  PROBE(56);
  if (fail && threadIdx.x == 0) *untag(d_info) = info_base + fail;
  trace_end(tr);
}

// ---- K1'' base case for 128 < n <= 256: the recursion's 256-node in ONE CTA
// (P:286-295 split at n1 = 128): the 128-node phases on A11, then
//   A21 := A21 L11^{-T}   rows in registers (RG = 2 groups of 8 rows per
//                          warp, trsm_regs.cuh), L11 read in place from the
//                          node's shared-memory square;
//   A22 -= A21 A21^T      DMMA on the lower 8x8 tiles, K = 128 in two halves
//                          of 64 staged through shared memory (warp w owns
//                          tile rows w and 15 - w: 17 tiles each), while A22
//                          streams into the square (cp.async);
// then the 128-node phases on A22.  One launch instead of the four of the
// plan's 256-node (node-128, TRSM, SYRK, node-128): no launch gaps and no
// global round trip of L11 / L21 between them on the base-case chain.
constexpr int kN2 = 128;             // the 256-node's split
constexpr int kHLd = 68;             // L21 half row stride (== 4 mod 16: conflict-free fragments)

struct Node256 {
  static constexpr int LDS = P2<kBaseMax>::LDS, NW = P2<kBaseMax>::NW, TH = P2<kBaseMax>::THREADS;
  static constexpr size_t SQ = sizeof(double) * (size_t)kBaseMax * LDS;         // the 128 x 128 square
  static constexpr size_t HALF = sizeof(double) * (size_t)kN2 * kHLd;          // L21[:, half] staging
  static constexpr size_t SMEM = SQ + HALF;                                     // 204.8 KB
};

__global__ void __launch_bounds__(Node256::TH, 1) k_potf2_node256(double* A, int64_t ld, int layout, int n,
                                                                   int* d_info, int info_base, TraceRec* tr) {
  const bool pairs = (layout & 0x100) != 0;
  layout &= 0xff;
  constexpr int LDS = Node256::LDS, NW = Node256::NW, TH = Node256::TH;
  PROBE(50);
  {
    const KState ks = ld_state(d_info);
    if (ks.info != 0) return;
    A = rebase(A, ks.base);
  }
  trace_begin(tr);
  extern __shared__ double s[];  // the 128 x 128 square (A11, then L21 rows for nothing, then A22)
  double* H = s + kBaseMax * LDS; // L21(r, k), k in one 64-column half: H[r * kHLd + k]
  __shared__ int fail_flag;
  __shared__ double rinv[kN2];
  if (threadIdx.x == 0) fail_flag = 0;
  const int n2 = n - kN2;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, tq = lane & 3;
  double* const A21 = A + lv_off(layout, kN2, 0, ld);
  double* const A22 = A + lv_off(layout, kN2, kN2, ld);
  // A21 and A22 towards L2 now (their first reads come after A11's factorization)
  {
    constexpr int kLine = 16;  // doubles per 128-byte line
    for (int e = threadIdx.x; e < 2 * kN2 * (kN2 / kLine); e += TH) {
      const int blk = e / (kN2 * (kN2 / kLine)), x = e % (kN2 * (kN2 / kLine));
      const int slow = x / (kN2 / kLine), fast = (x % (kN2 / kLine)) * kLine;  // fast: contiguous index
      const int i = layout == kLayoutN ? fast : slow, j = layout == kLayoutN ? slow : fast;
      if (i < n2 && (blk == 0 || j <= i + kLine))
        asm volatile("prefetch.global.L2 [%0];" ::"l"((blk ? A22 : A21) + lv_off(layout, i, j, ld)));
    }
  }
  copy_rect<kN1, kN1, LDS, TH, 0>(s, A, ld, layout, kN2, 0, 0, pairs);
  copy_rect<kBaseMax - kN1, kBaseMax, LDS, TH, 1>(s, A, ld, layout, kN2, kN1, 0, pairs);
  __syncthreads();
  PROBE(51);
  // one call site of the 128-node phases (code size): half 0 factors A11,
  // half 1 factors A22 after the TRSM and the SYRK below
  for (int half = 0;; ++half) {
    double* const Ah = half ? A22 : A;
    const int nh = half ? n2 : kN2;
    const int fail = node128_factor<LDS, NW>(s, nh, &fail_flag, rinv);
    if (half == 1 || fail) {
      pdl_trigger();
      node128_store<LDS, TH>(s, Ah, ld, layout, nh, fail, pairs);
      if (fail && threadIdx.x == 0) *untag(d_info) = info_base + half * kN2 + fail;
      break;
    }
  PROBE(62);
  // L11 is final: store it (the values leave shared memory before the next
  // barrier) and form 1 / L_jj of all 128 columns
  node128_store<LDS, TH>(s, A, ld, layout, kN2, 0, pairs);
  if (threadIdx.x < kN2) rinv[threadIdx.x] = 1.0 / s[threadIdx.x * (LDS + 1)];
  // this warp's 16 rows of A21 (two groups of 8) as DMMA accumulator tiles
  constexpr int RG = 2, NT = 16;
  double xs[RG][NT][2];
  const int row_base = warp * 8 * RG;
  const bool tpairs = layout == kLayoutT && (ld & 1) == 0 && (reinterpret_cast<uintptr_t>(A21) & 15) == 0;
#pragma unroll
  for (int r = 0; r < RG; ++r)
#pragma unroll
    for (int sb = 0; sb < NT; ++sb) {
      const int row = row_base + 8 * r + g, col = 8 * sb + 2 * tq;
      if (tpairs && row < n2) {
        const double2 v = *reinterpret_cast<const double2*>(A21 + lv_off(kLayoutT, row, col, ld));
        xs[r][sb][0] = v.x;
        xs[r][sb][1] = v.y;
      } else {
#pragma unroll
        for (int q = 0; q < 2; ++q) xs[r][sb][q] = row < n2 ? A21[lv_off(layout, row, col + q, ld)] : 0.0;
      }
    }
  __syncthreads();
  PROBE(57);
  // A21 := A21 L11^{-T}, L11(r, c) = s[r + c * LDS]
  solve_chunk_regs<RG, 0, NT, 1, LDS>(xs, s, rinv, lane, g, tq);
  update_chunk1_regs<RG, NT, 1, LDS>(xs, s + kN1, g, tq);
  solve_chunk_regs<RG, 1, NT, 1, LDS>(xs, s + kN1 + kN1 * LDS, rinv + kN1, lane, g, tq);
  PROBE(58);
  // L21 to global
#pragma unroll
  for (int r = 0; r < RG; ++r)
#pragma unroll
    for (int sb = 0; sb < NT; ++sb) {
      const int row = row_base + 8 * r + g, col = 8 * sb + 2 * tq;
      if (tpairs && row < n2) {
        *reinterpret_cast<double2*>(A21 + lv_off(kLayoutT, row, col, ld)) = make_double2(xs[r][sb][0], xs[r][sb][1]);
      } else {
#pragma unroll
        for (int q = 0; q < 2; ++q)
          if (row < n2) A21[lv_off(layout, row, col + q, ld)] = xs[r][sb][q];
      }
    }
  __syncthreads();  // every warp is done with L11 in the square: A22 streams in
  copy_rect<kN1, kN1, LDS, TH, 1>(s, A22, ld, layout, n2, 0, 0, pairs);
  copy_rect<kBaseMax - kN1, kBaseMax, LDS, TH, 1>(s, A22, ld, layout, n2, kN1, 0, pairs);
  // A22 -= L21 L21^T: warp w owns tile rows ra = w and rb = 15 - w (17 tiles:
  // slot j <= ra is tile (ra, j), slot j > ra is tile (rb, j - ra - 1))
  const int ra = warp, rb = 15 - warp;
  double acc[17][2];
  int boff[17];
#pragma unroll
  for (int j = 0; j < 17; ++j) {
    acc[j][0] = acc[j][1] = 0.0;
    boff[j] = (8 * (j <= ra ? j : j - ra - 1) + g) * kHLd + tq;
  }
  const int aoff = (8 * ra + g) * kHLd + tq, boff_b = (8 * rb + g) * kHLd + tq;
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    // stage L21[:, 64h .. 64h + 63]
#pragma unroll
    for (int r = 0; r < RG; ++r)
#pragma unroll
      for (int sb = 0; sb < 8; ++sb)
#pragma unroll
        for (int q = 0; q < 2; ++q) H[(row_base + 8 * r + g) * kHLd + 8 * sb + 2 * tq + q] = xs[r][8 * h + sb][q];
    __syncthreads();
#pragma unroll 4
    for (int k0 = 0; k0 < kN1; k0 += 4) {
      const double a0 = -H[aoff + k0], a1 = -H[boff_b + k0];
#pragma unroll
      for (int j = 0; j < 17; ++j) dmma_884(acc[j][0], acc[j][1], j <= ra ? a0 : a1, H[boff[j] + k0]);
    }
    __syncthreads();  // H free for the next half
  }
  PROBE(59);
  asm volatile("cp.async.wait_all;\n" ::: "memory");
  __syncthreads();
#pragma unroll
  for (int j = 0; j < 17; ++j) {
    const int ti = j <= ra ? ra : rb, tk = j <= ra ? j : j - ra - 1;
#pragma unroll
    for (int q = 0; q < 2; ++q) s[(8 * ti + g) + (8 * tk + 2 * tq + q) * LDS] += acc[j][q];
  }
  __syncthreads();
  PROBE(60);
  }
  PROBE(61);
  trace_end(tr);
}

// One warp, the whole block in registers (chol_regs.cuh): n <= 8 TN.  The
// block is read straight from global memory into the DMMA tile layout
// (identity beyond n, nothing above the diagonal is read) and written back the
// same way.
template <int TN>
__global__ void __launch_bounds__(32, 1) k_potf2_reg(double* A, int64_t ld, int layout, int n, int* d_info,
                                                      int info_base, TraceRec* tr) {
  using T = RegTri<TN>;
  {
    const KState ks = ld_state(d_info);
    if (ks.info != 0) return;
    A = rebase(A, ks.base);
  }
  trace_begin(tr);
  const int lane = threadIdx.x, g = lane >> 2, t = lane & 3;
  double v[T::NT][2];
#pragma unroll
  for (int i = 0; i < TN; ++i)
#pragma unroll
    for (int k = 0; k <= i; ++k)
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const int r = 8 * i + g, c = 8 * k + 2 * t + q;
        v[T::id(i, k)][q] = (r < n && c < n && r >= c) ? A[lv_off(layout, r, c, ld)] : (r == c ? 1.0 : 0.0);
      }
  const int fail = reg_potrf<TN>(v, lane);
  pdl_trigger();
#pragma unroll
  for (int i = 0; i < TN; ++i)
#pragma unroll
    for (int k = 0; k <= i; ++k)
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const int r = 8 * i + g, c = 8 * k + 2 * t + q;
        if (r < n && c < n && r >= c) A[lv_off(layout, r, c, ld)] = v[T::id(i, k)][q];
      }
  if (fail && fail <= n && lane == 0) *untag(d_info) = info_base + fail;
  trace_end(tr);
}

// Register kernel for n <= 32 (measured faster: 6.2 vs 10.3 us at n = 32),
// the shared-memory lookahead kernel for 32 < n <= 64 (15.9 vs 16.4 us);
// RELAPACK_POTF2=smem|reg forces one of them (A/B measurements).
static int potf2_regs_max() {
  static const int r = [] {
    const char* v = getenv("RELAPACK_POTF2");
    if (v && v[0] == 's') return 0;
    if (v && v[0] == 'r') return 64;
    return 32;
  }();
  return r;
}
static bool potf2_use_regs(int n) { return n <= potf2_regs_max(); }

// 64 < n <= 128: the in-CTA recursion node (default) or the flat right-looking
// kernel (RELAPACK_NODE128=0).
// 128-node copies as 16-byte pairs for uplo L (RELAPACK_COPY_PAIRS=0: 8-byte)
static bool copy_pairs() {
  static const bool r = [] {
    const char* v = getenv("RELAPACK_COPY_PAIRS");
    return !(v && v[0] == '0');
  }();
  return r;
}

// Shared memory requested per node-128 launch: RELAPACK_NODE_EXCLUSIVE=1 asks
// for (nearly) the whole SM so no other CTA (an update tile) shares it.
static int node128_smem() {
  static const int v = [] {
    const char* e = getenv("RELAPACK_NODE_EXCLUSIVE");
    return (e && e[0] == '0') ? (int)P2<kBaseMax>::SMEM : 220 * 1024;
  }();
  return v;
}

static bool potf2_node128() {
  static const bool r = [] {
    const char* v = getenv("RELAPACK_NODE128");
    return !(v && v[0] == '0');
  }();
  return r;
}

}  // namespace

cudaError_t configure_potf2() {
  const auto attr = cudaFuncAttributeMaxDynamicSharedMemorySize;
  cudaError_t e = cudaFuncSetAttribute(k_potf2_base, attr, (int)P2<kBaseMax>::SMEM);
  if (e != cudaSuccess) return e;
  if ((e = cudaFuncSetAttribute(k_potf2_node128, attr, node128_smem())) != cudaSuccess) return e;
  if ((e = cudaFuncSetAttribute(k_potf2_node256, attr, (int)Node256::SMEM)) != cudaSuccess) return e;
  return cudaFuncSetAttribute(k_potf2_base64, attr, (int)P2<64>::SMEM);
}

cudaError_t launch_potf2(double* A, int64_t ld, int layout, int n, int* d_info, int info_base, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  if (n > kPotf2Max) return cudaErrorInvalidValue;
  if (n > kBaseMax) {
    k_potf2_node256<<<1, Node256::TH, Node256::SMEM, st>>>(A, ld, layout | (copy_pairs() ? 0x100 : 0), n, d_info,
                                                            info_base, g_launch_trace);
  } else if (potf2_use_regs(n)) {
    switch ((n + 7) / 8) {
      case 1: k_potf2_reg<1><<<1, 32, 0, st>>>(A, ld, layout, n, d_info, info_base, g_launch_trace); break;
      case 2: k_potf2_reg<2><<<1, 32, 0, st>>>(A, ld, layout, n, d_info, info_base, g_launch_trace); break;
      case 3: k_potf2_reg<3><<<1, 32, 0, st>>>(A, ld, layout, n, d_info, info_base, g_launch_trace); break;
      case 4: k_potf2_reg<4><<<1, 32, 0, st>>>(A, ld, layout, n, d_info, info_base, g_launch_trace); break;
      case 5: k_potf2_reg<5><<<1, 32, 0, st>>>(A, ld, layout, n, d_info, info_base, g_launch_trace); break;
      case 6: k_potf2_reg<6><<<1, 32, 0, st>>>(A, ld, layout, n, d_info, info_base, g_launch_trace); break;
      case 7: k_potf2_reg<7><<<1, 32, 0, st>>>(A, ld, layout, n, d_info, info_base, g_launch_trace); break;
      default: k_potf2_reg<8><<<1, 32, 0, st>>>(A, ld, layout, n, d_info, info_base, g_launch_trace); break;
    }
  } else if (n <= 64)
    k_potf2_base64<<<1, P2<64>::THREADS, P2<64>::SMEM, st>>>(A, ld, layout, n, d_info, info_base, g_launch_trace);
  else if (potf2_node128())
    k_potf2_node128<<<1, P2<kBaseMax>::THREADS, node128_smem(), st>>>(A, ld, layout | (copy_pairs() ? 0x100 : 0), n,
                                                                          d_info, info_base, g_launch_trace);
  else
    k_potf2_base<<<1, P2<kBaseMax>::THREADS, P2<kBaseMax>::SMEM, st>>>(A, ld, layout, n, d_info, info_base, g_launch_trace);
  return cudaGetLastError();
}

}  // namespace relapack
