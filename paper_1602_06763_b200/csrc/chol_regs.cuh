// chol_regs.cuh — register-resident Cholesky of a small lower triangle by ONE
// warp (base case of the recursion, north_star subsystem (2); SPEC potf2
// post-condition S:219-227; "the unblocked kernel ... within the
// processor's L1 cache" -> on the GPU: within one warp's registers).
//
// The NMAX x NMAX block (NMAX = 8 TN <= 64) is held as its lower-triangular
// 8x8 tiles in the DMMA accumulator layout: lane (g = lane/4, t = lane%4)
// holds, for every tile (i, k) with k <= i,
//     v[id(i,k)][q] = L(8i + g, 8k + 2t + q),   q = 0, 1
// (the upper half of the diagonal tiles is don't-care and never stored).
// Right-looking by 8-column panels; per column j of panel p:
//     d = a_jj (shuffle from its owner lane); stop-flag if !(d > 0)
//     r = 1/sqrt(d) (rsqrt.approx + 2 Newton steps), l_jj = sqrt(d) (fma-exact)
//     l_ij = a_ij * r                             (panel rows i > j)
//     a_ik -= l_ij * l_kj                         (panel columns k > j)
// with the column values broadcast inside each lane quad; the rank-8 update of
// the trailing tiles runs on the FP64 tensor cores (mma.sync m8n8k4 f64 ->
// DMMA.8x8x4), the panel tiles' A/B fragments formed by quad shuffles.  The
// per-column dependent chain is shuffle -> rsqrt -> multiply -> shuffle ->
// fma; there is no shared memory and no barrier.
#pragma once
#include "common.cuh"

namespace relapack {

template <int TN>
struct RegTri {
  static constexpr int NT = TN * (TN + 1) / 2;
  static __host__ __device__ constexpr int id(int i, int k) { return i * (i + 1) / 2 + k; }
};

// A/B fragment (k-step ks) of an 8x8 tile held in the accumulator layout:
// returns T(g, 4ks + t) for lane (g, t).
__device__ __forceinline__ double tile_frag(double x0, double x1, int ks, int g, int t) {
  const int src = 4 * g + 2 * ks + (t >> 1);
  const double e0 = __shfl_sync(0xffffffffu, x0, src);
  const double e1 = __shfl_sync(0xffffffffu, x1, src);
  return (t & 1) ? e1 : e0;
}

// Deferred work of panel p, job range [lo, hi) (compile-time after unrolling):
// jobs 0 .. nX-1: L_ip = A_ip W^T and its fragments for i = p+2 .. TN-1;
// then one job per trailing tile (i, k), k >= p+1, except (p+1, p+1).
template <int TN>
__device__ __forceinline__ void panel_jobs(double (&v)[RegTri<TN>::NT][2], double (&fr)[TN][2], const double (&wb)[2],
                                           int p, int lo, int hi, int g, int t) {
  using T = RegTri<TN>;
#pragma unroll
  for (int i = p + 2; i < TN; ++i) {
    const int job = i - (p + 2);
    if (job < lo || job >= hi) continue;
    const double a0 = tile_frag(v[T::id(i, p)][0], v[T::id(i, p)][1], 0, g, t);
    const double a1 = tile_frag(v[T::id(i, p)][0], v[T::id(i, p)][1], 1, g, t);
    double x0 = 0.0, x1 = 0.0, y0 = 0.0, y1 = 0.0;
    dmma_884(x0, x1, a0, wb[0]);
    dmma_884(y0, y1, a1, wb[1]);
    v[T::id(i, p)][0] = x0 + y0;
    v[T::id(i, p)][1] = x1 + y1;
    fr[i][0] = tile_frag(v[T::id(i, p)][0], v[T::id(i, p)][1], 0, g, t);
    fr[i][1] = tile_frag(v[T::id(i, p)][0], v[T::id(i, p)][1], 1, g, t);
  }
#pragma unroll
  for (int k = p + 1; k < TN; ++k)
#pragma unroll
    for (int i = k; i < TN; ++i) {
      // tiles of the trailing grid in column order, (p+1, p+1) excluded
      const int q = (TN - p - 2) + (k - p - 1) * (TN - p - 1) - (k - p - 1) * (k - p - 2) / 2 + (i - k) - 1;
      if (!(i == p + 1 && k == p + 1) && q >= lo && q < hi) {
        dmma_884(v[T::id(i, k)][0], v[T::id(i, k)][1], -fr[i][0], fr[k][0]);
        dmma_884(v[T::id(i, k)][0], v[T::id(i, k)][1], -fr[i][1], fr[k][1]);
      }
    }
}

template <int TN>
__host__ __device__ constexpr int panel_njobs(int p) {
  return p + 2 > TN ? 0 : (TN - p - 2) + (TN - p - 1) * (TN - p) / 2 - 1;
}

// Factor in place.  Returns 0 or the 1-based first column whose pivot failed
// (!(d > 0): d <= 0, -0.0 or NaN); the values after a failure are unspecified.
//
// Panel p (8 columns):
//  (1) the diagonal tile D is factored column by column, with an identity tile
//      E carried along as if it were a tile below D: the unblocked elimination
//      of [D; I] leaves E = I L_pp^{-T} = W^T (W = L_pp^{-1});
//  (2) every tile below becomes L_ip = A_ip W^T (DMMA), no per-column work
//      below the diagonal;
//  (3) the rank-8 trailing update on DMMA.
// Only what the next panel's chain needs is done at once (L_{p+1,p} and the
// update of tile (p+1, p+1), each as two independent DMMAs summed); the rest
// of (2) and (3) is interleaved with the next panel's column chain, so the
// in-order issue of a long DMMA block never stalls the chain.
// Columns stay unscaled until the panel ends; a column value enters an update
// as a_ic * r_c, the same product that is stored.  Finished columns get a
// zero multiplier.
#ifndef RELAPACK_DEFER_JOBS
#define RELAPACK_DEFER_JOBS 0
#endif
constexpr bool kDeferJobs = RELAPACK_DEFER_JOBS != 0;

template <int TN>
__device__ __forceinline__ int reg_potrf(double (&v)[RegTri<TN>::NT][2], int lane) {
  using T = RegTri<TN>;
  const int g = lane >> 2, t = lane & 3;
  // failed pivots as a bit mask (branch-free: every shuffle stays in converged code)
  uint64_t bad = 0;
  double fr[TN][2];  // fragments of the previous panel's tiles below the diagonal
  double wb[2] = {0.0, 0.0};
#pragma unroll
  for (int p = 0; p < TN; ++p) {
    const int D = T::id(p, p);
    const bool below = p + 1 < TN;
    double E[2] = {g == 2 * t ? 1.0 : 0.0, g == 2 * t + 1 ? 1.0 : 0.0};
    double dv[8], rv[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const int e = c & 1, tc = c >> 1;
      const int quad_src = (lane & ~3) | tc;
      const double d = __shfl_sync(0xffffffffu, v[D][e], 4 * c + tc);
      double a0 = 0.0, a1 = 0.0, xD = 0.0, xE = 0.0;
      if (c < 7) {
        a0 = __shfl_sync(0xffffffffu, v[D][e], 8 * t + tc);      // a(8p + 2t,     8p + c)
        a1 = __shfl_sync(0xffffffffu, v[D][e], 8 * t + 4 + tc);  // a(8p + 2t + 1, 8p + c)
        xD = __shfl_sync(0xffffffffu, v[D][e], quad_src);        // a(8p + g,      8p + c)
        if (below) xE = __shfl_sync(0xffffffffu, E[e], quad_src);
      }
      bad |= (uint64_t)(!(d > 0.0)) << (8 * p + c);
      const double r = rsqrt_nr(d);
      dv[c] = d;
      rv[c] = r;
      if (c < 7) {
        const double l0 = 2 * t > c ? a0 * r : 0.0;
        const double l1 = 2 * t + 1 > c ? a1 * r : 0.0;
        const double x = xD * r;
        v[D][0] = fma(-x, l0, v[D][0]);
        v[D][1] = fma(-x, l1, v[D][1]);
        if (below) {
          const double y = xE * r;
          E[0] = fma(-y, l0, E[0]);
          E[1] = fma(-y, l1, E[1]);
        }
      }
      // the previous panel's deferred tiles, spread over this panel's chain
      if (kDeferJobs && p >= 1) {
        constexpr int kChunks = 8;
        const int nj = panel_njobs<TN>(p - 1);
        panel_jobs<TN>(v, fr, wb, p - 1, (c * nj) / kChunks, ((c + 1) * nj) / kChunks, g, t);
      }
    }
    // scale: column 2t + q by its r; the diagonal gets sqrt(d)
    double r0 = rv[0], r1 = rv[1], d0 = dv[0], d1 = dv[1];
#pragma unroll
    for (int q = 1; q < 4; ++q) {
      r0 = t == q ? rv[2 * q] : r0;
      r1 = t == q ? rv[2 * q + 1] : r1;
      d0 = t == q ? dv[2 * q] : d0;
      d1 = t == q ? dv[2 * q + 1] : d1;
    }
    v[D][0] = g == 2 * t ? sqrt_from_rsqrt(d0, r0) : v[D][0] * r0;
    v[D][1] = g == 2 * t + 1 ? sqrt_from_rsqrt(d1, r1) : v[D][1] * r1;
    if (below) {
      E[0] *= r0;
      E[1] *= r1;
      // B fragments of W^T: wb[ks] = W^T(4ks + t, g), held by lane 4(4ks + t) + g/2
#pragma unroll
      for (int ks = 0; ks < 2; ++ks) {
        const int src = 16 * ks + 4 * t + (g >> 1);
        const double e0 = __shfl_sync(0xffffffffu, E[0], src);
        const double e1 = __shfl_sync(0xffffffffu, E[1], src);
        wb[ks] = (g & 1) ? e1 : e0;
      }
      // critical: L_{p+1,p} = A W^T and the update of the next diagonal tile
      const int i = p + 1, N = T::id(p + 1, p + 1);
      const double a0 = tile_frag(v[T::id(i, p)][0], v[T::id(i, p)][1], 0, g, t);
      const double a1 = tile_frag(v[T::id(i, p)][0], v[T::id(i, p)][1], 1, g, t);
      double x0 = 0.0, x1 = 0.0, y0 = 0.0, y1 = 0.0;
      dmma_884(x0, x1, a0, wb[0]);
      dmma_884(y0, y1, a1, wb[1]);
      v[T::id(i, p)][0] = x0 + y0;
      v[T::id(i, p)][1] = x1 + y1;
      fr[i][0] = tile_frag(v[T::id(i, p)][0], v[T::id(i, p)][1], 0, g, t);
      fr[i][1] = tile_frag(v[T::id(i, p)][0], v[T::id(i, p)][1], 1, g, t);
      double z0 = 0.0, z1 = 0.0;
      dmma_884(v[N][0], v[N][1], -fr[i][0], fr[i][0]);
      dmma_884(z0, z1, -fr[i][1], fr[i][1]);
      v[N][0] += z0;
      v[N][1] += z1;
      if (!kDeferJobs) panel_jobs<TN>(v, fr, wb, p, 0, panel_njobs<TN>(p), g, t);
    }
  }
  return bad ? __ffsll((long long)bad) : 0;
}

// Element (row, col) of tile slot (i, k, q) for lane (g, t).
__device__ __forceinline__ int reg_row(int i, int g) { return 8 * i + g; }
__device__ __forceinline__ int reg_col(int k, int t, int q) { return 8 * k + 2 * t + q; }

}  // namespace relapack
