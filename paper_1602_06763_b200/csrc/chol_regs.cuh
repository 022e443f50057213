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

// Factor in place.  Returns 0 or the 1-based first column whose pivot failed
// (!(d >= kMinPivot): d <= 0, -0.0, NaN, or subnormal — common.cuh); the
// values after a failure are unspecified.
//
// Per panel column c the stored column stays unscaled until the panel ends;
// the column values are scaled as they are used (x = a_ic * r, the same
// product that is stored at the end), so every l_ij that enters an update is
// exactly the stored one.  Only lanes' own columns k > c are updated: the
// multiplier l_kc of a finished column is 0.  (Plain substitution, no
// explicit inverses: exact on integer factors whose pivots are perfect
// squares, backward stable otherwise.)
// sink(p) is called once panel p's tiles (i, p), i >= p, hold their final
// values, before the trailing update: a caller that stores them there (the
// batched kernel) lets them die early, which lowers the register peak.
struct NoSink {
  __device__ __forceinline__ void operator()(int) const {}
};

#ifndef RELAPACK_REG_DEFER
#define RELAPACK_REG_DEFER 0
#endif

// Deferred trailing update of panel PP (fragments fp) on the tiles (i, k),
// PP + 2 <= k <= i: DMMA number [lo, hi) of its list (all k-step 0 DMMAs
// first, then k-step 1, so a tile's two dependent DMMAs are far apart).
template <int TN, int PP>
__device__ __forceinline__ void reg_deferred(double (&v)[RegTri<TN>::NT][2], const double (&fp)[TN][2], int lo, int hi) {
  using T = RegTri<TN>;
#pragma unroll
  for (int ks = 0; ks < 2; ++ks)
#pragma unroll
    for (int k = PP + 2; k < TN; ++k)
#pragma unroll
      for (int i = k; i < TN; ++i) {
        // position of (ks, k, i) in the list
        const int idx = ks * ((TN - PP - 2) * (TN - PP - 1) / 2) + ((k - PP - 2) * (2 * TN - PP - k - 1)) / 2 + (i - k);
        if (idx >= lo && idx < hi) dmma_884(v[T::id(i, k)][0], v[T::id(i, k)][1], -fp[i][ks], fp[k][ks]);
      }
}

// Panel P of the register factorization (compile-time P: every register
// index is static), then panel P + 1.
template <int TN, int P, class Sink>
__device__ __forceinline__ void reg_panel(double (&v)[RegTri<TN>::NT][2], double (&fprev)[TN][2], int lane,
                                          uint64_t& bad, Sink& sink) {
  using T = RegTri<TN>;
  const int g = lane >> 2, t = lane & 3;
  constexpr int D = T::id(P, P);
  constexpr bool kDefer = RELAPACK_REG_DEFER != 0;
  constexpr int ndef = (kDefer && P >= 1) ? (TN - P - 1) * (TN - P) : 0;  // panel P-1's deferred DMMAs
  // this lane's columns 2t, 2t + 1: their 1/sqrt(d) and d, picked as the
  // panel's columns go by (no per-panel arrays of all eight)
  double r0 = 0.0, r1 = 0.0, d0 = 1.0, d1 = 1.0;
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    const int e = c & 1, tc = c >> 1;
    const int quad_src = (lane & ~3) | tc;
    const double d = __shfl_sync(0xffffffffu, v[D][e], 4 * c + tc);
    // unscaled column values
    double a0 = 0.0, a1 = 0.0;
    double xc[TN];
    if (c < 7) {
      a0 = __shfl_sync(0xffffffffu, v[D][e], 8 * t + tc);      // a(8P + 2t,     8P + c)
      a1 = __shfl_sync(0xffffffffu, v[D][e], 8 * t + 4 + tc);  // a(8P + 2t + 1, 8P + c)
#pragma unroll
      for (int i = P; i < TN; ++i) xc[i] = __shfl_sync(0xffffffffu, v[T::id(i, P)][e], quad_src);
    }
    bad |= (uint64_t)(!(d >= kMinPivot)) << (8 * P + c);
    const double r = rsqrt_nr(d);
    if constexpr (ndef > 0) reg_deferred<TN, (P >= 1 ? P - 1 : 0)>(v, fprev, ndef * c / 8, ndef * (c + 1) / 8);
    if (e == 0) {
      r0 = t == tc ? r : r0;
      d0 = t == tc ? d : d0;
    } else {
      r1 = t == tc ? r : r1;
      d1 = t == tc ? d : d1;
    }
    if (c < 7) {
      const double l0 = 2 * t > c ? a0 * r : 0.0;
      const double l1 = 2 * t + 1 > c ? a1 * r : 0.0;
#pragma unroll
      for (int i = P; i < TN; ++i) {
        const double x = xc[i] * r;  // l(8i + g, 8P + c)
        v[T::id(i, P)][0] = fma(-x, l0, v[T::id(i, P)][0]);
        v[T::id(i, P)][1] = fma(-x, l1, v[T::id(i, P)][1]);
      }
    }
  }
  // scale the panel: column 2t + q by its r; the diagonal gets sqrt(d)
#pragma unroll
  for (int i = P + 1; i < TN; ++i) {
    v[T::id(i, P)][0] *= r0;
    v[T::id(i, P)][1] *= r1;
  }
  v[D][0] = g == 2 * t ? sqrt_from_rsqrt(d0, r0) : v[D][0] * r0;
  v[D][1] = g == 2 * t + 1 ? sqrt_from_rsqrt(d1, r1) : v[D][1] * r1;
  if constexpr (P + 1 < TN) {
    // A/B fragments of the panel tiles: fr[i][ks] = L(8i + g, 8P + 4ks + t)
#pragma unroll
    for (int i = P + 1; i < TN; ++i) {
      fprev[i][0] = tile_frag(v[T::id(i, P)][0], v[T::id(i, P)][1], 0, g, t);
      fprev[i][1] = tile_frag(v[T::id(i, P)][0], v[T::id(i, P)][1], 1, g, t);
    }
    sink(P);
    // the next panel's column of tiles now; the rest deferred into panel P+1
    // (or at once without RELAPACK_REG_DEFER)
#pragma unroll
    for (int k = P + 1; k < (kDefer ? P + 2 : TN); ++k)
#pragma unroll
      for (int ks = 0; ks < 2; ++ks)
#pragma unroll
        for (int i = k; i < TN; ++i) dmma_884(v[T::id(i, k)][0], v[T::id(i, k)][1], -fprev[i][ks], fprev[k][ks]);
    reg_panel<TN, P + 1>(v, fprev, lane, bad, sink);
  } else {
    sink(P);
  }
}

template <int TN, class Sink = NoSink>
__device__ __forceinline__ int reg_potrf(double (&v)[RegTri<TN>::NT][2], int lane, Sink sink = Sink()) {
  // failed pivots as a bit mask (branch-free: every shuffle stays in converged code)
  uint64_t bad = 0;
  // Panel P-1's update of the columns k >= P+1 is not issued in one block
  // after panel P-1 (the warp would stall on the DMMA pipe in front of panel
  // P's column chain) but spread over panel P's eight column steps, where the
  // chain leaves issue slots idle (RELAPACK_REG_DEFER).
  double fprev[TN][2];
  reg_panel<TN, 0>(v, fprev, lane, bad, sink);
  return bad ? __ffsll((long long)bad) : 0;
}

// Element (row, col) of tile slot (i, k, q) for lane (g, t).
__device__ __forceinline__ int reg_row(int i, int g) { return 8 * i + g; }
__device__ __forceinline__ int reg_col(int k, int t, int q) { return 8 * k + 2 * t + q; }

}  // namespace relapack
