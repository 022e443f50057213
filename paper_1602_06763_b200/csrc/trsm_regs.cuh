// trsm_regs.cuh — the register-resident row solve of the TRSM base case
// (K5, north_star subsystem (3); SPEC trsm Right/Lower/Trans/NonUnit
// S:183-191):  X := X L^{-T} for the 64 columns of one chunk, every row x
// solving x L^T = b by forward substitution
//     x_j = (b_j - sum_{k<j} x_k L_jk) * (1 / L_jj).
// Shared by the TRSM base kernel (trsm_fused.cu: L staged as row-major 64x64
// blocks) and the 256-node base case (potf2.cu: L read in place from the
// node's column-major shared-memory square) — the L access is a template
// stride pair: L(r, c) of the chunk's diagonal block = sLd[r * RS + c * CS].
#pragma once
#include "chol_regs.cuh"
#include "common.cuh"

#ifndef RELAPACK_TRSM_MASKL
#define RELAPACK_TRSM_MASKL 1
#endif
#ifndef RELAPACK_TRSM_SPLITACC
#define RELAPACK_TRSM_SPLITACC 1
#endif

namespace relapack {

// A warp owns RG groups of 8 rows; xs[r][tile][q] holds X(8r + g, 8 tile + 2t + q)
// for lane (g, t) — the DMMA accumulator layout.  Solve the 64 columns of chunk
// CB (tiles 8 CB .. 8 CB + 7) against its diagonal block sLd (1 / L_jj in sRd),
// sub-block by sub-block: the 8 columns of a sub-block by quad shuffles (the
// owner lane of column c scales it, the 4 lanes of each row group update their
// two columns), then X_{s'} -= X_s L_{s',s}^T on DMMA for the later sub-blocks.
template <int RG, int CB, int NT, int RS, int CS>
__device__ __forceinline__ void solve_chunk_regs(double (&xs)[RG][NT][2], const double* sLd, const double* sRd,
                                                 int lane, int g, int tq) {
#pragma unroll
  for (int s = 0; s < 8; ++s) {
    double l0[8], l1[8], rc[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      // L(8s+2t, 8s+c), L(8s+2t+1, 8s+c): zero on/above the diagonal.  Masked
      // (not loaded) by default and always for an in-place L (RS == 1: the
      // node's square holds don't-care values there); unmasked only for the
      // zero-padded staged blocks.
      if (RELAPACK_TRSM_MASKL || RS == 1) {
        l0[c] = 2 * tq > c ? sLd[(8 * s + 2 * tq) * RS + (8 * s + c) * CS] : 0.0;
        l1[c] = 2 * tq + 1 > c ? sLd[(8 * s + 2 * tq + 1) * RS + (8 * s + c) * CS] : 0.0;
      } else {
        l0[c] = sLd[(8 * s + 2 * tq) * RS + (8 * s + c) * CS];
        l1[c] = sLd[(8 * s + 2 * tq + 1) * RS + (8 * s + c) * CS];
      }
      rc[c] = sRd[8 * s + c];
    }
#pragma unroll
    for (int c = 0; c < 8; ++c) {
#pragma unroll
      for (int r = 0; r < RG; ++r) {
        double& x0 = xs[r][8 * CB + s][0];
        double& x1 = xs[r][8 * CB + s][1];
        const double xj = __shfl_sync(0xffffffffu, (c & 1) ? x1 : x0, (lane & ~3) | (c >> 1)) * rc[c];
        x0 -= xj * l0[c];
        x1 -= xj * l1[c];
        if (tq == (c >> 1)) {
          if (c & 1)
            x1 = xj;
          else
            x0 = xj;
        }
      }
    }
#if RELAPACK_TRSM_SPLITACC
    // the next sub-block's tile first, its two k-halves into separate
    // accumulators (two independent DMMAs instead of a dependent pair: the
    // next substitution waits ~one DMMA latency less)
    if (s + 1 < 8) {
#pragma unroll
      for (int r = 0; r < RG; ++r) {
        double a[2];
#pragma unroll
        for (int ks = 0; ks < 2; ++ks) a[ks] = -tile_frag(xs[r][8 * CB + s][0], xs[r][8 * CB + s][1], ks, g, tq);
        double h0 = 0.0, h1 = 0.0;
        dmma_884(xs[r][8 * CB + s + 1][0], xs[r][8 * CB + s + 1][1], a[0],
                 sLd[(8 * (s + 1) + g) * RS + (8 * s + tq) * CS]);
        dmma_884(h0, h1, a[1], sLd[(8 * (s + 1) + g) * RS + (8 * s + 4 + tq) * CS]);
#pragma unroll
        for (int ks = 0; ks < 2; ++ks)
#pragma unroll
          for (int s2 = s + 2; s2 < 8; ++s2)
            dmma_884(xs[r][8 * CB + s2][0], xs[r][8 * CB + s2][1], a[ks],
                     sLd[(8 * s2 + g) * RS + (8 * s + 4 * ks + tq) * CS]);
        xs[r][8 * CB + s + 1][0] += h0;
        xs[r][8 * CB + s + 1][1] += h1;
      }
    }
#else
#pragma unroll
    for (int ks = 0; ks < 2; ++ks) {
#pragma unroll
      for (int r = 0; r < RG; ++r) {
        const double a = -tile_frag(xs[r][8 * CB + s][0], xs[r][8 * CB + s][1], ks, g, tq);  // -X_s[g][4ks + tq]
#pragma unroll
        for (int s2 = s + 1; s2 < 8; ++s2)
          dmma_884(xs[r][8 * CB + s2][0], xs[r][8 * CB + s2][1], a,
                   sLd[(8 * s2 + g) * RS + (8 * s + 4 * ks + tq) * CS]);
      }
    }
#endif
  }
}

// X_1 -= X_0 L_{1,0}^T between the two 64-column chunks (t > 64): A fragments
// of X_0 from the quads, B from the off-diagonal block, L(64 + r, c) =
// sLb[r * RS + c * CS].
template <int RG, int NT, int RS, int CS>
__device__ __forceinline__ void update_chunk1_regs(double (&xs)[RG][NT][2], const double* sLb, int g, int tq) {
#pragma unroll
  for (int k0 = 0; k0 < 64; k0 += 4) {
#pragma unroll
    for (int r = 0; r < RG; ++r) {
      const double a = -tile_frag(xs[r][k0 >> 3][0], xs[r][k0 >> 3][1], (k0 >> 2) & 1, g, tq);
#pragma unroll
      for (int sb = 0; sb < 8; ++sb)
        dmma_884(xs[r][(8 + sb) % NT][0], xs[r][(8 + sb) % NT][1], a, sLb[(8 * sb + g) * RS + (k0 + tq) * CS]);
    }
  }
}

}  // namespace relapack
