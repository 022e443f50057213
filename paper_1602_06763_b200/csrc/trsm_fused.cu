// trsm_fused.cu — K5: the base case of the recursive TRSM, up to 256 columns
// in ONE launch (north_star subsystem (3); SPEC trsm
// Right/Lower/Trans/NonUnit):
//     B (m x t) := B * L^{-T},   t <= 256,
// every row x of the result solving x L^T = b by forward substitution
//     x_j = (b_j - sum_{k<j} x_k L_jk) * (1 / L_jj).
//
// Organisation.  A CTA owns 64 rows of B (8 warps x 8 rows); its slab stays in
// shared memory for the whole solve.  Columns are walked in 64-wide chunks
// (left-looking): a warp holds its 8 rows of the current chunk as eight 8x8
// DMMA accumulator fragments (lane (g, t) holds X[g][2t], X[g][2t+1] of every
// 8x8 sub-block) and
//   (a) accumulates X_cb -= X_pb L_{cb,pb}^T for the earlier chunks pb on the
//       FP64 tensor cores (mma.sync m8n8k4 f64, A from the slab, B from the
//       staged 64x64 L block);
//   (b) solves the chunk's diagonal block sub-block by sub-block: the 8 columns
//       of a sub-block by quad shuffles (the owner lane of column c scales it,
//       the 4 lanes of each row group update their two columns — one
//       instruction stream serves 8 rows; chain = shuffle -> multiply -> FMA),
//       then X_{s'} -= X_s L_{s',s}^T on DMMA for the later sub-blocks.
// Shared-memory strides are 4 (mod 32) doubles so every fragment read hits
// each bank pair exactly twice.
#include <cstdlib>

#include "chol_regs.cuh"
#include "common.cuh"
#include "kernels.h"
#include "trsm_regs.cuh"

namespace relapack {

namespace {

constexpr int kFC = 64;                  // chunk width
constexpr int kFTmax = kTrsmFusedMax;    // 256
constexpr int kFLdL = kFC + 4;           // L block row stride (== 4 mod 32)

// NW warps x 8 rows per CTA; slab row stride for t columns = a multiple of 32
// plus 4 (== 4 mod 32); shared memory sized for t.
template <int NW>
struct TF {
  static constexpr int ROWS = 8 * NW, THREADS = 32 * NW;
  // (whole 64-column chunks: the solve walks the last chunk's columns past t)
  static __host__ __device__ int ldx(int t) { return ((t + kFC - 1) / kFC) * kFC + 4; }
  // t <= 128: every L block the solve needs (two diagonal, one below) is
  // staged once up front; t > 128: one block at a time
  static __host__ __device__ int lblocks(int t) { return t <= 2 * kFC ? 3 : 1; }
  static __host__ __device__ size_t smem(int t) {
    return sizeof(double) * ((size_t)ROWS * ldx(t) + (size_t)lblocks(t) * kFC * kFLdL + 2 * kFC);
  }
};

#ifdef RELAPACK_PROBE  // phase timestamps for tools/microbench only
__device__ long long g_tprobe[64];
#define TPROBE(k) \
  if (threadIdx.x == 0 && blockIdx.x == 0) g_tprobe[k] = clock64();
#else
#define TPROBE(k)
#endif

// Stage the 64x64 block of L with rows [r0, r0+64) and cols [c0, c0+64) into
// sL[j * kFLdL + k] = L(r0 + j, c0 + k), zero outside [0, t) and, for the
// diagonal block, on/above the diagonal (1/L_jj goes to rinv).
template <int NW>
__device__ __forceinline__ void stage_L(double* sL, double* rinv, const double* __restrict__ L, int64_t ldl,
                                        int layout, int t, int r0, int c0, bool diag) {
  constexpr int kFThreads = TF<NW>::THREADS;
  constexpr int kPer = kFC * kFC / kFThreads;
  double v[kPer];
#pragma unroll
  for (int u = 0; u < kPer; ++u) {
    const int e = threadIdx.x + u * kFThreads;
    const int a = e & (kFC - 1), b = e >> 6;  // a: contiguous index
    const int j = layout == kLayoutN ? a : b, k = layout == kLayoutN ? b : a;
    const int gi = r0 + j, gk = c0 + k;
    v[u] = (gi < t && gk < t && (!diag || gi >= gk)) ? L[lv_off(layout, gi, gk, ldl)] : 0.0;
  }
#pragma unroll
  for (int u = 0; u < kPer; ++u) {
    const int e = threadIdx.x + u * kFThreads;
    const int a = e & (kFC - 1), b = e >> 6;
    const int j = layout == kLayoutN ? a : b, k = layout == kLayoutN ? b : a;
    if (diag && j == k) rinv[j] = (r0 + j < t) ? 1.0 / v[u] : 0.0;
    sL[j * kFLdL + k] = (diag && j <= k) ? 0.0 : v[u];
  }
}

// t <= 128: stage L(0:64, 0:64), L(64:128, 64:128) (diagonal blocks) and
// L(64:128, 0:64) in one pass of asynchronous 8-byte copies (cp.async: no
// registers held, every copy of a thread in flight); finish_L_all completes it.
template <int NW>
__device__ __forceinline__ void stage_L_all(double* sL, const double* __restrict__ L, int64_t ldl, int layout,
                                            int t) {
  constexpr int kFThreads = TF<NW>::THREADS;
  constexpr int kPer = kFC * kFC / kFThreads;
  auto cp8 = [](double* dst, const double* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(smem_u32(dst)), "l"(src) : "memory");
  };
  // layout T: the L-view column index is contiguous in memory and in the
  // block's shared-memory rows, so whole pairs go as one 16-byte copy (half
  // the copy instructions, which bound this prologue)
  const bool pairs = layout == kLayoutT && (ldl & 1) == 0 && (reinterpret_cast<uintptr_t>(L) & 15) == 0;
#pragma unroll
  for (int bk = 0; bk < 3; ++bk) {
    const int r0 = bk == 0 ? 0 : kFC, c0 = bk == 1 ? kFC : 0;
    if (pairs) {
#pragma unroll 4
      for (int u = 0; u < kPer / 2; ++u) {
        const int e = threadIdx.x + u * kFThreads;
        const int k = 2 * (e & (kFC / 2 - 1)), j = e >> 5;
        const int gi = r0 + j, gk = c0 + k;
        double* dst = sL + bk * kFC * kFLdL + j * kFLdL + k;
        const bool ok0 = gi < t && gk < t && (bk == 2 || gi >= gk);
        const bool ok1 = gi < t && gk + 1 < t && (bk == 2 || gi >= gk + 1);
        const double* src = L + lv_off(kLayoutT, gi, gk, ldl);
        if (ok0 && ok1) {
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(dst)), "l"(src) : "memory");
        } else {
          if (ok0) cp8(dst, src); else dst[0] = 0.0;
          if (ok1) cp8(dst + 1, src + 1); else dst[1] = 0.0;
        }
      }
    } else if (layout == kLayoutN) {
      // transposing copy: a warp moves an 8 (rows j, contiguous in global)
      // x 4 (columns k) patch, so its eight 64-byte global segments are whole
      // and its shared-memory stores (row stride kFLdL = 4 mod 16 doubles) hit
      // every bank pair exactly twice (a 32-row column would be 8-way)
      const int lane = threadIdx.x & 31;
#pragma unroll 4
      for (int u = 0; u < kPer; ++u) {
        const int blk = (threadIdx.x >> 5) + u * (kFThreads / 32);  // 0 .. 127: 8 row patches x 16 column patches
        const int j = 8 * (blk & 7) + (lane & 7), k = 4 * (blk >> 3) + (lane >> 3);
        const int gi = r0 + j, gk = c0 + k;
        double* dst = sL + bk * kFC * kFLdL + j * kFLdL + k;
        if (gi < t && gk < t && (bk == 2 || gi >= gk))
          cp8(dst, L + lv_off(kLayoutN, gi, gk, ldl));
        else
          *dst = 0.0;
      }
    } else {
#pragma unroll 4
      for (int u = 0; u < kPer; ++u) {
        const int e = threadIdx.x + u * kFThreads;
        const int a = e & (kFC - 1), b = e >> 6;
        const int j = layout == kLayoutN ? a : b, k = layout == kLayoutN ? b : a;
        const int gi = r0 + j, gk = c0 + k;
        double* dst = sL + bk * kFC * kFLdL + j * kFLdL + k;
        if (gi < t && gk < t && (bk == 2 || gi >= gk))
          cp8(dst, L + lv_off(layout, gi, gk, ldl));
        else
          *dst = 0.0;
      }
    }
  }
}

// After stage_L_all: wait for the copies, then move the diagonal of the two
// diagonal blocks into 1/L_jj and zero it.
template <int NW>
__device__ __forceinline__ void finish_L_all(double* sL, double* rinv, int t) {
  asm volatile("cp.async.wait_all;\n" ::: "memory");
  __syncthreads();
  if (threadIdx.x < 2 * kFC) {
    const int bk = threadIdx.x / kFC, j = threadIdx.x % kFC;
    double* d = sL + bk * kFC * kFLdL + j * kFLdL + j;
    rinv[bk * kFC + j] = (bk * kFC + j < t) ? 1.0 / *d : 0.0;
    *d = 0.0;
  }
}

template <int NW>
__global__ void __launch_bounds__(TF<NW>::THREADS, 8 / NW)
    k_trsm_fused(const double* __restrict__ L, int64_t ldl, double* __restrict__ B, int64_t ldb, int layout, int m,
                 int t, const int* d_info, TraceRec* tr) {
  constexpr int kFRows = TF<NW>::ROWS, kFThreads = TF<NW>::THREADS;
  TPROBE(0);
  {
    const KState ks = ld_state(d_info);
    if (ks.info != 0) return;
    L = rebase(L, ks.base);
    B = rebase(B, ks.base);
  }
  trace_begin(tr);
  extern __shared__ double smem_t[];
  const int kFLdX = TF<NW>::ldx(t);
  double* sX = smem_t;                   // sX[r * kFLdX + c]
  const bool pre = TF<NW>::lblocks(t) == 3;
  double* sL = sX + kFRows * kFLdX;      // current 64x64 L block (pre: the three blocks)
  double* sRinv = sL + TF<NW>::lblocks(t) * kFC * kFLdL;  // 1 / L_jj of the diagonal chunk(s)
  const int row0 = blockIdx.x * kFRows;
  const int rows = min(kFRows, m - row0);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, tq = lane & 3;
  const int wrow = warp * 8;             // this warp's first slab row

  // ---- stage L (t <= 128: every block at once by cp.async, in flight while
  // the slab is loaded through registers, 16 loads in flight per thread)
  if (pre) stage_L_all<NW>(sL, L, ldl, layout, t);
  {
    const int total = kFRows * t;
    for (int e0 = tid; e0 < total; e0 += kFThreads * 16) {
      double v[16];
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        const int e = e0 + u * kFThreads;
        const int r = layout == kLayoutN ? e % kFRows : e / t, c = layout == kLayoutN ? e / kFRows : e % t;
        v[u] = (e < total && r < rows) ? B[lv_off(layout, row0 + r, c, ldb)] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        const int e = e0 + u * kFThreads;
        const int r = layout == kLayoutN ? e % kFRows : e / t, c = layout == kLayoutN ? e / kFRows : e % t;
        if (e < total) sX[r * kFLdX + c] = v[u];
      }
    }
  }
  if (pre) finish_L_all<NW>(sL, sRinv, t);
  __syncthreads();
  TPROBE(1);

  const int nc = (t + kFC - 1) / kFC;
  for (int cb = 0; cb < nc; ++cb) {
    const int cbase = cb * kFC;
    // this warp's 8 rows of chunk cb as eight 8x8 C fragments
    double xs[8][2];
#pragma unroll
    for (int s = 0; s < 8; ++s) {
      xs[s][0] = sX[(wrow + g) * kFLdX + cbase + 8 * s + 2 * tq];
      xs[s][1] = sX[(wrow + g) * kFLdX + cbase + 8 * s + 2 * tq + 1];
    }
    // ---- (a) X_cb -= X_pb L_{cb,pb}^T, pb < cb
    for (int pb = 0; pb < cb; ++pb) {
      const double* sLb = pre ? sL + 2 * kFC * kFLdL : sL;
      if (!pre) {
        __syncthreads();  // sL free
        stage_L<NW>(sL, sRinv, L, ldl, layout, t, cbase, pb * kFC, false);
        __syncthreads();
      }
#pragma unroll 4
      for (int k0 = 0; k0 < kFC; k0 += 4) {
        const double a = -sX[(wrow + g) * kFLdX + pb * kFC + k0 + tq];
#pragma unroll
        for (int s = 0; s < 8; ++s) dmma_884(xs[s][0], xs[s][1], a, sLb[(8 * s + g) * kFLdL + k0 + tq]);
      }
    }
    // ---- (b) solve the diagonal chunk
    const double* sLd = pre ? sL + cb * kFC * kFLdL : sL;
    const double* sRd = pre ? sRinv + cb * kFC : sRinv;
    if (!pre) {
      __syncthreads();
      stage_L<NW>(sL, sRinv, L, ldl, layout, t, cbase, cbase, true);
      __syncthreads();
    }
    TPROBE(2 + 2 * cb);
#pragma unroll
    for (int s = 0; s < 8; ++s) {
      // columns 8s .. 8s+7: the owner lane (quad position c/2) of column c
      // broadcasts x_c to its quad; each lane updates its columns 2t, 2t+1
      double l0[8], l1[8], rc[8];
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        l0[c] = sLd[(8 * s + 2 * tq) * kFLdL + 8 * s + c];      // L(8s+2t,   8s+c), 0 unless 2t > c
        l1[c] = sLd[(8 * s + 2 * tq + 1) * kFLdL + 8 * s + c];  // L(8s+2t+1, 8s+c)
        rc[c] = sRd[8 * s + c];
      }
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const double xj = __shfl_sync(0xffffffffu, (c & 1) ? xs[s][1] : xs[s][0], (lane & ~3) | (c >> 1)) * rc[c];
        xs[s][0] -= xj * l0[c];
        xs[s][1] -= xj * l1[c];
        if (tq == (c >> 1)) {
          if (c & 1)
            xs[s][1] = xj;
          else
            xs[s][0] = xj;
        }
      }
      // X_{s'} -= X_s L_{s',s}^T for s' > s: A fragment of X_s from the quad
#pragma unroll
      for (int ks = 0; ks < 2; ++ks) {
        const int src = (lane & ~3) | (2 * ks + (tq >> 1));
        const double e0 = __shfl_sync(0xffffffffu, xs[s][0], src);
        const double e1 = __shfl_sync(0xffffffffu, xs[s][1], src);
        const double a = -((tq & 1) ? e1 : e0);  // -X_s[g][4ks + tq]
#pragma unroll
        for (int s2 = s + 1; s2 < 8; ++s2)
          dmma_884(xs[s2][0], xs[s2][1], a, sLd[(8 * s2 + g) * kFLdL + 8 * s + 4 * ks + tq]);
      }
    }
#pragma unroll
    for (int s = 0; s < 8; ++s) {
      sX[(wrow + g) * kFLdX + cbase + 8 * s + 2 * tq] = xs[s][0];
      sX[(wrow + g) * kFLdX + cbase + 8 * s + 2 * tq + 1] = xs[s][1];
    }
    TPROBE(3 + 2 * cb);
  }
  __syncthreads();
  pdl_trigger();
  // ---- write the slab back
  {
    const int total = kFRows * t;
    for (int e = tid; e < total; e += kFThreads) {
      const int r = layout == kLayoutN ? e % kFRows : e / t, c = layout == kLayoutN ? e / kFRows : e % t;
      if (r < rows) B[lv_off(layout, row0 + r, c, ldb)] = sX[r * kFLdX + c];
    }
  }
  TPROBE(20);
  trace_end(tr);
}

// ---- t <= 128 with the row slab in REGISTERS: each warp owns RG groups of 8
// rows and all t columns (16 accumulator tiles per group), so shared memory
// holds only the three L blocks (104 KB) and a CTA covers 8 * RG * NW rows —
// twice the rows per SM of the shared-memory slab at the same per-warp chain
// (the RG groups' substitution chains interleave in one instruction stream).
template <int NW, int RG>
struct TRG {
  static constexpr int ROWS = 8 * RG * NW, THREADS = 32 * NW;
  static constexpr size_t SMEM = sizeof(double) * (3 * (size_t)kFC * kFLdL + 2 * kFC);
};

template <int NW, int RG, int NC>
__global__ void __launch_bounds__(TRG<NW, RG>::THREADS, 1)
    k_trsm_reg(const double* __restrict__ L, int64_t ldl, double* __restrict__ B, int64_t ldb, int layout, int m,
               int t, const int* d_info, TraceRec* tr) {
  {
    const KState ks = ld_state(d_info);
    if (ks.info != 0) return;
    L = rebase(L, ks.base);
    B = rebase(B, ks.base);
  }
  trace_begin(tr);
  TPROBE(0);
  extern __shared__ double smem_r[];
  double* sL = smem_r;                    // the three 64x64 L blocks
  double* sRinv = sL + 3 * kFC * kFLdL;   // 1 / L_jj of both diagonal blocks
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, tq = lane & 3;
  const int row_base = blockIdx.x * TRG<NW, RG>::ROWS + warp * 8 * RG;
  stage_L_all<NW>(sL, L, ldl, layout, t);  // async, overlaps the slab loads
  TPROBE(6);
  constexpr int NT = 8 * NC;  // 8-column tiles held (t <= 64 NC)
  double xs[RG][NT][2];
  const bool pairs = layout == kLayoutT && (ldb & 1) == 0 && (reinterpret_cast<uintptr_t>(B) & 15) == 0;
#pragma unroll
  for (int r = 0; r < RG; ++r)
#pragma unroll
    for (int sb = 0; sb < NT; ++sb) {
      const int row = row_base + 8 * r + g, col = 8 * sb + 2 * tq;
      if (pairs && row < m && col + 1 < t) {
        const double2 v = *reinterpret_cast<const double2*>(B + lv_off(kLayoutT, row, col, ldb));
        xs[r][sb][0] = v.x;
        xs[r][sb][1] = v.y;
      } else {
#pragma unroll
        for (int q = 0; q < 2; ++q)
          xs[r][sb][q] = (row < m && col + q < t) ? B[lv_off(layout, row, col + q, ldb)] : 0.0;
      }
    }
  TPROBE(7);
  finish_L_all<NW>(sL, sRinv, t);
  __syncthreads();
  TPROBE(1);
  solve_chunk_regs<RG, 0, NT, kFLdL, 1>(xs, sL, sRinv, lane, g, tq);
  TPROBE(2);
  if (NC == 2 && t > kFC) {  // (NC == 1 instances never get here: t <= 64)
    // X_1 -= X_0 L_{1,0}^T (A fragments of X_0 from the quads, B from block 2)
    update_chunk1_regs<RG, NT, kFLdL, 1>(xs, sL + 2 * kFC * kFLdL, g, tq);
    TPROBE(3);
    if constexpr (NC == 2) solve_chunk_regs<RG, 1, NT, kFLdL, 1>(xs, sL + kFC * kFLdL, sRinv + kFC, lane, g, tq);
    TPROBE(4);
  }
  pdl_trigger();
#pragma unroll
  for (int r = 0; r < RG; ++r)
#pragma unroll
    for (int sb = 0; sb < NT; ++sb) {
      const int row = row_base + 8 * r + g, col = 8 * sb + 2 * tq;
      if (pairs && row < m && col + 1 < t) {
        *reinterpret_cast<double2*>(B + lv_off(kLayoutT, row, col, ldb)) = make_double2(xs[r][sb][0], xs[r][sb][1]);
      } else {
#pragma unroll
        for (int q = 0; q < 2; ++q)
          if (row < m && col + q < t) B[lv_off(layout, row, col + q, ldb)] = xs[r][sb][q];
      }
    }
  TPROBE(5);
  trace_end(tr);
}

template <int NW, int RG>
cudaError_t launch_reg(const double* L, int64_t ldl, double* B, int64_t ldb, int layout, int m, int t,
                       const int* d_info, cudaStream_t st) {
  const int grid = (m + TRG<NW, RG>::ROWS - 1) / TRG<NW, RG>::ROWS;
  if (t <= kFC)
    k_trsm_reg<NW, RG, 1><<<grid, TRG<NW, RG>::THREADS, TRG<NW, RG>::SMEM, st>>>(L, ldl, B, ldb, layout, m, t, d_info,
                                                                                g_launch_trace);
  else
    k_trsm_reg<NW, RG, 2><<<grid, TRG<NW, RG>::THREADS, TRG<NW, RG>::SMEM, st>>>(L, ldl, B, ldb, layout, m, t, d_info,
                                                                                g_launch_trace);
  return cudaGetLastError();
}

template <int NW>
cudaError_t launch_nw(const double* L, int64_t ldl, double* B, int64_t ldb, int layout, int m, int t,
                      const int* d_info, cudaStream_t st) {
  const int grid = (m + TF<NW>::ROWS - 1) / TF<NW>::ROWS;
  k_trsm_fused<NW><<<grid, TF<NW>::THREADS, TF<NW>::smem(t), st>>>(L, ldl, B, ldb, layout, m, t, d_info,
                                                                     g_launch_trace);
  return cudaGetLastError();
}

}  // namespace

template <int NW>
size_t max_smem() {
  size_t m = 0;
  for (int t = 8; t <= kFTmax; t += 8) m = TF<NW>::smem(t) > m ? TF<NW>::smem(t) : m;
  return m;
}

cudaError_t configure_trsm_fused() {
  cudaError_t e =
      cudaFuncSetAttribute(k_trsm_fused<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)max_smem<8>());
  if (e != cudaSuccess) return e;
  if ((e = cudaFuncSetAttribute(k_trsm_fused<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)max_smem<4>())) !=
      cudaSuccess)
    return e;
  const auto attr = cudaFuncAttributeMaxDynamicSharedMemorySize;
  if ((e = cudaFuncSetAttribute(k_trsm_reg<8, 2, 2>, attr, (int)TRG<8, 2>::SMEM)) != cudaSuccess) return e;
  if ((e = cudaFuncSetAttribute(k_trsm_reg<8, 1, 2>, attr, (int)TRG<8, 1>::SMEM)) != cudaSuccess) return e;
  if ((e = cudaFuncSetAttribute(k_trsm_reg<4, 1, 2>, attr, (int)TRG<4, 1>::SMEM)) != cudaSuccess) return e;
  if ((e = cudaFuncSetAttribute(k_trsm_reg<8, 2, 1>, attr, (int)TRG<8, 2>::SMEM)) != cudaSuccess) return e;
  if ((e = cudaFuncSetAttribute(k_trsm_reg<8, 1, 1>, attr, (int)TRG<8, 1>::SMEM)) != cudaSuccess) return e;
  return cudaFuncSetAttribute(k_trsm_reg<4, 1, 1>, attr, (int)TRG<4, 1>::SMEM);
}

// 64-row CTAs (8 warps) for tall panels (m >= 2048), 32-row CTAs (4 warps, two
// CTAs per SM, twice the CTAs) for shorter ones — measured, profiles/
// (RELAPACK_TRSM_NW=4|8 forces one).
static int trsm_nw(int m) {
  static const int forced = [] {
    const char* v = getenv("RELAPACK_TRSM_NW");
    return v ? atoi(v) : 0;
  }();
  if (forced == 4 || forced == 8) return forced;
  static const int m8 = [] {  // RELAPACK_TRSM_NW8_FROM: panel height from which 64-row CTAs are used
    const char* v = getenv("RELAPACK_TRSM_NW8_FROM");
    return v ? atoi(v) : 2048;
  }();
  return m >= m8 ? 8 : 4;
}

// RELAPACK_TRSM_REG: 0 = shared-memory slab kernel only, 1 = register-slab
// kernel for t <= 128 (default), 2 = always 128-row register CTAs;
// RELAPACK_TRSM_RG2_FROM = panel height from which the 128-row CTAs are used,
// RELAPACK_TRSM_REG8_FROM = from which the 64-row (8-warp) CTAs are used
static int trsm_reg_mode() {
  static const int v = [] {
    const char* e = getenv("RELAPACK_TRSM_REG");
    return e ? atoi(e) : 1;
  }();
  return v;
}
static int trsm_rg2_from() {
  static const int v = [] {
    const char* e = getenv("RELAPACK_TRSM_RG2_FROM");
    return e ? atoi(e) : (1 << 30);  // the 2-group variant spills: off unless asked for
  }();
  return v;
}
static int trsm_reg8_from() {
  static const int v = [] {
    const char* e = getenv("RELAPACK_TRSM_REG8_FROM");
    return e ? atoi(e) : 2048;
  }();
  return v;
}

cudaError_t launch_trsm_fused(const double* L, int64_t ldl, double* B, int64_t ldb, int layout, int m, int t,
                              const int* d_info, cudaStream_t st) {
  if (m <= 0 || t <= 0) return cudaSuccess;
  if (t > kFTmax) return cudaErrorInvalidValue;
  if (t <= 2 * kFC && trsm_reg_mode() > 0) {
    // register-slab kernel: 128-row CTAs for tall panels, 64 / 32 rows below
    const int mode = trsm_reg_mode();
    if (mode == 2 || (mode == 1 && m >= trsm_rg2_from())) return launch_reg<8, 2>(L, ldl, B, ldb, layout, m, t, d_info, st);
    if (m >= trsm_reg8_from()) return launch_reg<8, 1>(L, ldl, B, ldb, layout, m, t, d_info, st);
    return launch_reg<4, 1>(L, ldl, B, ldb, layout, m, t, d_info, st);
  }
  return trsm_nw(m) == 8 ? launch_nw<8>(L, ldl, B, ldb, layout, m, t, d_info, st)
                        : launch_nw<4>(L, ldl, B, ldb, layout, m, t, d_info, st);
}

// Test hook dispatch (hooks.cu): 1 reg<4,1>, 2 reg<8,1>, 3 reg<8,2>, 4 smem-slab<4>, 5 smem-slab<8>.
cudaError_t launch_trsm_fused_variant(int v, const double* L, int64_t ldl, double* B, int64_t ldb, int layout, int m,
                                      int t, const int* d_info, cudaStream_t st) {
  if (m <= 0 || t <= 0) return cudaSuccess;
  if (t > kFTmax || (v <= 3 && t > 2 * kFC)) return cudaErrorInvalidValue;
  switch (v) {
    case 1: return launch_reg<4, 1>(L, ldl, B, ldb, layout, m, t, d_info, st);
    case 2: return launch_reg<8, 1>(L, ldl, B, ldb, layout, m, t, d_info, st);
    case 3: return launch_reg<8, 2>(L, ldl, B, ldb, layout, m, t, d_info, st);
    case 4: return launch_nw<4>(L, ldl, B, ldb, layout, m, t, d_info, st);
    case 5: return launch_nw<8>(L, ldl, B, ldb, layout, m, t, d_info, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace relapack
