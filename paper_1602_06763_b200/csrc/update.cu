// update.cu — K3/K4: the BLAS-3 trailing updates of the recursion on the FP64
// tensor cores of sm_100a.
//
//   C(M x N) -= A(M x K) * B(N x K)^T            (GEMM inside the recursive TRSM:
//                                                 B2 -= X1 Lb^T)
//   C(N x N) -= A A^T, lower triangle only        (SYRK A22 -= L21 L21^T, §8a a4;
//                                                 S:192-200)
//
// All operands are L-view blocks (common.cuh): layout N (uplo 'L', rows
// contiguous) or T (uplo 'U', the k index contiguous).  Design:
//  * CTA tile TBM x TBM (128, or 64 for problems too small to fill 148 SMs),
//    K-step 16, 4-stage shared-memory ring filled by TMA (cp.async.bulk.tensor,
//    128B swizzle) issued by thread 0, mbarrier full/empty handshake.
//  * FP64 tensor cores: mma.sync m8n8k4 f64 (SASS DMMA.8x8x4); each warp owns
//    a 64x32 (TBM 128, 8 warps) or 32x32 (TBM 64, 4 warps) register tile.
//  * the k -> MMA-k mapping differs per layout so both fragment reads are
//    shared-memory bank-conflict free (2 wavefronts per 256 B fragment).
//  * SYRK enumerates only lower-triangular tiles; diagonal tiles mask i < j,
//    so the other triangle is never read or written.
//  * epilogue staged through shared memory: coalesced C -= tile along the
//    contiguous global dimension with 16 loads in flight per thread.
//  * non-TMA fallback (odd ld or a base not 16-B aligned): the CTA fills the
//    same swizzled layout with plain loads, one stage at a time.
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "common.cuh"
#include "kernels.h"

namespace relapack {

namespace {

constexpr int BK = 16, STAGES = 4;
#ifndef RELAPACK_PREFETCH_C
#define RELAPACK_PREFETCH_C 1
#endif
constexpr bool kPrefetchC = RELAPACK_PREFETCH_C != 0;

template <int TBM>
struct Cfg {
  // 128: 8 warps of 64x32 (2 per SMSP, 255-reg budget); 64: 4 warps of
  // 32x32; 32: 4 warps of 16x16 (tiny latency-bound updates: a warp's DMMA
  // issue, K/4 x MT x NT x 16 cycles, is the floor, so small warp tiles)
// 64-tiles: 4 warps of 32x32 (default) or 8 of 32x16 (compile-time knob;
// measured n = 16384 47.06-47.53 vs 47.04 ms, n = 4096 2.25 vs 2.14 ms)
#ifndef RELAPACK_UPD64_WARPS
#define RELAPACK_UPD64_WARPS 4
#endif
  static constexpr int NUM_WARPS = TBM == 128 ? 8 : TBM == 64 ? RELAPACK_UPD64_WARPS : 4;
#ifndef RELAPACK_UPD64_BLOCKS
#define RELAPACK_UPD64_BLOCKS (RELAPACK_UPD64_WARPS == 8 ? 2 : 1)
#endif
  // resident CTAs per SM the register budget is sized for (64-tiles with a
  // 3-CTA budget measured slightly slower: compile-time knob, default 1)
  static constexpr int MIN_BLOCKS = TBM == 128 ? 1 : TBM == 64 ? RELAPACK_UPD64_BLOCKS : 2;
  static constexpr int THREADS = NUM_WARPS * 32;
  static constexpr int WTM = TBM == 128 ? 64 : TBM == 64 ? 32 : 16;  // warp tile rows
  static constexpr int WTN = TBM == 32 || (TBM == 64 && NUM_WARPS == 8) ? 16 : 32;  // warp tile cols
  static constexpr int MT = WTM / 8, NT = WTN / 8;      // DMMA tiles per warp
  static constexpr int WGM = TBM / WTM;                 // warps along M (2)
  static constexpr int TILE_BYTES = TBM * BK * 8;
  static constexpr int STAGE_BYTES = 2 * TILE_BYTES;
  static constexpr int CPAD = TBM + 1;                  // epilogue staging stride (odd)
  static constexpr int PIPE_BYTES =
      STAGES * STAGE_BYTES > TBM * CPAD * 8 ? STAGES * STAGE_BYTES : TBM * CPAD * 8;
  static constexpr int SMEM_BYTES = PIPE_BYTES + 1024 /*align*/ + 2 * STAGES * 8 /*barriers*/;
};

// Byte offset of operand element (row r, k) inside a TBM x 16 stage tile.
// Layout N: TBM/16 TMA boxes of [16 k][16 rows] (128 B rows, 128B swizzle:
// 16-B chunk index XOR (k mod 8)).  Layout T: one box of [TBM rows][16 k].
template <int LAYOUT>
__device__ __forceinline__ uint32_t tile_off(int r, int k) {
  if (LAYOUT == kLayoutN)
    return (uint32_t)((r >> 4) * 2048 + k * 128 + ((((r & 15) >> 1) ^ (k & 7)) << 4) + ((r & 1) << 3));
  else
    return (uint32_t)(r * 128 + ((((k >> 1) ^ (r & 7))) << 4) + ((k & 1) << 3));
}

// MMA k-slot (t = lane%4) of k-step s -> tile k.  Chosen per layout so that
// the 32 lanes of a fragment read hit every bank exactly twice.
template <int LAYOUT>
__device__ __forceinline__ int kmap(int s, int t) {
  return LAYOUT == kLayoutN ? 4 * t + s : 4 * s + t;
}

// Element (i, j) of C belongs to the updated part: every element (tri 0), the
// lower triangle i >= j (tri 1, SYRK) or the upper triangle i <= j (tri 2):
// (i - j) * sign >= 0 with sign = 0 / 1 / -1 — one branch-free test.
__device__ __forceinline__ int tri_sign(int tri) { return tri == 1 ? 1 : tri == 2 ? -1 : 0; }
__device__ __forceinline__ bool tri_keep(int sign, int i, int j) { return (i - j) * sign >= 0; }

__device__ __forceinline__ void tri_index(int x, int& ti, int& tj) {
  int r = (int)((sqrt(8.0 * (double)x + 1.0) - 1.0) * 0.5);
  while ((r + 1) * (r + 2) / 2 <= x) ++r;
  while (r * (r + 1) / 2 > x) --r;
  ti = r;
  tj = x - r * (r + 1) / 2;
}

// Fallback loader: the whole CTA fills one stage with plain loads (zero outside).
template <int LAYOUT, int TBM, int NTHREADS>
__device__ __forceinline__ void fill_tile_ldg(uint8_t* tile, const double* X, int64_t ldx, int rows, int r0, int K,
                                              int k0) {
  for (int e = threadIdx.x; e < TBM * BK; e += NTHREADS) {
    int r, k;
    if (LAYOUT == kLayoutN) {
      r = e % TBM;
      k = e / TBM;
    } else {
      k = e % BK;
      r = e / BK;
    }
    double v = 0.0;
    if (r0 + r < rows && k0 + k < K) v = X[lv_off(LAYOUT, r0 + r, k0 + k, ldx)];
    *reinterpret_cast<double*>(tile + tile_off<LAYOUT>(r, k)) = v;
  }
}

template <int LA, int LB, int TBM>
__device__ __forceinline__ void issue_stage(uint8_t* smem, uint64_t* full, const CUtensorMap* tmA,
                                            const CUtensorMap* tmB, int it, int kt, int m0, int n0) {
  using C = Cfg<TBM>;
  const int s = it % STAGES;
  uint8_t* sa = smem + s * C::STAGE_BYTES;
  uint8_t* sb = sa + C::TILE_BYTES;
  mbar_arrive_expect_tx(&full[s], C::STAGE_BYTES);
  if (LA == kLayoutN) {
#pragma unroll
    for (int b = 0; b < TBM / 16; ++b) tma_load_2d(sa + b * 2048, tmA, m0 + 16 * b, kt * BK, &full[s]);
  } else {
    tma_load_2d(sa, tmA, kt * BK, m0, &full[s]);
  }
  if (LB == kLayoutN) {
#pragma unroll
    for (int b = 0; b < TBM / 16; ++b) tma_load_2d(sb + b * 2048, tmB, n0 + 16 * b, kt * BK, &full[s]);
  } else {
    tma_load_2d(sb, tmB, kt * BK, n0, &full[s]);
  }
}

// One BK-deep step of the warp tile: 4 MMA k-steps x (MT x NT) DMMA.8x8x4.
// Both fragments use the k-map of A's layout (the k permutation must agree
// between the two operands); for mixed layouts B's reads are 4-way instead of
// 2-way bank-conflicted, which DMMA's issue rate hides.
template <int LA, int LB, int TBM>
__device__ __forceinline__ void mma_stage(double (&acc)[Cfg<TBM>::MT][Cfg<TBM>::NT][2], const uint8_t* sa,
                                          const uint8_t* sb, int wm, int wn, int g, int t) {
  using C = Cfg<TBM>;
#pragma unroll
  for (int ks = 0; ks < BK / 4; ++ks) {
    const int k = kmap<LA>(ks, t);
    double a[C::MT], b[C::NT];
#pragma unroll
    for (int mt = 0; mt < C::MT; ++mt)
      a[mt] = *reinterpret_cast<const double*>(sa + tile_off<LA>(wm * C::WTM + mt * 8 + g, k));
#pragma unroll
    for (int nt = 0; nt < C::NT; ++nt)
      b[nt] = *reinterpret_cast<const double*>(sb + tile_off<LB>(wn * C::WTN + nt * 8 + g, k));
#pragma unroll
    for (int mt = 0; mt < C::MT; ++mt)
#pragma unroll
      for (int nt = 0; nt < C::NT; ++nt) dmma_884(acc[mt][nt][0], acc[mt][nt][1], a[mt], b[nt]);
  }
}

// One work item (tile, split) of the update; the CTA may process several
// (persistent launch with a capped grid, see launch_tbm).
// GM: the A / B descriptors are the global copies a pointer-independent plan's
// first node rebased (args.gmap, a parameter-space pointer) instead of the
// kernel's own __grid_constant__ parameters — a compile-time choice, so the
// producer's loop holds no runtime select (a register-held select spilled the
// 128-tile kernel; reading it from shared memory slowed the producer).
template <int LA, int LB, int LAYOUT, bool USE_TMA, int TBM, bool GM>
__device__ __forceinline__ void update_item(const CUtensorMap* tmA_p, const CUtensorMap* tmB_p, const UpdateArgs& args,
                                            uint8_t* smem, int work, bool last, const uintptr_t* s_base) {
#define RELAPACK_TMA_A (GM ? args.gmap : tmA_p)
#define RELAPACK_TMA_B (GM ? args.gmap + 1 : tmB_p)
  using C = Cfg<TBM>;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::PIPE_BYTES);
  uint64_t* empty = full + STAGES;

  // work item -> (tile, split): uniform split-K (full_items = 0) is
  // split-major over all tiles; a tail split runs tiles [0, full_items) whole
  // and splits only the rest
  const int ntail = args.ntiles - args.full_items;
  const bool whole = work < args.full_items;
  const int tail_j = work - args.full_items;
  const int tile = whole ? work : args.full_items + tail_j % ntail;
  const int split = whole ? 0 : tail_j / ntail;
  const int ksplit = whole ? 1 : args.ksplit;
  int tm, tn;
  if (args.tri) {
    tri_index(tile, tm, tn);  // tm >= tn: lower tile
    if (args.tri == 2) {      // upper triangle: the transposed tile
      const int x = tm;
      tm = tn;
      tn = x;
    }
  } else {
    // grouped raster: kGroupM tile rows at a time, so the CTAs resident at
    // once share ~12 A panels and ~12 B panels in L2 instead of streaming all
    // of A once per wave of tile columns
    constexpr int kGroupM = 12;
    const int tiles_n = args.ntiles / args.tiles_m;
    const int per_group = kGroupM * tiles_n;
    const int first_m = (tile / per_group) * kGroupM;
    const int gm = min(args.tiles_m - first_m, kGroupM);
    const int local = tile % per_group;
    tm = first_m + local % gm;
    tn = local / gm;
  }
  const int m0 = tm * TBM, n0 = tn * TBM;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wm = warp % C::WGM, wn = warp / C::WGM;
  const int g = lane >> 2, t = lane & 3;
  const int KT_all = (args.K + BK - 1) / BK;
  const int kt_per = (KT_all + ksplit - 1) / ksplit;
  const int kt0 = split * kt_per;
  const int KT = max(0, min(KT_all, kt0 + kt_per) - kt0);  // k-tiles of this split, from kt0

  // Pull this tile of C towards L2 now, so the epilogue's read-modify-write
  // does not start with a DRAM round trip (matters for short K).  Lines along
  // the contiguous dimension; diagonal SYRK tiles are skipped (their upper
  // half belongs to the other triangle).
  if (kPrefetchC && split == 0 && !(args.tri && tm == tn)) {
    const int flim = LAYOUT == kLayoutN ? args.M : args.N, slim = LAYOUT == kLayoutN ? args.N : args.M;
    const int f0 = LAYOUT == kLayoutN ? m0 : n0, s0 = LAYOUT == kLayoutN ? n0 : m0;
    const int fext = min(TBM, flim - f0), sext = min(TBM, slim - s0);
    constexpr int kLineD = 16;  // doubles per 128-byte line
    const int lines = (fext + kLineD - 1) / kLineD;
    for (int e = threadIdx.x; e < lines * sext; e += C::THREADS) {
      const double* pc = rebase(args.C, plan_base(args.d_info)) + (f0 + (e % lines) * kLineD) +
                         (int64_t)(s0 + e / lines) * args.ldc;
      asm volatile("prefetch.global.L2 [%0];" ::"l"(pc));
    }
  }

  double acc[C::MT][C::NT][2];
#pragma unroll
  for (int i = 0; i < C::MT; ++i)
#pragma unroll
    for (int j = 0; j < C::NT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  if (USE_TMA) {
    // Producer = thread 0 (inside warp 0): keeps STAGES-1 TMA stages in flight;
    // a stage is refilled once every warp released it (empty barrier).
    if (threadIdx.x == 0) {
      for (int s = 0; s < STAGES; ++s) {
        mbar_init(&full[s], 1);
        mbar_init(&empty[s], C::NUM_WARPS);
      }
      fence_barrier_init();
      tma_prefetch_desc(RELAPACK_TMA_A);
      tma_prefetch_desc(RELAPACK_TMA_B);
    }
    __syncthreads();
    if (threadIdx.x == 0)
      for (int it = 0; it < STAGES - 1 && it < KT; ++it)
        issue_stage<LA, LB, TBM>(smem, full, RELAPACK_TMA_A, RELAPACK_TMA_B, it, kt0 + it, m0, n0);
    for (int kt = 0; kt < KT; ++kt) {
      if (threadIdx.x == 0 && kt + STAGES - 1 < KT) {
        if (kt >= 1) mbar_wait(&empty[(kt - 1) % STAGES], ((kt - 1) / STAGES) & 1);
        issue_stage<LA, LB, TBM>(smem, full, RELAPACK_TMA_A, RELAPACK_TMA_B, kt + STAGES - 1, kt0 + kt + STAGES - 1,
                                 m0, n0);
      }
      const int s = kt % STAGES;
      mbar_wait(&full[s], (kt / STAGES) & 1);
      const uint8_t* sa = smem + s * C::STAGE_BYTES;
      mma_stage<LA, LB, TBM>(acc, sa, sa + C::TILE_BYTES, wm, wn, g, t);
      // release the stage to the producer's next TMA: the fragment reads are
      // generic-proxy LDS and the refill an async-proxy write of the same
      // bytes, so each lane fences the proxies first (which also waits for its
      // reads to be performed: the scheduler otherwise issues the arrive right
      // behind the last LDS, before its data is back — a WAR race that
      // corrupted ~half of the n = 16384 replays, tools/race_check.py)
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }
  } else {
    for (int kt = 0; kt < KT; ++kt) {
      __syncthreads();
      fill_tile_ldg<LA, TBM, C::THREADS>(smem, rebase(args.A, *s_base), args.lda, args.M, m0, args.K, (kt0 + kt) * BK);
      fill_tile_ldg<LB, TBM, C::THREADS>(smem + C::TILE_BYTES, rebase(args.B, *s_base), args.ldb, args.N, n0, args.K,
                                         (kt0 + kt) * BK);
      __syncthreads();
      mma_stage<LA, LB, TBM>(acc, smem, smem + C::TILE_BYTES, wm, wn, g, t);
    }
  }

  // Epilogue: stage the accumulator tile in shared memory (the pipeline
  // buffers are free now), then C -= tile with coalesced accesses along the
  // contiguous global dimension, 16 independent loads in flight per thread.
  // SYRK tiles write only i >= j.
  if (last) pdl_trigger();  // this CTA's last tile: dependents may launch
  __syncthreads();
  double* sC = reinterpret_cast<double*>(smem);
#pragma unroll
  for (int mt = 0; mt < C::MT; ++mt)
#pragma unroll
    for (int nt = 0; nt < C::NT; ++nt)
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const int il = wm * C::WTM + mt * 8 + g, jl = wn * C::WTN + nt * 8 + 2 * t + c;
        // fast index = the globally contiguous one (i for layout N, j for layout T)
        sC[LAYOUT == kLayoutN ? jl * C::CPAD + il : il * C::CPAD + jl] = acc[mt][nt][c];
      }
  __syncthreads();
  if (ksplit > 1) {
    // deterministic split-K reduction: publish this split's partial tile; the
    // last CTA of the tile sums all partials in split order 0..ksplit-1.
    constexpr int T2 = TBM * TBM;
    double* wsl = args.ws + ((int64_t)split * ntail + (tile - args.full_items)) * T2;
    for (int e = threadIdx.x; e < T2; e += C::THREADS) wsl[e] = sC[(e / TBM) * C::CPAD + (e % TBM)];
    __threadfence();
    __syncthreads();
    __shared__ int s_last;
    if (threadIdx.x == 0) s_last = atomicAdd(&args.counters[tile], 1) == ksplit - 1;
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    // 4 elements x all splits in flight per thread, summed in split order
    constexpr int KSMAX = 16, EB = 4;
    const int64_t sstride = (int64_t)ntail * T2;
    const double* wt = args.ws + (int64_t)(tile - args.full_items) * T2;
    for (int e0 = threadIdx.x; e0 < T2; e0 += C::THREADS * EB) {
      double v[EB][KSMAX];
#pragma unroll
      for (int q = 0; q < EB; ++q)
#pragma unroll
        for (int sp = 0; sp < KSMAX; ++sp) {
          const int e = e0 + q * C::THREADS;
          v[q][sp] = (sp < ksplit && e < T2) ? __ldcg(wt + sp * sstride + e) : 0.0;
        }
#pragma unroll
      for (int q = 0; q < EB; ++q) {
        const int e = e0 + q * C::THREADS;
        double sum = 0.0;
#pragma unroll
        for (int sp = 0; sp < KSMAX; ++sp)
          if (sp < ksplit) sum += v[q][sp];
        if (e < T2) sC[(e / TBM) * C::CPAD + (e % TBM)] = sum;
      }
    }
    if (threadIdx.x == 0) args.counters[tile] = 0;  // ready for the next launch / graph replay
    __syncthreads();
  }
  constexpr int SLOW_STEP = C::THREADS / TBM;  // 2
  const int f = threadIdx.x % TBM;             // fast index
  const int s0 = threadIdx.x / TBM;
  const int fi = (LAYOUT == kLayoutN ? m0 : n0) + f;
  const int flim = LAYOUT == kLayoutN ? args.M : args.N;
  const int slim = LAYOUT == kLayoutN ? args.N : args.M;
  const int sbase = LAYOUT == kLayoutN ? n0 : m0;
  const int tsign = tri_sign(args.tri);
  if (fi < flim) {
    double* Cf = rebase(args.C, *s_base) + fi;  // + slow * ldc
#pragma unroll 1
    constexpr int kRows = TBM / SLOW_STEP, kQ = kRows < 16 ? kRows : 16;  // rows per thread, in flight
    for (int q0 = 0; q0 < kRows; q0 += kQ) {
      double v[kQ];
#pragma unroll
      for (int q = 0; q < kQ; ++q) {
        const int sg = sbase + s0 + SLOW_STEP * (q0 + q);
        const int i = LAYOUT == kLayoutN ? fi : sg, j = LAYOUT == kLayoutN ? sg : fi;
        v[q] = (sg < slim && tri_keep(tsign, i, j)) ? Cf[(int64_t)sg * args.ldc] : 0.0;
      }
#pragma unroll
      for (int q = 0; q < kQ; ++q) {
        const int sl = s0 + SLOW_STEP * (q0 + q);
        const int sg = sbase + sl;
        const int i = LAYOUT == kLayoutN ? fi : sg, j = LAYOUT == kLayoutN ? sg : fi;
        // alpha = -1 (the factorization's C -= A B^T) rounds exactly like v - s
        if (sg < slim && tri_keep(tsign, i, j)) Cf[(int64_t)sg * args.ldc] = fma(args.alpha, sC[sl * C::CPAD + f], v[q]);
      }
    }
  }
}

#undef RELAPACK_TMA_A
#undef RELAPACK_TMA_B

template <int LA, int LB, int LAYOUT, bool USE_TMA, int TBM, bool GM>
__global__ void __launch_bounds__(Cfg<TBM>::THREADS, Cfg<TBM>::MIN_BLOCKS)
    k_update(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, const UpdateArgs args,
             TraceRec* tr) {
  // the global descriptors were rewritten through the generic proxy by the
  // plan's first node (complete before any plan kernel starts, PDL included):
  // acquire them for the tensormap proxy before griddepcontrol.wait, so the
  // fence overlaps the wait instead of delaying the first TMA
  if (GM && threadIdx.x == 0) {
    tma_acquire_desc(args.gmap);
    tma_acquire_desc(args.gmap + 1);
  }
  const KState ks = ld_state(args.d_info);
  if (ks.info != 0) return;  // dpotrf2 semantics: stop after a failed pivot
  trace_begin(tr);
  // the base is read back from shared memory where the offsets become
  // pointers after the main loop (every such use follows a barrier)
  __shared__ uintptr_t s_base;
  if (threadIdx.x == 0) s_base = ks.base;
  extern __shared__ uint8_t smem_raw[];
  // 1024-byte aligned (128B-swizzle atoms) by an integer offset from the
  // __shared__ array, so the compiler keeps the shared address space: the
  // fragment reads are LDS with 32-bit addresses (rounding the pointer through
  // uintptr_t made them generic LD.E with 64-bit address arithmetic per load)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const int nwork = args.full_items + (args.ntiles - args.full_items) * args.ksplit;
  for (int work = blockIdx.x; work < nwork; work += gridDim.x) {
    if (work != (int)blockIdx.x) {
      // previous item fully drained (smem, barriers); its generic-proxy
      // accesses of the ring (fragment reads, the epilogue's staging tile)
      // are ordered before this item's TMA writes into the same bytes
      fence_proxy_async_smem();
      __syncthreads();
    }
    update_item<LA, LB, LAYOUT, USE_TMA, TBM, GM>(&tmA, &tmB, args, smem, work, work + (int)gridDim.x >= nwork,
                                                  &s_base);
  }
  trace_end(tr);
}

template <int LA, int LB, int LC, bool USE_TMA, int TBM, bool GM>
cudaError_t launch_one(const CUtensorMap& ta, const CUtensorMap& tb, const UpdateArgs& a, int grid, cudaStream_t st) {
  k_update<LA, LB, LC, USE_TMA, TBM, GM><<<grid, Cfg<TBM>::THREADS, Cfg<TBM>::SMEM_BYTES, st>>>(ta, tb, a,
                                                                                              g_launch_trace);
  return cudaGetLastError();
}

template <int LA, int LB, int LC, int TBM>
cudaError_t launch_combo(const UpdateOp& op, int grid, cudaStream_t st) {
  if (!op.use_tma) return launch_one<LA, LB, LC, false, TBM, false>(op.tmA, op.tmB, op.args, grid, st);
  return op.args.gmap ? launch_one<LA, LB, LC, true, TBM, true>(op.tmA, op.tmB, op.args, grid, st)
                      : launch_one<LA, LB, LC, true, TBM, false>(op.tmA, op.tmB, op.args, grid, st);
}

// Operand-layout combinations (la, lb, lc): the factorization's (N,N,N) and
// (T,T,T), plus the mixed ones of the other recursive operations (trtri,
// lauum, potrs, getrf), all normalised to lc = N by update_normalize.
template <int TBM>
cudaError_t launch_tbm(const UpdateOp& op, cudaStream_t st) {
  const UpdateArgs& a = op.args;
  int grid = a.full_items + (a.ntiles - a.full_items) * a.ksplit;
  if (op.max_ctas > 0 && grid > op.max_ctas) grid = op.max_ctas;  // persistent, leaves SMs to other streams
  const int combo = a.la * 4 + a.lb * 2 + a.layout;
  switch (combo) {
    case 0: return launch_combo<kLayoutN, kLayoutN, kLayoutN, TBM>(op, grid, st);
    case 7: return launch_combo<kLayoutT, kLayoutT, kLayoutT, TBM>(op, grid, st);
    case 2: return launch_combo<kLayoutN, kLayoutT, kLayoutN, TBM>(op, grid, st);
    case 4: return launch_combo<kLayoutT, kLayoutN, kLayoutN, TBM>(op, grid, st);
    case 6: return launch_combo<kLayoutT, kLayoutT, kLayoutN, TBM>(op, grid, st);
    default: return cudaErrorInvalidValue;  // lc = T with mixed operands: normalise first
  }
}

template <int LA, int LB, int LC, int TBM>
cudaError_t configure_combo() {
  cudaError_t e;
  const int sm = Cfg<TBM>::SMEM_BYTES;
  const auto attr = cudaFuncAttributeMaxDynamicSharedMemorySize;
  if ((e = cudaFuncSetAttribute(k_update<LA, LB, LC, true, TBM, false>, attr, sm)) != cudaSuccess) return e;
  if ((e = cudaFuncSetAttribute(k_update<LA, LB, LC, true, TBM, true>, attr, sm)) != cudaSuccess) return e;
  return cudaFuncSetAttribute(k_update<LA, LB, LC, false, TBM, false>, attr, sm);
}

template <int TBM>
cudaError_t configure_tbm() {
  cudaError_t e;
  if ((e = configure_combo<kLayoutN, kLayoutN, kLayoutN, TBM>()) != cudaSuccess) return e;
  if ((e = configure_combo<kLayoutT, kLayoutT, kLayoutT, TBM>()) != cudaSuccess) return e;
  if ((e = configure_combo<kLayoutN, kLayoutT, kLayoutN, TBM>()) != cudaSuccess) return e;
  if ((e = configure_combo<kLayoutT, kLayoutN, kLayoutN, TBM>()) != cudaSuccess) return e;
  return configure_combo<kLayoutT, kLayoutT, kLayoutN, TBM>();
}

}  // namespace

// RELAPACK_SPLIT128=1: small-grid long-K updates split K over 128-tiles
// instead of dropping to 64-tiles (measured slower: n = 4096 2.43 vs 2.30 ms,
// n = 16384 49.1 vs 48.2 ms, tools/exp22.sh) — off by default
static bool split128_enabled() {
  static const bool on = [] {
    const char* v = getenv("RELAPACK_SPLIT128");
    return v && v[0] == '1';
  }();
  return on;
}

// 64-tile count below which 32-tiles are used (RELAPACK_TILE32_BELOW, 0 = never)
static long small_tile_threshold() {
  static const long t = [] {
    const char* v = getenv("RELAPACK_TILE32_BELOW");
    return v ? atol(v) : 32L;
  }();
  return t;
}

// (RELAPACK_TILE32_MAX_TILES / RELAPACK_TILE32_MAX_K: 32-tiles for any update
// with at most that many 32-tiles and K at most that long)
static long tile32_max_tiles() {
  static const long t = [] {
    const char* v = getenv("RELAPACK_TILE32_MAX_TILES");
    return v ? atol(v) : 0L;
  }();
  return t;
}
static int tile32_max_k() {
  static const int t = [] {
    const char* v = getenv("RELAPACK_TILE32_MAX_K");
    return v ? atoi(v) : 1024;
  }();
  return t;
}

// Tile size for an update: 128 x 128 CTA tiles when they fill the 148 SMs,
// else 64 x 64 (4x the CTAs; latency of the small updates near the leaves),
// and 32 x 32 one-warp tiles when even the 64-tiles would leave most SMs
// idle (the n <= 512 updates on the base-case chain: a 64 x 64 x 128 tile is
// ~4 us of DMMA on one SM).
int update_tile_for(int M, int N, int K, int tri) {
  auto tiles = [&](int t) -> long {
    const long tm = (M + t - 1) / t, tn = (N + t - 1) / t;
    return tri ? tm * (tm + 1) / 2 : tm * tn;
  };
  if (tiles(128) >= 148) return 128;
  // fewer than 148 big tiles but a long K: keep the 128-tiles (8 warps, ~95 %
  // of an SM's DMMA rate) and fill the GPU with split-K rather than dropping
  // to 64-tiles, whose 4 warps of 32 x 32 reach about half of it
  const int KT = (K + BK - 1) / BK;
  if (split128_enabled() && tiles(128) * (KT / 16) >= 148) return 128;
  // short-K updates whose 32-tiles still fit ~4 CTAs per SM: the 4-warp
  // 16x16 tiles finish sooner than 64-tiles (tools/microbench/update_small:
  // gemm 2048x128x128 11.9 -> 7.1 us, gemm 512^2 x 512 24.2 -> 18.8 us)
  if (K <= tile32_max_k() && tiles(32) <= tile32_max_tiles()) return 32;
  if (tiles(64) >= small_tile_threshold()) return 64;
  return 32;
}

static long ntiles_of(int M, int N, int tri, int tile) {
  const long tm = (M + tile - 1) / tile, tn = (N + tile - 1) / tile;
  return tri ? tm * (tm + 1) / 2 : tm * tn;
}

// Split K when the tile grid leaves most of the 148 SMs idle and K is long:
// aim for ~2 CTAs per SM, each split keeping >= 8 k-tiles (128 of K).
// Mid-size grids (1..8 waves of 148 tiles) may also split by 2..4 when that
// shortens the last-wave tail: modelled time = waves(tiles * ks) * (KT / ks +
// 1.5) k-tiles (1.5 = writing one partial tile) + the final sum, against
// waves(tiles) * KT.  Off by default (RELAPACK_SPLITK_MID=1 turns it on):
// measured slower inside the DAG (n = 16384: 49.6 vs 48.6 ms), where
// concurrent launches already fill the tail SMs (tools/exp9.sh).
static bool splitk_mid_enabled() {
  static const bool on = [] {
    const char* v = getenv("RELAPACK_SPLITK_MID");
    return v && v[0] == '1';
  }();
  return on;
}

int update_ksplit_for(int M, int N, int K, int tri, int tile, bool chain) {
  const long tiles = ntiles_of(M, N, tri, tile);
  const int KT = (K + BK - 1) / BK;
  if (tiles >= 148) {
    const long w1 = (tiles + 147) / 148;
    if (!splitk_mid_enabled() || w1 > 8 || KT < 32) return 1;
    double best = (double)w1 * KT;
    int bks = 1;
    for (int ks = 2; ks <= 4; ++ks) {
      const long w = (tiles * ks + 147) / 148;
      const double tcost = (double)w * ((double)KT / ks + 1.5) + 1.5 * (ks + 1);
      if (tcost < 0.95 * best) {
        best = tcost;
        bks = ks;
      }
    }
    return bks;
  }
  static const int min_kt = [] {  // k-tiles per split (RELAPACK_SPLITK_KT, default 8)
    const char* v = getenv("RELAPACK_SPLITK_KT");
    const int x = v ? atoi(v) : 8;
    return x < 1 ? 1 : x;
  }();
  // k-tiles per split on the chain (RELAPACK_SPLITK_CHAIN_KT, 0 = as the
  // other updates): n = 4096 2.058 -> 2.036 ms, n = 16384 unchanged
  static const int chain_kt = [] {
    const char* v = getenv("RELAPACK_SPLITK_CHAIN_KT");
    return v ? atoi(v) : 2;
  }();
  if (chain && chain_kt > 0 && KT >= 16) {
    int ks = (int)((2 * 148 + tiles - 1) / tiles);
    ks = ks < KT / chain_kt ? ks : KT / chain_kt;
    ks = ks < 16 ? ks : 16;
    return ks >= 2 ? ks : 1;
  }
  if (KT < 2 * min_kt) return 1;
  int ks = (int)((2 * 148 + tiles - 1) / tiles);
  ks = ks < KT / min_kt ? ks : KT / min_kt;
  ks = ks < 16 ? ks : 16;
  return ks >= 2 ? ks : 1;
}

int64_t update_ws_elems(int M, int N, int tri, int tile, int ksplit, int full_items) {
  return ksplit > 1 ? (int64_t)ksplit * (ntiles_of(M, N, tri, tile) - full_items) * tile * tile : 0;
}

// RELAPACK_TAIL_SPLIT=1 turns the tail split on in the plans (off by
// default: measured neutral inside the DAG, where concurrent launches already
// fill the last wave's idle SMs — n = 16384 46.78-46.81 vs 46.76-46.77 ms,
// n = 65536 2795-2796 vs 2793-2794 ms, tools/experiments/exp_tail.sh); the
// kernel tests force it through the hook either way
static bool tail_split_enabled() {
  static const bool on = [] {
    const char* v = getenv("RELAPACK_TAIL_SPLIT");
    return v && v[0] == '1';
  }();
  return on;
}

int update_tail_split(int ntiles, int K, int tile, int max_ctas, int* full_items, bool always) {
  *full_items = 0;
  if (!(always || tail_split_enabled()) || tile != 128) return 1;
  const int slots = max_ctas > 0 && max_ctas < 148 ? max_ctas : 148;  // 128-tile CTAs: one per SM
  if (ntiles <= slots) return 1;
  const int r = ntiles % slots;
  if (r == 0) return 1;
  const int KT = (K + BK - 1) / BK;
  int s = slots / r;
  s = s < 4 ? s : 4;
  while (s >= 2 && KT / s < 8) --s;
  if (s < 2) return 1;
  *full_items = ntiles - r;
  return s;
}

void init_update(UpdateOp& u, double* C, int64_t ldc, int lc, const double* A, int64_t lda, int la, const double* B,
                 int64_t ldb, int lb, int M, int N, int K, double alpha, int tri, int tile, bool allow_tma) {
  if (lc == kLayoutT && !(la == kLayoutT && lb == kLayoutT)) {
    // C^T (layout N) += alpha * B A^T
    const double* X = A;
    A = B;
    B = X;
    const int64_t lx = lda;
    lda = ldb;
    ldb = lx;
    const int l = la;
    la = lb;
    lb = l;
    const int m = M;
    M = N;
    N = m;
    tri = tri == 1 ? 2 : tri == 2 ? 1 : 0;
    lc = kLayoutN;
  }
  UpdateArgs& a = u.args;
  memset(&a, 0, sizeof(a));
  a.C = C;
  a.ldc = ldc;
  a.layout = lc;
  a.la = la;
  a.lb = lb;
  a.alpha = alpha;
  a.M = M;
  a.N = N;
  a.K = K;
  a.tri = tri;
  a.A = A;
  a.lda = lda;
  a.B = B;
  a.ldb = ldb;
  a.ksplit = 1;
  a.full_items = 0;
  u.tile = tile > 0 ? tile : update_tile_for(M, N, K, tri != 0);
  a.tiles_m = (M + u.tile - 1) / u.tile;
  const int tiles_n = (N + u.tile - 1) / u.tile;
  a.ntiles = tri ? a.tiles_m * (a.tiles_m + 1) / 2 : a.tiles_m * tiles_n;
  u.max_ctas = 0;
  u.use_tma = allow_tma && make_operand_map(&u.tmA, A, lda, la, M, K, u.tile) &&
              make_operand_map(&u.tmB, B, ldb, lb, N, K, u.tile);
}

cudaError_t configure_update() {
  cudaError_t e = configure_tbm<128>();
  if (e != cudaSuccess) return e;
  if ((e = configure_tbm<64>()) != cudaSuccess) return e;
  return configure_tbm<32>();
}

cudaError_t launch_update(const UpdateOp& op, cudaStream_t st) {
  const UpdateArgs& a = op.args;
  if (a.M <= 0 || a.N <= 0 || a.K <= 0) return cudaSuccess;
  return op.tile == 128 ? launch_tbm<128>(op, st) : op.tile == 64 ? launch_tbm<64>(op, st) : launch_tbm<32>(op, st);
}

// Host: TMA descriptor for an operand block of the L-view (rows x K) with
// box rows `box_rows` (= the CTA tile).  Layout N: dims {rows, K}, box {16, 16};
// layout T: dims {K, rows}, box {16, box_rows}.
bool make_operand_map(CUtensorMap* map, const double* base, int64_t ld, int layout, int rows, int K, int box_rows) {
  typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                    const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                    CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  static EncodeTiledFn encode = nullptr;
  if (!encode) {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || fn == nullptr)
      return false;
    encode = reinterpret_cast<EncodeTiledFn>(fn);
  }
  if ((reinterpret_cast<uintptr_t>(base) & 15) != 0 || (ld & 1) != 0 || rows <= 0 || K <= 0) return false;
  cuuint64_t dims[2];
  cuuint64_t strides[1] = {(cuuint64_t)ld * 8};
  cuuint32_t box[2];
  cuuint32_t estr[2] = {1, 1};
  if (layout == kLayoutN) {
    dims[0] = (cuuint64_t)rows;
    dims[1] = (cuuint64_t)K;
    box[0] = 16;
    box[1] = BK;
  } else {
    dims[0] = (cuuint64_t)K;
    dims[1] = (cuuint64_t)rows;
    box[0] = BK;
    box[1] = (cuuint32_t)box_rows;
  }
  CUresult r = encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(base), dims, strides, box, estr,
                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

}  // namespace relapack
