// kernels.h — launch interface between the host recursion driver (driver.cu)
// and the sm_100a kernels.  Internal to the library (not part of the C ABI).
#pragma once
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

namespace relapack {

constexpr int kMaxDevices = 64;

struct TraceRec;
// Trace slot of the launch being issued (set by the driver around each op in
// trace mode, read by the launch functions; null otherwise).
extern thread_local TraceRec* g_launch_trace;
constexpr int RELAPACK_BATCH_NMAX_ = 64;  // == RELAPACK_BATCH_NMAX in include/relapack.h

// ---- K3/K4 update (update.cu) ----
struct UpdateArgs {
  double* C;          // block (M x N) to update: C += alpha * A B^T
  int64_t ldc;
  int M, N, K;
  int layout;         // layout of C: kLayoutN / kLayoutT (element (i,j) at lv_off(layout, i, j, ld))
  int la, lb;         // layouts of A (M x K) and B (N x K); the factorization uses la = lb = layout
  double alpha;       // -1 for the factorization's C -= A B^T
  int tri;            // 1: SYRK, lower-triangular tiles only (M == N); 2: upper triangle
  int tiles_m;
  const int* d_info;  // device info flag: kernels return immediately if != 0
  const double* A;    // fallback (non-TMA) operand pointers, L-view blocks
  int64_t lda;
  const double* B;
  int64_t ldb;
  // deterministic split-K: grid = ntiles * ksplit; split s covers k-tiles
  // [s*per, (s+1)*per); partial tiles go to ws, the last CTA of a tile (per
  // counters[tile], self-resetting) sums them in split order and applies C -=.
  int ksplit;         // 1 = no split
  int ntiles;
  // tail split (ksplit > 1 and full_items > 0): tiles [0, full_items) run
  // whole, one work item each; only the last partial wave's tiles
  // [full_items, ntiles) are split ksplit ways (update_tail_split).  Work
  // items: full_items + (ntiles - full_items) * ksplit; the partials of tail
  // tile t at ws + (split * (ntiles - full_items) + t - full_items) * tile^2
  int full_items;
  double* ws;         // ksplit * (ntiles - full_items) * tile^2 doubles
  int* counters;      // ntiles ints, zero between launches
  // pointer-independent plan graph: the A / B descriptors in global memory
  // (rebased per run by the plan's first node); C / A / B above are then byte
  // offsets from the matrix base and d_info is tagged (common.cuh PlanState)
  const CUtensorMap* gmap;
};

struct UpdateOp {
  UpdateArgs args;
  CUtensorMap tmA, tmB;
  bool use_tma;
  int tile;      // CTA tile (128 or 64), see update_tile_for
  int max_ctas;  // > 0: persistent launch with at most this many CTAs
};

cudaError_t launch_update(const UpdateOp& op, cudaStream_t st);
bool make_operand_map(CUtensorMap* map, const double* base, int64_t ld, int layout, int rows, int K, int box_rows);
// Fill an UpdateOp for C(M x N) += alpha * A(M x K) * B(N x K)^T with per-operand
// layouts (tri 0 full, 1 lower, 2 upper triangle of C).  A C of layout T with
// mixed operand layouts is rewritten as C^T += alpha * B A^T (layout N, triangle
// flipped), the form the kernels are instantiated for.  tile <= 0: the size
// rule update_tile_for; allow_tma = false forces the plain-load operand path.
// ksplit stays 1 (setup by the caller).
void init_update(UpdateOp& u, double* C, int64_t ldc, int lc, const double* A, int64_t lda, int la, const double* B,
                 int64_t ldb, int lb, int M, int N, int K, double alpha, int tri, int tile = 0, bool allow_tma = true);
int update_tile_for(int M, int N, int K, int tri);
// Split-K factor for an update of (M, N, K) on `tile` x `tile` CTA tiles (1 = none)
// and the workspace it needs (doubles) — see update.cu.
// chain: the update sits on the base-case chain (non-deferred SYRK): latency
// over efficiency, down to 2 k-tiles per split
int update_ksplit_for(int M, int N, int K, int tri, int tile, bool chain = false);
int64_t update_ws_elems(int M, int N, int tri, int tile, int ksplit, int full_items = 0);
// Tail split of a big-grid update (tile 128, ntiles over several waves of
// `slots` concurrent CTAs: 148, or the launch's CTA cap): returns the split
// factor s (2..4) for the last partial wave's r tiles when r * s fits one wave
// and every piece keeps >= 8 k-tiles, with *full_items = ntiles - r; else 1.
// Plans apply it only with RELAPACK_TAIL_SPLIT=1 (measured neutral in the DAG);
// always = true ignores the knob (kernel test hook).
int update_tail_split(int ntiles, int K, int tile, int max_ctas, int* full_items, bool always = false);

// ---- K1 base-case potf2 (potf2.cu) ----
// Factor the n x n L-view block at A (n <= kPotf2Max) in shared memory; on a
// non-positive pivot at local column j write d_info = info_base + j + 1.
// n <= 128: one CTA holds the block (register / shared-memory kernels, the
// 128-node); 128 < n <= 256: the 256-node kernel (split at 128, TRSM and SYRK
// inside the CTA).
constexpr int kPotf2Max = 256;
// default crossover c of the recursion (RELAPACK_CROSSOVER / relapack_set_crossover
// override): 128 — the 256-node kernel measured slower on the chain (one SM
// does the TRSM and SYRK the separate launches spread over 4-10 SMs: n = 4096
// 2.82 vs 2.09 ms, n = 256 0.117 vs 0.105 ms; tools/experiments/exp_node256.sh)
constexpr int kCrossoverDefault = 128;
cudaError_t launch_potf2(double* A, int64_t ld, int layout, int n, int* d_info, int info_base, cudaStream_t st);

// ---- K5 base TRSM (trsm.cu): B(m x t) := B * L^{-T}, L t x t lower (t <= kTrsmMax)
constexpr int kTrsmMax = 64;
cudaError_t launch_trsm_base(const double* L, int64_t ldl, double* B, int64_t ldb, int layout, int m, int t,
                             const int* d_info, cudaStream_t st);

// ---- K5' fused TRSM base (trsm_fused.cu): t <= kTrsmFusedMax columns in one launch
constexpr int kTrsmFusedMax = 256;
cudaError_t launch_trsm_fused(const double* L, int64_t ldl, double* B, int64_t ldb, int layout, int m, int t,
                              const int* d_info, cudaStream_t st);
cudaError_t configure_trsm_fused();
cudaError_t launch_trsm_fused_variant(int v, const double* L, int64_t ldl, double* B, int64_t ldb, int layout, int m,
                                      int t, const int* d_info, cudaStream_t st);
// TRSM base dispatch (measured, profiles/): the row-parallel K5 for t <= 64 on
// short panels, the chunked DMMA K5' otherwise.
inline cudaError_t launch_trsm_any(const double* L, int64_t ldl, double* B, int64_t ldb, int layout, int m, int t,
                                   const int* d_info, cudaStream_t st) {
  return (t <= kTrsmMax && m < 2048) ? launch_trsm_base(L, ldl, B, ldb, layout, m, t, d_info, st)
                                     : launch_trsm_fused(L, ldl, B, ldb, layout, m, t, d_info, st);
}

// ---- K2 batched potf2 (batched.cu)
cudaError_t launch_potf2_batched(int layout, int batch, const int* d_n, double* const* d_A, const int* d_lda,
                                 int* d_info, cudaStream_t st);
void release_batched_workspace();

// ---- one-time per-device kernel attributes (max dynamic smem); call before graph capture
cudaError_t configure_update();
cudaError_t configure_potf2();
cudaError_t configure_trsm();
inline cudaError_t configure_kernels() {
  cudaError_t e = configure_update();
  if (e == cudaSuccess) e = configure_potf2();
  if (e == cudaSuccess) e = configure_trsm();
  if (e == cudaSuccess) e = configure_trsm_fused();
  return e;
}

// ---- misc device helpers (driver.cu)
cudaError_t launch_set_int(int* p, int v, cudaStream_t st);

}  // namespace relapack
