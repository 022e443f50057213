// hooks.cu — kernel-level test hooks of the C ABI (include/relapack.h, "Kernel
// test hooks").  Each launches exactly one of the hot path's kernels on
// caller-provided device blocks, with the choices the plan makes by size rule
// (CTA tile, split-K, TMA or plain-load operands, TRSM variant) forced by the
// caller, so the tests can compare every instantiation the factorization runs
// with the oracle's BLAS-3 definitions (oracle_dgemm_nt / dsyrk_ln /
// dtrsm_rlt) element by element.  Synchronous; not for production.
#include <cuda_runtime.h>

#include "../../include/relapack.h"
#include "common.cuh"
#include "driver_internal.h"
#include "kernels.h"

using namespace relapack;

namespace {

struct HookScratch {
  int* d_info = nullptr;
  double* ws = nullptr;
  int* cnt = nullptr;
  ~HookScratch() {
    if (d_info) cudaFree(d_info);
    if (ws) cudaFree(ws);
    if (cnt) cudaFree(cnt);
  }
};

int finish(cudaError_t e, cudaStream_t st, const char* what) {
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  return e == cudaSuccess ? 0 : cuda_fail(e, what);
}

}  // namespace

extern "C" {

int relapack_update_test(int la, int lb, int lc, int tri, int M, int N, int K, double alpha, double* C, int64_t ldc,
                         const double* A, int64_t lda, const double* B, int64_t ldb, int tile, int ksplit,
                         int allow_tma, int max_ctas, int full_items, relapack_stream_t stream, int* chosen) {
  if (la < 0 || la > 1 || lb < 0 || lb > 1 || lc < 0 || lc > 1 || tri < 0 || tri > 2 || M < 0 || N < 0 || K < 0)
    return -1;
  if (tri && M != N) return -1;
  if (tile != 0 && tile != 32 && tile != 64 && tile != 128) return -1;
  if (ksplit < 0 || ksplit > 16 || max_ctas < 0 || full_items < 0) return -1;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  cudaError_t e = configure_kernels();
  if (e != cudaSuccess) return cuda_fail(e, "configure");
  HookScratch s;
  if ((e = cudaMalloc(&s.d_info, sizeof(int))) != cudaSuccess) return cuda_fail(e, "hook info");
  if ((e = cudaMemsetAsync(s.d_info, 0, sizeof(int), st)) != cudaSuccess) return cuda_fail(e, "hook info");
  UpdateOp u{};
  init_update(u, C, ldc, lc, A, lda, la, B, ldb, lb, M, N, K, alpha, tri, tile, allow_tma != 0);
  u.args.d_info = s.d_info;
  u.max_ctas = max_ctas;
  int ks = ksplit;
  int full = full_items;
  if (ks == 0) {
    ks = update_ksplit_for(u.args.M, u.args.N, K, u.args.tri != 0, u.tile);
    if (ks <= 1) ks = update_tail_split(u.args.ntiles, K, u.tile, max_ctas, &full, true);
  }
  if (ks > 1 && full >= u.args.ntiles) return -1;
  if (ks > 1) {
    u.args.ksplit = ks;
    u.args.full_items = full;
    const int64_t wse = update_ws_elems(u.args.M, u.args.N, u.args.tri != 0, u.tile, ks, full);
    if ((e = cudaMalloc(&s.ws, wse * sizeof(double))) != cudaSuccess) return cuda_fail(e, "hook ws");
    if ((e = cudaMalloc(&s.cnt, u.args.ntiles * sizeof(int))) != cudaSuccess) return cuda_fail(e, "hook cnt");
    if ((e = cudaMemsetAsync(s.cnt, 0, u.args.ntiles * sizeof(int), st)) != cudaSuccess) return cuda_fail(e, "cnt");
    u.args.ws = s.ws;
    u.args.counters = s.cnt;
  }
  if (chosen) {
    chosen[0] = u.tile;
    chosen[1] = u.use_tma ? 1 : 0;
    chosen[2] = u.args.ksplit;
  }
  return finish(launch_update(u, st), st, "update hook");
}

int relapack_trsm_test(int layout, int m, int t, const double* L, int64_t ldl, double* B, int64_t ldb, int variant,
                       relapack_stream_t stream) {
  if (layout < 0 || layout > 1 || m < 0 || t < 0 || variant < 0 || variant > 6) return -1;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  cudaError_t e = configure_kernels();
  if (e != cudaSuccess) return cuda_fail(e, "configure");
  HookScratch s;
  if ((e = cudaMalloc(&s.d_info, sizeof(int))) != cudaSuccess) return cuda_fail(e, "hook info");
  if ((e = cudaMemsetAsync(s.d_info, 0, sizeof(int), st)) != cudaSuccess) return cuda_fail(e, "hook info");
  if (variant == 0)
    e = launch_trsm_any(L, ldl, B, ldb, layout, m, t, s.d_info, st);
  else if (variant == 6)
    e = launch_trsm_base(L, ldl, B, ldb, layout, m, t, s.d_info, st);
  else
    e = launch_trsm_fused_variant(variant, L, ldl, B, ldb, layout, m, t, s.d_info, st);
  return finish(e, st, "trsm hook");
}

int relapack_potf2_test(int layout, int n, double* A, int64_t lda, int* info, relapack_stream_t stream) {
  if (layout < 0 || layout > 1 || n < 0 || n > kPotf2Max || !info) return -1;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  cudaError_t e = configure_kernels();
  if (e != cudaSuccess) return cuda_fail(e, "configure");
  HookScratch s;
  if ((e = cudaMalloc(&s.d_info, sizeof(int))) != cudaSuccess) return cuda_fail(e, "hook info");
  if ((e = cudaMemsetAsync(s.d_info, 0, sizeof(int), st)) != cudaSuccess) return cuda_fail(e, "hook info");
  if ((e = launch_potf2(A, lda, layout, n, s.d_info, 0, st)) != cudaSuccess) return cuda_fail(e, "potf2 hook");
  if ((e = cudaMemcpyAsync(info, s.d_info, sizeof(int), cudaMemcpyDeviceToHost, st)) != cudaSuccess)
    return cuda_fail(e, "potf2 hook");
  return finish(cudaSuccess, st, "potf2 hook");
}

}  // extern "C"
