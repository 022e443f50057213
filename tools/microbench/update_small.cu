// Latency of small update launches (the SYRK/GEMM shapes on the n = 4096
// critical path), graph-replayed back to back, with and without split-K.
#include <cstdio>
#include <cstring>
#include <vector>
#include "../../paper_1602_06763_b200/csrc/update.cu"
namespace relapack {
thread_local TraceRec* g_launch_trace = nullptr;
}
using namespace relapack;

static UpdateOp make(double* A, int64_t ld, int M, int N, int K, int tri, const int* info, double* ws, int* cnt,
                     int ks_force, int tile_force = 0) {
  UpdateOp u{};
  UpdateArgs& a = u.args;
  memset(&a, 0, sizeof(a));
  // C at rows/cols [K, K+M), A/B = columns [0, K) of the same rows
  a.C = A + K + (int64_t)K * ld;
  a.ldc = ld;
  a.layout = kLayoutN;
  a.d_info = info;
  a.K = K;
  a.M = M;
  a.N = N;
  a.tri = tri;
  u.tile = tile_force ? tile_force : update_tile_for(M, N, K, tri);
  a.tiles_m = (M + u.tile - 1) / u.tile;
  const int tn = (N + u.tile - 1) / u.tile;
  a.ntiles = tri ? a.tiles_m * (a.tiles_m + 1) / 2 : a.tiles_m * tn;
  a.A = A + K;
  a.lda = ld;
  a.B = A + K;
  a.ldb = ld;
  a.ksplit = ks_force > 0 ? ks_force : update_ksplit_for(M, N, K, tri, u.tile);
  a.ws = ws;
  a.counters = cnt;
  u.use_tma = make_operand_map(&u.tmA, a.A, ld, kLayoutN, M, K, u.tile) &&
              make_operand_map(&u.tmB, a.B, ld, kLayoutN, N, K, u.tile);
  return u;
}

int main() {
  const int n = 4096;
  double* A;
  cudaMalloc(&A, (size_t)n * n * 8);
  cudaMemset(A, 0, (size_t)n * n * 8);
  int* info;
  cudaMalloc(&info, 4);
  cudaMemset(info, 0, 4);
  double* ws;
  cudaMalloc(&ws, 64ull << 20);
  int* cnt;
  cudaMalloc(&cnt, 1 << 16);
  cudaMemset(cnt, 0, 1 << 16);
  configure_update();
  cudaStream_t st;
  cudaStreamCreate(&st);
  struct Shape { int M, N, K, tri; } shapes[] = {{128, 128, 128, 1}, {128, 128, 256, 1}, {256, 256, 512, 1},
                                                {512, 512, 1024, 1}, {1024, 1024, 2048, 1}, {128, 128, 128, 0},
                                                {2048, 128, 128, 0}, {512, 512, 512, 0}, {1024, 1024, 2048, 0}, {2048, 1024, 1024, 0}};
  for (auto sh : shapes)
  for (int tf : {0, 32, 64, 128}) {
    if (tf && sh.M < 2 * tf) continue;
    for (int ksf : {0, 1, 2, 4, 8, 16}) {
      UpdateOp u = make(A, n, sh.M, sh.N, sh.K, sh.tri, info, ws, cnt, ksf, tf);
      if (tf && ksf == 0) continue;
      if ((sh.K + 15) / 16 < 2 * u.args.ksplit) continue;
      if (u.args.ksplit > 1 && (int64_t)u.args.ksplit * u.args.ntiles * u.tile * u.tile * 8 > (64ll << 20)) continue;
      cudaGraph_t g;
      cudaGraphExec_t ge;
      cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal);
      for (int r = 0; r < 20; ++r) launch_update(u, st);
      cudaStreamEndCapture(st, &g);
      cudaGraphInstantiate(&ge, g, 0);
      cudaGraphLaunch(ge, st);
      cudaStreamSynchronize(st);
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      cudaEventRecord(a, st);
      for (int r = 0; r < 10; ++r) cudaGraphLaunch(ge, st);
      cudaEventRecord(b, st);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      const double fl = sh.tri ? (double)sh.N * sh.N * sh.K : 2.0 * sh.M * sh.N * sh.K;
      printf("%s M=%4d N=%4d K=%4d tile=%3d%s ksplit=%2d%s: %7.2f us/launch  %6.2f TF/s (%s)\n", sh.tri ? "syrk" : "gemm",
             sh.M, sh.N, sh.K, u.tile, tf ? "f" : " ", u.args.ksplit, ksf == 0 ? " (auto)" : "", ms * 1e3 / 200,
             fl / (ms * 1e-3 / 200) / 1e12, cudaGetErrorString(cudaGetLastError()));
      cudaGraphExecDestroy(ge);
      cudaGraphDestroy(g);
    }
  }
  return 0;
}
