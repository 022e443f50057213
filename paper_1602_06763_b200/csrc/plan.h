// plan.h — the host-side recursion driver's plan: the recursive xpotrf of
// arXiv:1602.06763 unrolled into an ordered list of kernel launches.
//
// Recursion (P:275-307 blocked->recursive, quadrant split, crossover c;
// P:366-370 / S:358-366 for Cholesky; north_star subsystem (1)):
//   potrf(A, n):  n <= c            -> POTF2(A)                       [K1]
//                 else n1 = split(n), n2 = n - n1
//                      potrf(A11, n1)
//                      trsm(L11, A21)        A21 := A21 L11^{-T}      [K5 + K3]
//                      SYRK(A22 -= A21 A21^T, lower)                  [K4]
//                      potrf(A22, n2), info offset n1
//   trsm(L, B, m, k): k <= t_base   -> TRSM_BASE(L, B)                [K5]
//                 else p = split(k), q = k - p
//                      trsm(La, B1); GEMM(B2 -= B1 Lb^T) [K3]; trsm(Lc, B2)
// Offsets are element offsets of L-view positions; the plan is built without
// any CUDA call (host-only; used for the FLOP ledger and by the executor).
#pragma once
#include <cstdint>
#include <vector>

namespace relapack {

enum OpKind : int { OP_POTF2 = 0, OP_TRSM = 1, OP_GEMM = 2, OP_SYRK = 3 };

struct PlanOp {
  OpKind kind;
  int level;       // recursion level of the potrf node issuing it (top split = 1; base = its node's level)
  // L-view coordinates (row, col) of the blocks, relative to the matrix origin
  int c_i, c_j;    // output block (POTF2: the diagonal block; TRSM: B; GEMM/SYRK: C)
  int a_i, a_j;    // operand A (TRSM: L block; GEMM/SYRK: A)
  int b_i, b_j;    // operand B (GEMM: B; SYRK: same as A)
  int m, n, k;     // POTF2: n; TRSM: m rows, k = t; GEMM: M=m, N=n, K=k; SYRK: N=n, K=k
  int info_base;   // POTF2 only
  double flops;    // leading-term algorithmic flops of this op
};

struct PlanParams {
  int crossover = 64;   // c: base case when n <= c
  int split_tile = 64;  // T: n1 = T floor(n / 2T)
  int trsm_base = 64;   // t_base: TRSM base case when k <= t_base
};

int split_point(int n, int align);
void build_potrf_plan(int n, const PlanParams& p, std::vector<PlanOp>& ops);
int plan_depth(int n, const PlanParams& p);

}  // namespace relapack
