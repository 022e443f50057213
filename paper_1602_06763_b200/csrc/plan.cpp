// plan.cpp — host-only construction of the recursion plan (see plan.h).
#include "plan.h"

#include <algorithm>

namespace relapack {

// Split rule (P:286-292 with the footnote P:288-291 "where possible, the sizes
// of the sub-matrices are multiples of 8"; SPEC split_point S:49-58 rounds
// down; north_star "n/2 rounded to a tile multiple"; reading R1):
//   n1 = align * floor(n / (2 align))  if that is >= align
//   else 8 * floor(n / 16)             if that is >= 8   (the paper's 8-alignment)
//   else floor(n / 2).
int split_point(int n, int align) {
  if (n < 2 || align < 1) return -1;
  int n1 = align * (n / (2 * align));
  if (n1 >= align) return n1;
  if (align > 8) {
    n1 = 8 * (n / 16);
    if (n1 >= 8) return n1;
  }
  return n / 2;
}

namespace {

void build_trsm(int L_off, int B_i, int B_j, int m, int k, int level, const PlanParams& p,
                std::vector<PlanOp>& ops) {
  // L block origin is (L_off, L_off) on the diagonal; B block origin (B_i, B_j), m x k.
  if (k <= p.trsm_base) {
    PlanOp op{};
    op.kind = OP_TRSM;
    op.level = level;
    op.c_i = B_i; op.c_j = B_j;
    op.a_i = L_off; op.a_j = L_off;
    op.m = m; op.k = k;
    op.flops = (double)m * k * k;
    ops.push_back(op);
    return;
  }
  const int pp = split_point(k, p.split_tile), q = k - pp;
  build_trsm(L_off, B_i, B_j, m, pp, level, p, ops);
  PlanOp g{};
  g.kind = OP_GEMM;
  g.level = level;
  g.c_i = B_i; g.c_j = B_j + pp;       // B2 (m x q)
  g.a_i = B_i; g.a_j = B_j;            // X1 (m x p)
  g.b_i = L_off + pp; g.b_j = L_off;   // Lb (q x p)
  g.m = m; g.n = q; g.k = pp;
  g.flops = 2.0 * m * q * pp;
  ops.push_back(g);
  build_trsm(L_off + pp, B_i, B_j + pp, m, q, level, p, ops);
}

void build_potrf(int off, int n, int level, int info_base, const PlanParams& p, std::vector<PlanOp>& ops) {
  if (n <= 0) return;
  if (n <= p.crossover) {
    PlanOp op{};
    op.kind = OP_POTF2;
    op.level = level;
    op.c_i = off; op.c_j = off;
    op.n = n;
    op.info_base = info_base;
    op.flops = (double)n * n * n / 3.0;
    ops.push_back(op);
    return;
  }
  const int n1 = split_point(n, p.split_tile), n2 = n - n1;
  build_potrf(off, n1, level + 1, info_base, p, ops);
  build_trsm(off, off + n1, off, n2, n1, level + 1, p, ops);
  PlanOp s{};
  s.kind = OP_SYRK;
  s.level = level + 1;
  s.c_i = off + n1; s.c_j = off + n1;
  s.a_i = off + n1; s.a_j = off;
  s.b_i = off + n1; s.b_j = off;
  s.n = n2; s.m = n2; s.k = n1;
  s.flops = (double)n2 * n2 * n1;
  ops.push_back(s);
  build_potrf(off + n1, n2, level + 1, info_base + n1, p, ops);
}

}  // namespace

void build_potrf_plan(int n, const PlanParams& p, std::vector<PlanOp>& ops) {
  ops.clear();
  build_potrf(0, n, 0, 0, p, ops);
}

int plan_depth(int n, const PlanParams& p) {
  if (n <= p.crossover) return 0;
  const int n1 = split_point(n, p.split_tile);
  return 1 + std::max(plan_depth(n1, p), plan_depth(n - n1, p));
}

}  // namespace relapack
