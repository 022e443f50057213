// xplan.cpp — the recursions of SURVEY §8(f) as launch lists (see xplan.h).
#include "xplan.h"

#include <algorithm>

#include "plan.h"
#include "xkernels.h"

namespace relapack {

namespace {

XView sub(XView v, int i, int j) {  // logical block (i, j) of a view
  if (v.trans) {
    v.r0 += j;
    v.c0 += i;
  } else {
    v.r0 += i;
    v.c0 += j;
  }
  return v;
}

XView tr(XView v) {
  v.trans ^= 1;
  return v;
}

void gemm(std::vector<XOp>& ops, XView c, XView a, XView b, int m, int n, int k, double alpha, int tri, int level) {
  if (m <= 0 || n <= 0 || k <= 0) return;
  XOp g;
  g.kind = XK_GEMM;
  g.level = level;
  g.c = c;
  g.a = a;
  g.b = b;
  g.m = m;
  g.n = n;
  g.k = k;
  g.alpha = alpha;
  g.tri = tri;
  g.flops = tri ? (double)n * n * k : 2.0 * m * n * k;
  ops.push_back(g);
}

int xsplit(int n, int T) {
  const int s = split_point(n, T);
  return s > 0 ? s : n / 2;
}

// xplan_tri on row panels of B: the rows of B(m x k) := op(B, T) do not depend
// on one another, so each panel is its own chain of leaves and updates
// (footprint-disjoint: the DAG runs one panel's leaves under another's GEMMs).
void tri_panels(std::vector<XOp>& ops, const XParams& p, int rows, int mode, XView T, XView B, int m, int k,
                double alpha, int unit, int level) {
  if (rows <= 0 || m <= rows + rows / 2) {
    xplan_tri(ops, p, mode, T, B, m, k, alpha, unit, level);
    return;
  }
  const int np = (m + rows - 1) / rows;
  for (int q = 0; q < np; ++q) {
    const int r0 = (int)((int64_t)m * q / np / 8 * 8), r1 = q + 1 == np ? m : (int)((int64_t)m * (q + 1) / np / 8 * 8);
    xplan_tri(ops, p, mode, T, sub(B, r0, 0), r1 - r0, k, alpha, unit, level);
  }
}

}  // namespace

void xplan_tri(std::vector<XOp>& ops, const XParams& p, int mode, XView T, XView B, int m, int k, double alpha,
               int unit, int level) {
  if (m <= 0 || k <= 0) return;
  if (k <= p.tri_base) {
    XOp o;
    o.kind = XK_TRI;
    o.level = level;
    o.c = B;
    o.a = T;
    o.m = m;
    o.k = k;
    o.mode = mode;
    o.unit = unit;
    o.alpha = alpha;
    o.flops = (double)m * k * k;
    ops.push_back(o);
    return;
  }
  const int s = xsplit(k, p.split_tile), q = k - s;
  const XView T11 = T, T21 = sub(T, s, 0), T22 = sub(T, s, s);
  const XView B1 = B, B2 = sub(B, 0, s);
  switch (mode) {
    case kTriSolveLT:  // X1 = B1 T11^-T; B2 -= X1 T21^T; X2 = B2 T22^-T
      xplan_tri(ops, p, mode, T11, B1, m, s, alpha, unit, level);
      gemm(ops, B2, B1, T21, m, q, s, -1.0, 0, level);
      xplan_tri(ops, p, mode, T22, B2, m, q, 1.0, unit, level);
      break;
    case kTriSolveL:  // X2 = B2 T22^-1; B1 -= X2 T21; X1 = B1 T11^-1
      xplan_tri(ops, p, mode, T22, B2, m, q, alpha, unit, level);
      gemm(ops, B1, B2, tr(T21), m, s, q, -1.0, 0, level);
      xplan_tri(ops, p, mode, T11, B1, m, s, 1.0, unit, level);
      break;
    case kTriMulL:  // Y1 = a (B1 T11 + B2 T21); Y2 = a B2 T22
      xplan_tri(ops, p, mode, T11, B1, m, s, alpha, unit, level);
      gemm(ops, B1, B2, tr(T21), m, s, q, alpha, 0, level);
      xplan_tri(ops, p, mode, T22, B2, m, q, alpha, unit, level);
      break;
    default:  // kTriMulLT: Y2 = a (B2 T22^T + B1 T21^T); Y1 = a B1 T11^T
      xplan_tri(ops, p, mode, T22, B2, m, q, alpha, unit, level);
      gemm(ops, B2, B1, T21, m, q, s, alpha, 0, level);
      xplan_tri(ops, p, mode, T11, B1, m, s, alpha, unit, level);
      break;
  }
}

void xplan_trtri(std::vector<XOp>& ops, const XParams& p, int off, int n, int unit, int level) {
  if (n <= 0) return;
  if (n <= p.tri_base) {
    XOp o;
    o.kind = XK_TRTI2;
    o.level = level;
    o.c = XView{0, off, off, 0};
    o.n = n;
    o.unit = unit;
    o.flops = (double)n * n * n / 3.0;
    ops.push_back(o);
    return;
  }
  // invert A_TL, two BLAS-3 calls on A_BL, invert A_BR; SPEC
  // rec_trtri S:348-357: A_BL := A_BL A_TL^{-1} (trmm), A_BL := -A_BR^{-1} A_BL
  // (trsm, the stable form the paper keeps) — the sign goes into
  // the trmm so the solve runs with alpha = 1
  const int s = xsplit(n, p.split_tile), q = n - s;
  const XView A11{0, off, off, 0}, A21{0, off + s, off, 0}, A22{0, off + s, off + s, 0};
  if (p.trtri_order == 1) {
    // -A_BR^{-1} A_BL A_TL^{-1} with the solve first: A_BL := A_BR^{-1} A_BL needs only the original
    // A_BR, so trtri(A_TL) and [solve; trtri(A_BR)] share no footprint and run side by side; the trmm
    // with the inverted A_TL closes the level (same two BLAS-3 kinds as the paper's form)
    tri_panels(ops, p, p.tri_rows, kTriSolveLT, A22, tr(A21), s, q, 1.0, unit, level + 1);
    xplan_trtri(ops, p, off, s, unit, level + 1);
    xplan_trtri(ops, p, off + s, q, unit, level + 1);
    tri_panels(ops, p, p.tri_rows, kTriMulL, A11, A21, q, s, -1.0, unit, level + 1);
    return;
  }
  xplan_trtri(ops, p, off, s, unit, level + 1);
  tri_panels(ops, p, p.tri_rows, kTriMulL, A11, A21, q, s, -1.0, unit, level + 1);
  tri_panels(ops, p, p.tri_rows, kTriSolveLT, A22, tr(A21), s, q, 1.0, unit, level + 1);
  xplan_trtri(ops, p, off + s, q, unit, level + 1);
}

void xplan_trtri_blocked(std::vector<XOp>& ops, const XParams& p, int n, int b, int unit) {
  for (int j = 0; j < n; j += b) {
    const int jb = std::min(b, n - j);
    if (j > 0) {
      const XView A00{0, 0, 0, 0}, A10{0, j, 0, 0}, A11{0, j, j, 0};
      xplan_tri(ops, p, kTriMulL, A00, A10, jb, j, -1.0, unit, 1);   // A10 := -A10 A00 (A00 inverted)
      xplan_tri(ops, p, kTriSolveLT, A11, tr(A10), j, jb, 1.0, unit, 1);  // A10 := A11^{-1} A10
    }
    xplan_trtri(ops, p, j, jb, unit, 2);  // A11 := A11^{-1} (the unblocked kernel for jb <= 64)
  }
}

void xplan_lauum(std::vector<XOp>& ops, const XParams& p, int off, int n, int level) {
  if (n <= 0) return;
  if (n <= p.tri_base) {
    XOp o;
    o.kind = XK_LAUU2;
    o.level = level;
    o.c = XView{0, off, off, 0};
    o.n = n;
    o.flops = (double)n * n * n / 3.0;
    ops.push_back(o);
    return;
  }
  // lauum(A_TL); A_TL += A_BL^T A_BL (syrk); A_BL := A_BR^T A_BL (trmm); lauum(A_BR)
  const int s = xsplit(n, p.split_tile), q = n - s;
  const XView A11{0, off, off, 0}, A21{0, off + s, off, 0}, A22{0, off + s, off + s, 0};
  xplan_lauum(ops, p, off, s, level + 1);
  gemm(ops, A11, tr(A21), tr(A21), s, s, q, 1.0, 1, level + 1);
  tri_panels(ops, p, p.tri_rows, kTriMulL, A22, tr(A21), s, q, 1.0, 0, level + 1);
  xplan_lauum(ops, p, off + s, q, level + 1);
}

void xplan_potrs(std::vector<XOp>& ops, const XParams& p, int n, int nrhs) {
  const XView L{0, 0, 0, 0}, Bt{1, 0, 0, 1};
  // every column panel of B runs both solves on its own (a panel's second solve
  // follows its first; nothing orders two panels)
  const int cols = p.potrs_cols, np = cols > 0 && nrhs > cols + cols / 2 ? (nrhs + cols - 1) / cols : 1;
  for (int q = 0; q < np; ++q) {
    const int c0 = (int)((int64_t)nrhs * q / np / 8 * 8), c1 = q + 1 == np ? nrhs : (int)((int64_t)nrhs * (q + 1) / np / 8 * 8);
    const XView Bq = sub(Bt, c0, 0);
    xplan_tri(ops, p, kTriSolveLT, L, Bq, c1 - c0, n, 1.0, 0, 1);  // L Y = B    <=> Y^T L^T = B^T
    xplan_tri(ops, p, kTriSolveL, L, Bq, c1 - c0, n, 1.0, 0, 1);   // L^T X = Y  <=> X^T L = Y^T
  }
}

// Panel width of a getrf leaf with m rows on a cluster: the configured width,
// narrowed to what the register panels hold (rows per CTA: <= 512 at 32
// columns, <= 1024 at 16, <= 2048 at 8); 0: the cooperative grid kernel.
static int cluster_leaf_width(const XParams& p, int m) {
  if (p.getf2_cluster <= 0) return 0;
  const int rows = (m + p.getf2_cluster - 1) / p.getf2_cluster;
  const int cap = rows <= kGetf2ClRows32 ? 32 : rows <= kGetf2ClRows16 ? 16 : rows <= kGetf2ClRows8 ? 8 : 0;
  return std::min(cap, p.getrf_base);
}

namespace {
// The recursion with the interchanges of a panel-only (cluster) leaf applied
// at once to the columns [zlo, zhi) of the matrix outside the leaf
// (xplan_getrf: the whole matrix; the lookahead plan: its window).
void getrf_rec(std::vector<XOp>& ops, const XParams& p, int r0, int c0, int m, int n, int level, int zlo, int zhi) {
  if (m <= 0 || n <= 0) return;
  const int mn = std::min(m, n);
  const int wcl = cluster_leaf_width(p, m);
  const int base = wcl > 0 ? wcl : p.getrf_base;
  if (n <= base) {
    XOp o;
    o.kind = XK_GETF2;
    o.level = level;
    o.c = XView{0, r0, c0, 0};
    o.m = m;
    o.n = n;
    o.mode = wcl > 0 ? 1 : 0;  // 1: cluster panel (panel columns only)
    o.info_base = c0;
    o.flops = (double)m * n * n - (double)n * n * n / 3.0;
    ops.push_back(o);
    if (o.mode == 1) {
      // the panel's interchanges in the other columns: the right part first
      // (its solve and update read those rows), the left part off the path
      const int npiv = std::min(m, n);
      for (int side = 0; side < 2; ++side) {
        XOp q;
        q.kind = XK_PERM;
        q.level = level;
        q.c = side == 0 ? XView{0, r0, c0 + n, 0} : XView{0, r0, zlo, 0};
        q.n = side == 0 ? zhi - (c0 + n) : c0 - zlo;
        q.m = npiv;
        q.k = c0;
        if (q.n > 0) ops.push_back(q);
      }
    }
    return;
  }
  // split the columns at n1; getrf(left panel) -> P1; laswp P1 on
  // the right panel; A12 := L11^{-1} A12 (unit); A22 -= A21 A12; getrf(A22)
  // -> P2; laswp P2 on the left panel's lower rows.
  // The interchanges of a panel are applied to every other column of the
  // matrix right after the panel (k_permute; the cooperative kernel k_getf2
  // does it itself), which is what the two laswp calls of the recursion do (P1
  // on the right part before its solve and update, P2 on the left part's
  // lower rows after the right recursion): nothing reads those rows of the
  // other columns in between, so the order does not matter.
  const int n1 = mn <= base ? mn : xsplit(mn, base);
  getrf_rec(ops, p, r0, c0, m, n1, level + 1, zlo, zhi);
  const XView L11{0, r0, c0, 0}, A12{0, r0, c0 + n1, 0}, A21{0, r0 + n1, c0, 0}, A22{0, r0 + n1, c0 + n1, 0};
  tri_panels(ops, p, p.tri_rows, kTriSolveLT, L11, tr(A12), n - n1, n1, 1.0, 1, level + 1);
  gemm(ops, A22, A21, tr(A12), m - n1, n - n1, n1, -1.0, 0, level + 1);
  getrf_rec(ops, p, r0 + n1, c0 + n1, m - n1, n - n1, level + 1, zlo, zhi);
}

XOp laswp(int c0, int ncols, int k0, int k1, int level) {
  XOp q;
  q.kind = XK_LASWP;
  q.level = level;
  q.c = XView{0, 0, c0, 0};
  q.n = ncols;
  q.m = k0;
  q.k = k1;
  return q;
}

// Lookahead recursion (xplan_getrf_la): S:367-375 with the two laswp calls
// of each level kept where the recursion puts them (P1 on the right part
// before its solve, P2 on the left part after the right recursion), and the
// right part's laswp / solve / update issued as column pieces along the left
// spine of the right recursion — its first window only waits for the first
// piece, the later pieces (deferred) overlap the windows before them.
void getrf_la(std::vector<XOp>& ops, const XParams& p, int r0, int c0, int m, int n, int level) {
  if (m <= 0 || n <= 0) return;
  const int W = p.getrf_window, mn = std::min(m, n);
  if (n <= W || mn <= W) {
    getrf_rec(ops, p, r0, c0, m, n, level, c0, c0 + n);  // a window: eager interchanges inside it
    return;
  }
  const int wcl = cluster_leaf_width(p, m);
  const int base = wcl > 0 ? wcl : p.getrf_base;
  const int n1 = xsplit(mn, base);
  getrf_la(ops, p, r0, c0, m, n1, level + 1);
  const int M = m - n1, wR = n - n1;
  // piece bounds (offsets into the right part): the left spine of getrf_la(M, wR)
  std::vector<int> cuts{wR};
  for (int w = wR; w > W && std::min(M, w) > W;) {
    const int wb = cluster_leaf_width(p, M), bb = wb > 0 ? wb : p.getrf_base;
    w = xsplit(std::min(M, w), bb);
    cuts.push_back(w);
  }
  cuts.push_back(0);
  std::reverse(cuts.begin(), cuts.end());
  const XView L11{0, r0, c0, 0}, A21{0, r0 + n1, c0, 0};
  int first_update = -1;
  for (size_t i = 0; i + 1 < cuts.size(); ++i) {
    const int a = cuts[i], w = cuts[i + 1] - a;
    const size_t first = ops.size();
    ops.push_back(laswp(c0 + n1 + a, w, c0, c0 + n1, level + 1));  // P1 on the piece
    const XView A12{0, r0, c0 + n1 + a, 0}, A22{0, r0 + n1, c0 + n1 + a, 0};
    xplan_tri(ops, p, kTriSolveLT, L11, tr(A12), w, n1, 1.0, 1, level + 1);
    gemm(ops, A22, A21, tr(A12), M, w, n1, -1.0, 0, level + 1);
    if (i == 0 && ops.size() > first && ops.back().kind == XK_GEMM) first_update = (int)ops.size() - 1;
    if (i > 0)
      for (size_t q = first; q < ops.size(); ++q) {
        ops[q].defer = 1;
        if (ops[q].kind == XK_GEMM && p.getrf_first_piece) ops[q].after = first_update;
      }
  }
  getrf_la(ops, p, r0 + n1, c0 + n1, M, wR, level + 1);
  if (mn > n1) ops.push_back(laswp(c0, n1, c0 + n1, c0 + mn, level + 1));  // P2 on the left part
}

}  // namespace

void xplan_getrf(std::vector<XOp>& ops, const XParams& p, int r0, int c0, int m, int n, int level) {
  getrf_rec(ops, p, r0, c0, m, n, level, 0, p.getrf_cols);
}

void xplan_getrf_la(std::vector<XOp>& ops, const XParams& p, int m, int n) {
  getrf_la(ops, p, 0, 0, m, n, 0);
}

// ------------------------------------------------------------------ dependencies
namespace {

struct XRect {
  int buf, r0, r1, c0, c1;
};

XRect rect(XView v, int rows, int cols) {
  if (v.trans) return XRect{v.buf, v.r0, v.r0 + cols, v.c0, v.c0 + rows};
  return XRect{v.buf, v.r0, v.r0 + rows, v.c0, v.c0 + cols};
}

bool hit(const XRect& a, const XRect& b) {
  if (a.buf == -2 || b.buf == -2) return true;
  if (a.buf < 0 || b.buf < 0 || a.buf != b.buf) return false;
  return a.r0 < b.r1 && b.r0 < a.r1 && a.c0 < b.c1 && b.c0 < a.c1;
}

void footprint(const XOp& o, int total_rows, XRect* w, XRect* r) {
  const XRect none{-1, 0, 0, 0, 0};
  for (int i = 0; i < 2; ++i) w[i] = r[i] = none;
  switch (o.kind) {
    case XK_GEMM:
      w[0] = rect(o.c, o.m, o.n);
      r[0] = rect(o.a, o.m, o.k);
      r[1] = rect(o.b, o.n, o.k);
      break;
    case XK_TRI:
      w[0] = rect(o.c, o.m, o.k);
      r[0] = rect(o.a, o.k, o.k);
      break;
    case XK_TRTI2:
    case XK_LAUU2:
    case XK_POTF2:
      w[0] = rect(o.c, o.n, o.n);
      break;
    case XK_GETF2:  // the panel (mode 1) or also its interchanges in every other column: rows [r0, m) of the matrix
      w[0] = o.mode == 1 ? XRect{o.c.buf, o.c.r0, total_rows, o.c.c0, o.c.c0 + o.n}
                         : XRect{o.c.buf, o.c.r0, total_rows, 0, 1 << 30};
      w[1] = XRect{2, 0, 1, o.c.c0, o.c.c0 + std::min(o.m, o.n)};  // its pivots
      break;
    case XK_PERM:
      w[0] = XRect{o.c.buf, o.c.r0, total_rows, o.c.c0, o.c.c0 + o.n};
      r[0] = XRect{2, 0, 1, o.k, o.k + o.m};
      break;
    case XK_LASWP:
      // interchanges rows >= m among the columns; reads the pivots [m, k)
      w[0] = XRect{o.c.buf, o.m, total_rows, o.c.c0, o.c.c0 + o.n};
      r[0] = XRect{2, 0, 1, o.m, o.k};
      break;
    case XK_CHECK:
      w[0] = XRect{-2, 0, 0, 0, 0};  // before everything
      break;
  }
}

}  // namespace

void xplan_deps(const std::vector<XOp>& ops, int total_rows, std::vector<std::vector<int>>& deps,
                std::vector<uint64_t>* anc_out) {
  const size_t n = ops.size();
  deps.assign(n, {});
  std::vector<XRect> W(2 * n), R(2 * n);
  for (size_t i = 0; i < n; ++i) footprint(ops[i], total_rows, &W[2 * i], &R[2 * i]);
  const size_t words = (n + 63) / 64;
  std::vector<uint64_t> anc(n * words, 0);
  for (size_t j = 0; j < n; ++j) {
    uint64_t* aj = &anc[j * words];
    for (size_t ii = j; ii-- > 0;) {
      if (aj[ii / 64] >> (ii % 64) & 1) continue;
      bool conflict = false;
      for (int x = 0; x < 2 && !conflict; ++x)
        for (int y = 0; y < 2 && !conflict; ++y)
          conflict = hit(W[2 * ii + x], W[2 * j + y]) || hit(W[2 * ii + x], R[2 * j + y]) ||
                     hit(R[2 * ii + x], W[2 * j + y]);
      if (!conflict) continue;
      deps[j].push_back((int)ii);
      const uint64_t* ai = &anc[ii * words];
      for (size_t q = 0; q < words; ++q) aj[q] |= ai[q];
      aj[ii / 64] |= uint64_t(1) << (ii % 64);
    }
  }
  if (anc_out) anc_out->swap(anc);
}

}  // namespace relapack
