// plan.cpp — host-only construction of the recursion plan (see plan.h).
#include "plan.h"

#include <algorithm>
#include <functional>

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

void build_trsm(int L_off, int b_buf, int B_i, int B_j, int m, int k, int level, const PlanParams& p,
                std::vector<PlanOp>& ops) {
  // L block origin is (L_off, L_off) on the diagonal of BUF_A; B block origin
  // (B_i, B_j) of buffer b_buf, m x k.
  if (m <= 0 || k <= 0) return;
  if (k <= p.trsm_base) {
    PlanOp op{};
    op.kind = OP_TRSM;
    op.level = level;
    op.c_i = B_i; op.c_j = B_j;
    op.a_i = L_off; op.a_j = L_off;
    op.m = m; op.k = k;
    op.flops = (double)m * k * k;
    op.c_buf = b_buf;
    ops.push_back(op);
    return;
  }
  const int pp = split_point(k, p.split_tile), q = k - pp;
  build_trsm(L_off, b_buf, B_i, B_j, m, pp, level, p, ops);
  const int cw = p.host_gemm_cols > 0 && q > p.host_gemm_cols ? p.host_gemm_cols : q;
  for (int c0 = 0; c0 < q; c0 += cw) {
    const int w = q - c0 < cw ? q - c0 : cw;
    PlanOp g{};
    g.kind = OP_GEMM;
    g.level = level;
    g.c_i = B_i; g.c_j = B_j + pp + c0;       // B2 (m x q), columns [c0, c0 + w)
    g.a_i = B_i; g.a_j = B_j;                 // X1 (m x p)
    g.b_i = L_off + pp + c0; g.b_j = L_off;   // Lb (q x p), rows [c0, c0 + w)
    g.m = m; g.n = w; g.k = pp;
    g.flops = 2.0 * m * w * pp;
    g.c_buf = b_buf; g.a_buf = b_buf; g.b_buf = BUF_A;
    ops.push_back(g);
  }
  build_trsm(L_off + pp, b_buf, B_i, B_j + pp, m, q, level, p, ops);
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
  if (p.trsm_rows > 0 && n2 > p.trsm_rows) {
    for (int r = 0; r < n2; r += p.trsm_rows)
      build_trsm(off, BUF_A, off + n1 + r, off, std::min(p.trsm_rows, n2 - r), n1, level + 1, p, ops);
  } else {
    build_trsm(off, BUF_A, off + n1, off, n2, n1, level + 1, p, ops);
  }
  auto syrk = [&](int r0, int nn) {
    PlanOp s{};
    s.kind = OP_SYRK;
    s.level = level + 1;
    s.c_i = r0; s.c_j = r0;
    s.a_i = r0; s.a_j = off;
    s.b_i = r0; s.b_j = off;
    s.n = nn; s.m = nn; s.k = n1;
    s.flops = (double)nn * nn * n1;
    ops.push_back(s);
  };
  if (p.lookahead && n2 > p.crossover) {
    // A22 = [B11 .; B21 B22] along the child's split: the same update in three
    // footprints, B11 first (the child's potrf(B11) depends only on it), B11
    // itself split again lookahead_depth - 1 times
    std::function<void(int, int, int)> trailing = [&](int r0, int nn, int depth) {
      if (depth == 0 || nn <= p.crossover) {
        syrk(r0, nn);
        return;
      }
      const int n1c = split_point(nn, p.split_tile), n2c = nn - n1c;
      const int r1 = r0 + n1c;
      trailing(r0, n1c, depth - 1);
      // GEMM(B21) in column chunks (b21_chunks, each a multiple of the split
      // tile): the TRSM of B21 starts on its first columns as soon as their
      // chunk is done
      const int nch = p.b21_chunks < 1 ? 1 : p.b21_chunks;
      int cw = (n1c + nch - 1) / nch;
      cw = (cw + p.split_tile - 1) / p.split_tile * p.split_tile;
      for (int c0 = 0; c0 < n1c; c0 += cw) {
        const int w = n1c - c0 < cw ? n1c - c0 : cw;
        PlanOp g{};
        g.kind = OP_GEMM;
        g.level = level + 1;
        g.c_i = r1; g.c_j = r0 + c0;   // rows of B2 x cols of B1
        g.a_i = r1; g.a_j = off;       // A21 rows of B2
        g.b_i = r0 + c0; g.b_j = off;  // A21 rows of B1
        g.m = n2c; g.n = w; g.k = n1;
        g.flops = 2.0 * n2c * w * n1;
        g.deferred = p.defer_b21 ? 1 : 0;  // the TRSM of B21 needs it: on the critical path
        ops.push_back(g);
      }
      syrk(r1, n2c);
      ops.back().deferred = 1;
    };
    trailing(off + n1, n2, p.lookahead_depth < 1 ? 1 : p.lookahead_depth);
  } else {
    syrk(off + n1, n2);
  }
  build_potrf(off + n1, n2, level + 1, info_base + n1, p, ops);
}

}  // namespace

// Blocked right-looking Cholesky (SPEC blocked_potrf S:297-305):
// per step of b columns, potrf(A11) — the base kernel when b <= c, else the
// recursive algorithm on the diagonal block (as LAPACK >= 3.6 does with
// dpotrf2) —, A21 := A21 L11^{-T} (the library's TRSM), A22 -= A21 A21^T
// (one SYRK over the whole trailing matrix, no lookahead: LAPACK's order).
void build_blocked(int n, const PlanParams& p, std::vector<PlanOp>& ops) {
  PlanParams q = p;
  q.blocked_nb = 0;
  q.lookahead = false;
  const int b = p.blocked_nb;
  for (int j = 0; j < n; j += b) {
    const int jb = std::min(b, n - j), rest = n - j - jb;
    build_potrf(j, jb, 1, j, q, ops);
    if (rest <= 0) break;
    build_trsm(j, BUF_A, j + jb, j, rest, jb, 1, q, ops);
    PlanOp s{};
    s.kind = OP_SYRK;
    s.level = 1;
    s.c_i = j + jb; s.c_j = j + jb;
    s.a_i = j + jb; s.a_j = j;
    s.b_i = j + jb; s.b_j = j;
    s.n = s.m = rest; s.k = jb;
    s.flops = (double)rest * rest * jb;
    ops.push_back(s);
  }
}

void build_potrf_plan(int n, const PlanParams& p, std::vector<PlanOp>& ops) {
  ops.clear();
  if (p.blocked_nb > 0) {
    build_blocked(n, p, ops);
    return;
  }
  build_potrf(0, n, 0, 0, p, ops);
}

void append_potrf(int off, int n, int level, int info_base, const PlanParams& p, std::vector<PlanOp>& ops) {
  build_potrf(off, n, level, info_base, p, ops);
}

void append_trsm(int l_off, int b_buf, int b_i, int b_j, int m, int k, int level, const PlanParams& p,
                 std::vector<PlanOp>& ops) {
  build_trsm(l_off, b_buf, b_i, b_j, m, k, level, p, ops);
}

// ---------------------------------------------------------------- dependencies
void op_regions(const PlanOp& op, Rect* w, Rect* r1, Rect* r2) {
  const Rect none{-1, 0, 0, 0, 0};
  constexpr int kAll = 1 << 30;
  *r1 = none;
  *r2 = none;
  switch (op.kind) {
    case OP_POTF2:
      *w = Rect{BUF_A, op.c_i, op.c_i + op.n, op.c_j, op.c_j + op.n};
      break;
    case OP_TRSM:
      *w = Rect{op.c_buf, op.c_i, op.c_i + op.m, op.c_j, op.c_j + op.k};
      *r1 = Rect{BUF_A, op.a_i, op.a_i + op.k, op.a_j, op.a_j + op.k};
      break;
    case OP_GEMM:
      *w = Rect{op.c_buf, op.c_i, op.c_i + op.m, op.c_j, op.c_j + op.n};
      *r1 = Rect{op.a_buf, op.a_i, op.a_i + op.m, op.a_j, op.a_j + op.k};
      *r2 = Rect{op.b_buf, op.b_i, op.b_i + op.n, op.b_j, op.b_j + op.k};
      break;
    case OP_SYRK:
      *w = Rect{op.c_buf, op.c_i, op.c_i + op.n, op.c_j, op.c_j + op.n};
      *r1 = Rect{op.a_buf, op.a_i, op.a_i + op.n, op.a_j, op.a_j + op.k};
      break;
    case OP_H2D:
      *w = Rect{BUF_A, op.c_i, op.c_i + op.m, op.c_j, op.c_j + op.k};
      break;
    case OP_D2H:
      *w = none;
      *r1 = Rect{BUF_A, op.c_i, op.c_i + op.m, op.c_j, op.c_j + op.k};
      break;
    case OP_PACK:  // owned rows of an A block -> the send buffer
      *w = Rect{BUF_SEND, 0, kAll, 0, kAll};
      *r1 = Rect{BUF_A, op.c_i, op.c_i + op.m, op.c_j, op.c_j + op.k};
      break;
    case OP_ALLGATHER:
      *w = Rect{BUF_RECV, 0, kAll, 0, kAll};
      *r1 = Rect{BUF_SEND, 0, kAll, 0, kAll};
      break;
    case OP_UNPACK:  // every rank's rows -> the A block
      *w = Rect{BUF_A, op.c_i, op.c_i + op.m, op.c_j, op.c_j + op.k};
      *r1 = Rect{BUF_RECV, 0, kAll, 0, kAll};
      break;
    default:  // unknown: a barrier over everything
      *w = Rect{-2, 0, 0, 0, 0};
      break;
  }
}

static bool overlap(const Rect& a, const Rect& b) {
  if (a.buf == -2 || b.buf == -2) return true;
  if (a.buf < 0 || b.buf < 0 || a.buf != b.buf) return false;
  return a.r0 < b.r1 && b.r0 < a.r1 && a.c0 < b.c1 && b.c0 < a.c1;
}

void compute_deps(const std::vector<PlanOp>& ops, std::vector<std::vector<int>>& deps,
                  std::vector<uint64_t>* anc_out) {
  const size_t n = ops.size();
  deps.assign(n, {});
  std::vector<Rect> W(n), R1(n), R2(n);
  for (size_t i = 0; i < n; ++i) op_regions(ops[i], &W[i], &R1[i], &R2[i]);
  // ancestors as bitsets (n is a few thousand at most)
  const size_t words = (n + 63) / 64;
  std::vector<uint64_t> anc(n * words, 0);
  for (size_t j = 0; j < n; ++j) {
    uint64_t* aj = &anc[j * words];
    for (size_t ii = j; ii-- > 0;) {
      if (aj[ii / 64] >> (ii % 64) & 1) continue;  // already implied
      // the packed send chunk is this rank's slot of the receive buffer (the
      // all-gather runs in place): a write to BUF_SEND also touches BUF_RECV
      auto recv_hit = [](const Rect& w, const Rect& x) { return w.buf == BUF_SEND && x.buf == BUF_RECV; };
      const bool conflict = overlap(W[ii], W[j]) || overlap(W[ii], R1[j]) || overlap(W[ii], R2[j]) ||
                            overlap(R1[ii], W[j]) || overlap(R2[ii], W[j]) || recv_hit(W[ii], W[j]) ||
                            recv_hit(W[ii], R1[j]) || recv_hit(W[ii], R2[j]) || recv_hit(W[j], W[ii]) ||
                            recv_hit(W[j], R1[ii]) || recv_hit(W[j], R2[ii]);
      if (!conflict) continue;
      deps[j].push_back((int)ii);
      const uint64_t* ai = &anc[ii * words];
      for (size_t q = 0; q < words; ++q) aj[q] |= ai[q];
      aj[ii / 64] |= uint64_t(1) << (ii % 64);
    }
  }
  if (anc_out) anc_out->swap(anc);
}

// ---------------------------------------------------------------- multi-GPU
int dist_owned_rows(int lo, int hi, int rank, const DistParams& d) {
  int cnt = 0;
  for (int b = lo / d.nb; b * d.nb < hi; ++b) {
    if (dist_owner_block(b, d) != rank) continue;
    const int r0 = b * d.nb > lo ? b * d.nb : lo;
    const int r1 = (b + 1) * d.nb < hi ? (b + 1) * d.nb : hi;
    if (r1 > r0) cnt += r1 - r0;
  }
  return cnt;
}

namespace {

struct DistCtx {
  const PlanParams& p;
  const DistParams& d;
  std::vector<PlanOp>& ops;
  int64_t send_elems = 0;
  int max_rows = 0, max_cols = 0;
};

int max_owned(int lo, int hi, const DistParams& d) {
  int m = 0;
  for (int r = 0; r < d.nranks; ++r) {
    const int c = dist_owned_rows(lo, hi, r, d);
    m = c > m ? c : m;
  }
  return m;
}

// Exchange rows [lo, hi) x cols [c0, c0 + ncols): every rank packs its owned
// rows, all-gathers, and scatters all ranks' rows back (replicating them).
void exchange_rows(DistCtx& x, int lo, int hi, int c0, int ncols, int level) {
  const int rows_max = max_owned(lo, hi, x.d);
  if (rows_max <= 0 || ncols <= 0) return;
  PlanOp pk{};
  pk.kind = OP_PACK;
  pk.level = level;
  pk.c_i = lo; pk.c_j = c0; pk.m = hi - lo; pk.k = ncols; pk.n = rows_max;
  x.ops.push_back(pk);
  PlanOp ag{};
  ag.kind = OP_ALLGATHER;
  ag.level = level;
  ag.m = rows_max; ag.k = ncols;
  x.ops.push_back(ag);
  PlanOp up = pk;
  up.kind = OP_UNPACK;
  x.ops.push_back(up);
  const int64_t e = (int64_t)rows_max * ncols;
  if (e > x.send_elems) x.send_elems = e;
  if (rows_max > x.max_rows) x.max_rows = rows_max;
  if (ncols > x.max_cols) x.max_cols = ncols;
}

void dist_potrf(DistCtx& x, int off, int n, int level, int info_base) {
  if (n <= 0) return;
  if (n < x.d.dist_min) {
    // replicated leaf: gather the block's rows (their owners hold the updated
    // values) and factor it redundantly on every rank (same info everywhere)
    if (x.d.nranks > 1) exchange_rows(x, off, off + n, off, n, level);
    build_potrf(off, n, level, info_base, x.p, x.ops);
    return;
  }
  const int n1 = split_point(n, x.p.split_tile), n2 = n - n1;
  dist_potrf(x, off, n1, level + 1, info_base);  // L11 replicated on return
  // TRSM on this rank's rows of A21, packed contiguously in the send buffer
  const int lo = off + n1, hi = off + n;
  const int own = dist_owned_rows(lo, hi, x.d.rank, x.d);
  const int rows_max = max_owned(lo, hi, x.d);
  PlanOp pk{};
  pk.kind = OP_PACK;
  pk.level = level + 1;
  pk.c_i = lo; pk.c_j = off; pk.m = n2; pk.k = n1; pk.n = rows_max;
  x.ops.push_back(pk);
  build_trsm(off, BUF_SEND, 0, 0, own, n1, level + 1, x.p, x.ops);
  PlanOp ag{};
  ag.kind = OP_ALLGATHER;
  ag.level = level + 1;
  ag.m = rows_max; ag.k = n1;
  x.ops.push_back(ag);
  PlanOp up = pk;
  up.kind = OP_UNPACK;
  x.ops.push_back(up);  // L21 replicated
  const int64_t e = (int64_t)rows_max * n1;
  if (e > x.send_elems) x.send_elems = e;
  if (rows_max > x.max_rows) x.max_rows = rows_max;
  if (n1 > x.max_cols) x.max_cols = n1;
  // SYRK on this rank's row blocks of A22: for an owned row block [r0, r1)
  // (relative to A22), C(r0:r1, 0:r0) -= L21(r0:r1) L21(0:r0)^T (GEMM) and the
  // diagonal block C(r0:r1, r0:r1) -= L21(r0:r1) L21(r0:r1)^T (SYRK).
  for (int b = lo / x.d.nb; b * x.d.nb < hi; ++b) {
    if (dist_owner_block(b, x.d) != x.d.rank) continue;
    const int g0 = b * x.d.nb > lo ? b * x.d.nb : lo;
    const int g1 = (b + 1) * x.d.nb < hi ? (b + 1) * x.d.nb : hi;
    if (g1 <= g0) continue;
    if (g0 > lo) {
      PlanOp g{};
      g.kind = OP_GEMM;
      g.level = level + 1;
      g.c_i = g0; g.c_j = lo;      // C rows [g0, g1), cols [lo, g0)
      g.a_i = g0; g.a_j = off;     // L21 rows [g0, g1)
      g.b_i = lo; g.b_j = off;     // L21 rows [lo, g0)
      g.m = g1 - g0; g.n = g0 - lo; g.k = n1;
      g.flops = 2.0 * g.m * g.n * g.k;
      x.ops.push_back(g);
    }
    // the diagonal block needs only this rank's own rows of L21: read them
    // from the packed send buffer (solved in place there), so this SYRK —
    // the local x local tiles — runs while the all-gather is in flight
    // (SURVEY §8e); the GEMM above reads other ranks' rows after the unpack
    PlanOp sy{};
    sy.kind = OP_SYRK;
    sy.level = level + 1;
    sy.c_i = g0; sy.c_j = g0;
    sy.a_buf = BUF_SEND; sy.b_buf = BUF_SEND;
    sy.a_i = dist_owned_rows(lo, g0, x.d.rank, x.d); sy.a_j = 0;
    sy.b_i = sy.a_i; sy.b_j = 0;
    sy.n = sy.m = g1 - g0; sy.k = n1;
    sy.flops = (double)sy.n * sy.n * n1;
    x.ops.push_back(sy);
  }
  dist_potrf(x, off + n1, n2, level + 1, info_base + n1);  // L22 replicated on return
}

}  // namespace

void build_dist_plan(int n, const PlanParams& p, const DistParams& d, std::vector<PlanOp>& ops, int64_t* send_elems,
                     int* max_rows, int* max_cols) {
  ops.clear();
  DistCtx x{p, d, ops};
  dist_potrf(x, 0, n, 0, 0);
  if (send_elems) *send_elems = x.send_elems;
  if (max_rows) *max_rows = x.max_rows;
  if (max_cols) *max_cols = x.max_cols;
}

void append_copies(int n, int w, int rows, OpKind kind, std::vector<PlanOp>& ops) {
  for (int j0 = 0; j0 < n; j0 += w) {
    const int jw = n - j0 < w ? n - j0 : w;
    for (int r0 = j0; r0 < n; r0 += rows) {
      PlanOp op{};
      op.kind = kind;
      op.c_i = r0;
      op.c_j = j0;
      op.m = n - r0 < rows ? n - r0 : rows;
      op.k = jw;
      ops.push_back(op);
    }
  }
}

int plan_depth(int n, const PlanParams& p) {
  if (n <= p.crossover) return 0;
  const int n1 = split_point(n, p.split_tile);
  return 1 + std::max(plan_depth(n1, p), plan_depth(n - n1, p));
}

}  // namespace relapack
