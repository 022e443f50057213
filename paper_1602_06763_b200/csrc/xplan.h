// xplan.h — host-side plans of the other recursive operations of the paper
// (SURVEY §8(f)): the recursions of P:275-307 written out as ordered lists of
// kernel launches on views of the operands.  Host only (no CUDA calls);
// executed by xdriver.cu.
//
// Views.  Buffers are addressed in logical coordinates: buffer 0 is the
// triangular / general matrix (for the triangular operations its L-view:
// uplo 'U' works on L = U^T, as the factorization does), buffer 1 the
// right-hand sides of potrs, buffer 2 the pivot vector of getrf.  A view of
// a block at (r0, c0) is either the block itself (trans 0: view(i, j) =
// buf(r0 + i, c0 + j)) or its transpose (trans 1: view(i, j) = buf(r0 + j,
// c0 + i)).  Left-sided triangular operations are the right-sided ones on
// the transposed view of B (L X = B  <=>  X^T L^T = B^T).
#pragma once
#include <cstdint>
#include <vector>

namespace relapack {

struct XView {
  int buf = 0;
  int r0 = 0, c0 = 0;
  int trans = 0;
};

enum XKind : int {
  XK_GEMM = 0,   // C(m x n) += alpha A(m x k) B(n x k)^T on the tri part of C   [update kernel]
  XK_TRI = 1,    // rows of B(m x k) against T = a (k x k lower), mode / unit / alpha [k_tri_rows, k <= 64]
  XK_TRTI2 = 2,  // c := c^{-1}, n x n lower (n <= 64)                             [k_trti2]
  XK_LAUU2 = 3,  // c := c^T c, n x n lower (n <= 64)                              [k_lauu2]
  XK_POTF2 = 4,  // Cholesky of the n x n block (n <= 128)                        [potf2.cu]
  XK_GETF2 = 5,  // LU with partial pivoting of the m x n panel at c (n <= 32)    [k_getf2]
  XK_LASWP = 6,  // row interchanges ipiv[m .. k) on columns [c.c0, c.c0 + n)      [k_laswp]
  XK_CHECK = 7,  // info := first zero diagonal of the n x n L-view (trtri)      [k_diag_check]
  XK_PERM = 8    // pivots [k, k + m) of the panel at row c.r0 applied to columns [c.c0, c.c0 + n) [k_permute]
};

struct XOp {
  XKind kind = XK_GEMM;
  int level = 0;
  XView c, a, b;
  int m = 0, n = 0, k = 0;
  double alpha = -1.0;
  int tri = 0;    // GEMM: 0 all, 1 lower, 2 upper triangle of C (logical)
  int mode = 0;   // TRI: XTriMode
  int unit = 0;   // TRI / TRTI2: unit diagonal
  int info_base = 0;
  double flops = 0.0;  // leading-term algorithmic flops
  int defer = 0;       // 1: off the critical path (getrf lookahead pieces): low priority, capped grid
  int after = -1;      // >= 0: an extra dependency on that (earlier) op (getrf lookahead: the first piece's update)
};

struct XParams {
  int tri_base = 64;    // triangular base width (TRI / TRTI2 / LAUU2 leaves)
  int split_tile = 64;  // n1 = T floor(n / 2T)
  int getrf_base = 32;  // panel width of the getrf leaves
  int potrf_base = 128; // Cholesky leaves (blocked dpotrf's diagonal blocks)
  // getrf panels on one thread-block cluster (k_getf2_clr): cluster size (0:
  // the cooperative grid kernel k_getf2)
  int getf2_cluster = 0;
  int getrf_cols = 0;   // columns of the whole matrix (the interchanges' extent)
  int getrf_window = 256;  // lookahead plan: column windows factored with eager interchanges
  int getrf_first_piece = 0;  // lookahead plan: deferred updates of a level after its first piece's update
  // potrs: the right-hand sides in panels of this many columns, each panel its
  // own pair of recursive solves (independent chains the DAG overlaps); 0: one panel
  // (measured r7a, n = 16384, nrhs = 1024: 28.5 ms whole, 25.0 / 24.6 / 25.7 ms at 128 / 256 / 512)
  int potrs_cols = 256;
  // trtri: 0 = the paper's order (trtri(A_TL); trmm; trsm; trtri(A_BR): one chain); 1 = the solve with the
  // original A_BR first, then both recursive calls (independent in the DAG), then the trmm with A_TL^{-1}
  // (measured r7c, n = 16384: 54.6 -> 50.1 ms; DESIGN R16b)
  int trtri_order = 1;
  // trtri / lauum / getrf: the rows of a level's TRMM / TRSM operand in panels of this many rows (0: whole;
  // measured r7a: trtri 54.6 -> 59.6 / 56.1 / 54.4 ms at 512 / 1024 / 2048, lauum 49.0 -> 48.6 at 2048 — off)
  int tri_rows = 0;
};

// Recursive TRSM / TRMM on rows: B(m x k) := op(B, T) with T (k x k) lower,
// op one of XTriMode (solves need alpha = 1).
void xplan_tri(std::vector<XOp>& ops, const XParams& p, int mode, XView T, XView B, int m, int k, double alpha,
               int unit, int level);
// Recursive trtri of the n x n L-view block at (off, off)
void xplan_trtri(std::vector<XOp>& ops, const XParams& p, int off, int n, int unit, int level);
// Blocked trtri with block b: per step A10 := -A10 A00,
// A10 := A11^{-1} A10, A11 := A11^{-1}
void xplan_trtri_blocked(std::vector<XOp>& ops, const XParams& p, int n, int b, int unit);
// Recursive lauum (L^T L) of the n x n block at (off, off)
void xplan_lauum(std::vector<XOp>& ops, const XParams& p, int off, int n, int level);
// potrs: B (buffer 1, n x nrhs) := A^{-1} B with the factor L in buffer 0
void xplan_potrs(std::vector<XOp>& ops, const XParams& p, int n, int nrhs);
// Recursive getrf of the m x n block at (r0, c0) (pivots in buffer 2)
void xplan_getrf(std::vector<XOp>& ops, const XParams& p, int r0, int c0, int m, int n, int level);
// The same recursion with lookahead (needs panel-only leaves: p.getf2_cluster
// > 0 and every leaf within the cluster kernel's rows): each level's P1 laswp,
// solve and update on the right part issued as column pieces along the left
// spine of the right recursion (pieces after the first: XOp::defer), windows
// of <= p.getrf_window columns factored with eager interchanges inside them.
void xplan_getrf_la(std::vector<XOp>& ops, const XParams& p, int m, int n);

// Footprint rectangles of an op in logical buffer coordinates and the
// transitively reduced dependency lists they imply (earlier ops only).
void xplan_deps(const std::vector<XOp>& ops, int total_rows, std::vector<std::vector<int>>& deps,
                std::vector<uint64_t>* anc);

}  // namespace relapack
