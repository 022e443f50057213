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

enum OpKind : int {
  OP_POTF2 = 0, OP_TRSM = 1, OP_GEMM = 2, OP_SYRK = 3,
  // multi-GPU steps (dist schedule only)
  OP_PACK = 10,       // gather this rank's owned rows of a block into the send buffer
  OP_ALLGATHER = 11,  // ncclAllGather(send, recv, m * k doubles per rank)
  OP_UNPACK = 12,     // scatter every rank's packed rows back into the matrix
  // host-matrix path: copies of L-view blocks between the caller's pinned host
  // matrix and the device staging buffer, captured into the same DAG
  OP_H2D = 20,        // block rows [c_i, c_i + m) x cols [c_j, c_j + k): host -> device
  OP_D2H = 21         // same block: device -> host
};

// Buffers an op can address (L-view, same layout as the matrix).
enum BufId : int { BUF_A = 0, BUF_SEND = 1, BUF_RECV = 2 };

struct PlanOp {
  OpKind kind;
  int level;       // recursion level of the potrf node issuing it (top split = 1; base = its node's level)
  // L-view coordinates (row, col) of the blocks, relative to the buffer origin
  int c_i, c_j;    // output block (POTF2: the diagonal block; TRSM: B; GEMM/SYRK: C)
  int a_i, a_j;    // operand A (TRSM: L block; GEMM/SYRK: A)
  int b_i, b_j;    // operand B (GEMM: B; SYRK: same as A)
  int m, n, k;     // POTF2: n; TRSM: m rows, k = t; GEMM: M=m, N=n, K=k; SYRK: N=n, K=k
  int info_base;   // POTF2 only
  double flops;    // leading-term algorithmic flops of this op
  int c_buf = BUF_A, a_buf = BUF_A, b_buf = BUF_A;
  int deferred = 0;  // lookahead trailing update (off the next panel's chain): low priority
  // PACK/UNPACK: rows [c_i, c_i + m) x cols [c_j, c_j + k) of the matrix,
  // block-cyclic ownership with row block nb over nranks (rows counted from 0)
  // ALLGATHER: m = rows per rank (padded), k = columns
};

struct PlanParams {
  int crossover = 64;   // c: base case when n <= c
  int split_tile = 64;  // T: n1 = T floor(n / 2T)
  int trsm_base = 64;   // t_base: TRSM base case when k <= t_base
  // lookahead: split SYRK(A22) along the child's split into SYRK(B11) +
  // GEMM(B21) + SYRK(B22), so potrf(B11) only waits for SYRK(B11) and the
  // bulk of the trailing update can run concurrently with it
  bool lookahead = false;
  // lookahead depth: the top-left part B11 of the split is itself split the
  // same way this many times (1 = one split), so the first leaf of potrf(A22)
  // waits only for the update of its own corner
  int lookahead_depth = 1;
  // lookahead GEMM(B21) as a deferred (low-priority, CTA-capped) update too
  bool defer_b21 = true;
  // GEMM(B21) issued as this many column chunks
  int b21_chunks = 1;
  // > 0: the TRSM of a node's A21 is issued as independent row panels of this
  // many rows (rows of B are independent), so the DAG can overlap the panels'
  // chains with each other and start the trailing updates of finished rows
  int trsm_rows = 0;
  // > 0 (host-matrix path): the TRSM's GEMM updates B2 -= X1 Lb^T are issued
  // as column chunks of this width, so each starts as soon as its own host
  // blocks have arrived instead of waiting for all of B2
  int host_gemm_cols = 0;
  // > 0: the blocked right-looking algorithm with this block size instead of
  // the recursive one (relapack_dpotrf_blocked)
  int blocked_nb = 0;
};

// Rectangle of an op's footprint in L-view coordinates of buffer `buf`.
struct Rect {
  int buf, r0, r1, c0, c1;  // rows [r0, r1), cols [c0, c1)
};
// Footprint of a compute op: written rect and up to two read-only rects.
void op_regions(const PlanOp& op, Rect* w, Rect* r1, Rect* r2);
// Transitively reduced dependency lists (indices of earlier ops) from
// read/write footprint overlaps; the op order itself is a valid serial order.
// If `anc` is given it receives the ancestor bitsets (ops.size() rows of
// (ops.size() + 63) / 64 words): bit i of row j set iff op i precedes op j.
void compute_deps(const std::vector<PlanOp>& ops, std::vector<std::vector<int>>& deps,
                  std::vector<uint64_t>* anc = nullptr);

int split_point(int n, int align);
void build_potrf_plan(int n, const PlanParams& p, std::vector<PlanOp>& ops);
// Append the plan of potrf on the diagonal block at `off` (order n) of BUF_A.
void append_potrf(int off, int n, int level, int info_base, const PlanParams& p, std::vector<PlanOp>& ops);
// Append the recursive TRSM  B := B L^{-T}: L = k x k diagonal block of BUF_A
// at (l_off, l_off); B = m x k block of buffer b_buf at (b_i, b_j).
void append_trsm(int l_off, int b_buf, int b_i, int b_j, int m, int k, int level, const PlanParams& p,
                 std::vector<PlanOp>& ops);
int plan_depth(int n, const PlanParams& p);
// Copy ops covering the lower triangle of the n x n L-view in column panels of
// `w` columns split into row chunks of `rows` (each block a 2-D copy; the
// w x w diagonal block of a panel goes whole).
void append_copies(int n, int w, int rows, OpKind kind, std::vector<PlanOp>& ops);

// ---- multi-GPU schedule ----
// Row-block-cyclic ownership of L-view rows, "snake" order so every rank gets
// an equal share of the lower triangle: block b = i / nb, round q = b / P,
// position p = b % P; owner = p on even rounds, P - 1 - p on odd rounds.
struct DistParams {
  int nranks = 1, rank = 0;
  int nb = 512;         // row block of the cyclic distribution
  int dist_min = 4096;  // nodes smaller than this are factored redundantly on every rank
};
inline int dist_owner_block(int b, const DistParams& d) {
  const int q = b / d.nranks, p = b % d.nranks;
  return (q & 1) ? d.nranks - 1 - p : p;
}
inline int dist_owner(int row, const DistParams& d) { return dist_owner_block(row / d.nb, d); }
// Rows of [lo, hi) owned by `rank` (count).
int dist_owned_rows(int lo, int hi, int rank, const DistParams& d);
// Build this rank's step list for the distributed factorization of order n.
// Returns the largest packed row count times the largest column count that
// any PACK/ALLGATHER uses (the send-buffer size in doubles) via *send_elems.
void build_dist_plan(int n, const PlanParams& p, const DistParams& d, std::vector<PlanOp>& ops, int64_t* send_elems,
                     int* max_rows, int* max_cols);

}  // namespace relapack
