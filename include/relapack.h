/*
 * relapack.h — C ABI of the B200-native recursive FP64 Cholesky (xpotrf) of
 * Peise & Bientinesi, "Recursive Algorithms for Dense Linear Algebra: The
 * ReLAPACK Collection", arXiv:1602.06763.
 *
 * Citation convention: P:a-b = PAPER.md lines a-b, S:a-b =
 * SPEC.md lines a-b of the reference text.
 *
 * The operation.  For a symmetric positive definite A (only the `uplo`
 * triangle is read) compute, in place, the lower factor L with A = L L^T
 * (uplo 'L') or the upper factor U with A = U^T U (uplo 'U', U = L^T).  The
 * method is the recursive algorithm of P:275-307 (blocked -> recursive with
 * b = n/2, quadrant split, "two BLAS-3 invocations surrounded by two
 * recursive applications", crossover size c) applied to Cholesky as in
 * LAPACK's dpotrf2 and SPEC rec_potrf:
 *     potrf(A11); A21 := A21 L11^{-T} (recursive TRSM);
 *     A22 := A22 - A21 A21^T (SYRK, lower triangle only); potrf(A22).
 * The call mirrors LAPACK xPOTRF(UPLO, N, A, LDA, INFO) as north_star asks.
 *
 * Storage.  Column-major FP64, element (i, j) at A[i + j*lda].
 * Only the `uplo` triangle (diagonal included) is read or written; the
 * opposite strict triangle and rows n..lda-1 are bitwise untouched.
 *
 * Errors (LAPACK info convention; no printing, no abort):
 *   info = 0    success
 *   info = -1   uplo not one of 'L','l','U','u'
 *   info = -2   n < 0
 *   info = -3   A is NULL while n > 0 (extension)
 *   info = -4   lda < max(1, n)
 *   info = k>0  the leading minor of order k is not positive definite: the
 *               k-th pivot d satisfied !(d > 0) (d <= 0 or NaN).  The
 *               factorization stops there (dpotrf2 semantics):
 *               the leading (k-1) x (k-1) block holds the factor of the
 *               leading minor of order k-1; every later update is skipped and
 *               the rest of the triangle is unspecified.
 *   info <= -1000  CUDA runtime failure; relapack_last_error() describes it.
 *
 * Threading / streams.  Entry points are reentrant; the per-device plan
 * cache (captured CUDA graphs) is mutex-guarded.  Work is ordered on the
 * stream set by relapack_set_stream — a per-thread setting (default: the
 * legacy default stream), so concurrent threads never redirect each other's
 * calls — or passed explicitly to the _async / _batched variants.
 *
 * Ownership.  The caller owns every matrix buffer; the library never frees
 * caller memory.  The library owns per-device workspace (info scalars,
 * staging buffer for host matrices, captured graphs, TMA descriptors),
 * released by relapack_finalize().
 */
#ifndef RELAPACK_B200_H_
#define RELAPACK_B200_H_

#include <stdint.h>

#if defined(__GNUC__)
#define RELAPACK_API __attribute__((visibility("default")))
#else
#define RELAPACK_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

/* A CUDA stream handle (cudaStream_t) passed as an opaque pointer so that this
 * header does not require the CUDA headers.  NULL = legacy default stream. */
typedef void* relapack_stream_t;

/*
 * relapack_dpotrf — synchronous LAPACK-style entry point (north_star; P:226-229
 * "conforming to the established interfaces").
 *   uplo  in   'L' or 'U' (case-insensitive)
 *   n     in   order of A, n >= 0
 *   A     in/out  DEVICE or HOST pointer to the lda x n column-major matrix.
 *               Device memory (cudaMalloc / PyTorch storage) is factored in
 *               place.  Host memory (pageable or pinned) is staged through a
 *               library-owned device buffer: the uplo triangle is copied in
 *               (whole diagonal blocks, whose other-triangle values are never
 *               used), factored on the GPU and copied back.  Pageable: only
 *               the uplo triangle is written back.  Pinned: the copies are
 *               2-D blocks overlapped with the factorization, and the 512 x
 *               512 diagonal blocks go back whole, so the other strict
 *               triangle inside them is rewritten with the values it held at
 *               the call (its contents never change, but the caller must not
 *               modify them concurrently).
 *   lda   in   leading dimension, lda >= max(1, n)
 *   info  out  host int, see "Errors" above
 * Returns after the factorization completed (stream synchronised).
 */
RELAPACK_API void relapack_dpotrf(const char* uplo, const int* n, double* A, const int* lda, int* info);

/*
 * relapack_dpotrf_async — device-only, stream-ordered variant.
 *   A       DEVICE pointer (lda x n, column-major)
 *   d_info  DEVICE int written with the info value when the work completes
 *   stream  CUDA stream the work is ordered on
 * Returns the argument-check code immediately (0, -1, -2, -3, -4 as above, or
 * <= -1000 for a CUDA error during enqueue); the numerical info (k > 0) is
 * only known through d_info after the stream has progressed.
 */
RELAPACK_API int relapack_dpotrf_async(char uplo, int n, double* A, int lda, int* d_info, relapack_stream_t stream);

/*
 * relapack_dpotrf_batched — independent small factorizations (CFG[4]).
 * Matrix b is d_A[b] (DEVICE pointer, d_lda[b] x d_n[b]).
 *   d_n, d_A, d_lda, d_info  DEVICE arrays of length `batch`
 * Per matrix: info as relapack_dpotrf; n outside [0, RELAPACK_BATCH_NMAX] sets
 * that matrix's info to -2, lda < max(1, n) sets -4; such matrices are skipped.
 * Work on `stream`: a bucketing kernel, then one kernel per size class
 * (16/32/48/64) on library streams forked from and joined back into `stream`.
 * Eager calls use a library-owned bucketing workspace per device (released by
 * relapack_finalize); calls on different streams are ordered by the library
 * (an event after each call) so they never share it concurrently.  The call
 * is capturable into a CUDA graph: inside a capture the workspace is a
 * graph-owned allocation (cudaMallocAsync / cudaFreeAsync nodes of the
 * captured graph), so replays are independent of later eager calls and of
 * each other's workspace.
 * Returns 0, -1 (bad uplo), -2 (batch < 0) or <= -1000 (CUDA error).
 */
#define RELAPACK_BATCH_NMAX 64
RELAPACK_API int relapack_dpotrf_batched(char uplo, int batch, const int* d_n, double* const* d_A, const int* d_lda,
                            int* d_info, relapack_stream_t stream);

/*
 * relapack_batch_split — host-only: the multi-GPU split of a batch (SURVEY
 * §8e "independent batched small factorizations are simply split across
 * GPUs"): contiguous ranges [bounds[r], bounds[r+1]) of the batch, r = 0 ..
 * nranks-1, balanced by the leading-term work sum n_b^3 (n: HOST array of
 * the batch's orders).  Each rank then calls relapack_dpotrf_batched on its
 * range; no collective is needed in the data path.  Returns 0 or -1.
 */
RELAPACK_API int relapack_batch_split(int batch, const int* n, int nranks, int* bounds);

/* ---- multi-GPU: one process per GPU, NCCL over NVLink ---- */
typedef struct relapack_comm relapack_comm_t;

/* Writes a 128-byte NCCL unique id (rank 0 creates it; broadcast it with any
 * transport, e.g. torch.distributed).  Returns 0 or <= -1000. */
RELAPACK_API int relapack_comm_unique_id(char uid[128]);

/* Creates a communicator over `nranks` processes; `device` is this rank's GPU.
 * Returns 0 or <= -1000 (NCCL or CUDA failure; see relapack_last_error). */
RELAPACK_API int relapack_comm_init(relapack_comm_t** comm, const char uid[128], int nranks, int rank, int device);
RELAPACK_API void relapack_comm_destroy(relapack_comm_t* comm);

/*
 * relapack_dpotrf_dist — SPMD distributed factorization of one matrix.
 * Every rank passes a full-size DEVICE buffer A (lda x n, identical input on
 * every rank).  The top recursion levels' trailing updates (TRSM rows and
 * SYRK row-blocks of the L-view; for uplo 'U' these are memory block-columns)
 * are sharded block-cyclically over the ranks with block `nb`; the freshly
 * solved panel blocks are all-gathered with NCCL.  Below `dist_min` the
 * recursion runs redundantly on every rank.  On return every rank holds the
 * full factor and the same info.
 *   nb        row-block size of the block-cyclic distribution (>= 64, mult. of 64)
 *   dist_min  subproblem order below which the recursion is replicated
 * (SURVEY §8(b) sketched `const int* nb`; nb and dist_min are SPMD tuning
 * knobs, not LAPACK arguments, so both are passed by value; -5 if either is
 * out of range or comm is NULL.)  Every rank captures the whole distributed
 * plan — kernels, NCCL all-gathers and the final info all-reduce — once per
 * (shape, knobs, A) into a CUDA graph and replays it; the wait polls
 * ncclCommGetAsyncError with a timeout (env RELAPACK_DIST_TIMEOUT_S, default
 * 600 s) and aborts the communicator on an error (info <= -1000; later calls
 * on it fail with -1000).
 */
RELAPACK_API void relapack_dpotrf_dist(const char* uplo, const int* n, double* A, const int* lda, int nb, int dist_min,
                          relapack_comm_t* comm, int* info);

/*
 * Test hooks of the multi-GPU mode (no NCCL needed):
 *   relapack_dpotrf_dist_loopback  runs the distributed schedule for `nranks`
 *     virtual ranks on the current GPU; A_ranks[s] is rank s's full DEVICE
 *     copy of A.  Collectives are emulated by device copies between the ranks'
 *     buffers and the ranks run one after another between collectives, so no
 *     kernel waits on another rank.  infos[s] (host) = rank s's info.
 *     Returns 0 or an argument / CUDA error code.
 *   relapack_dist_schedule  host-only: rank `rank`'s step list, 16 int64 per
 *     step (kind, level, c_i, c_j, a_i, a_j, b_i, b_j, m, n, k, info_base,
 *     c_buf, a_buf, b_buf, 0); kinds 0 potf2, 1 trsm, 2 gemm, 3 syrk,
 *     10 pack, 11 allgather, 12 unpack.  Returns the step count or -1.
 */
RELAPACK_API int relapack_dpotrf_dist_loopback(const char* uplo, int n, double* const* A_ranks, int lda, int nb,
                                               int dist_min, int nranks, int* infos);
RELAPACK_API int relapack_dist_schedule(int n, int c, int T, int nb, int dist_min, int rank, int nranks, int64_t* out,
                                        int max_ops);

/* ---- configuration, introspection, teardown ---- */
RELAPACK_API void relapack_set_stream(relapack_stream_t stream);
RELAPACK_API const char* relapack_last_error(void);
RELAPACK_API void relapack_finalize(void);

/* Tuning knobs (also read from env RELAPACK_CROSSOVER / RELAPACK_SPLIT_TILE /
 * RELAPACK_GRAPH).  crossover c: base case when n <= c (16 <= c <= 128);
 * split tile T: n1 = T*floor(n/(2T)) (T in {8,16,32,64,128}); graphs 0/1.
 * Return 0, or -1 on an out-of-range value. */
RELAPACK_API int relapack_set_crossover(int c);
RELAPACK_API int relapack_set_split_tile(int t);
RELAPACK_API int relapack_set_graphs(int enabled);
RELAPACK_API int relapack_get_crossover(void);

/*
 * Host-only plan introspection (no GPU needed):
 *   relapack_split_point(n, align) -> n1 of the split rule
 *     n1 = align*floor(n/(2*align)) if that is >= align, else floor(n/2).
 *   relapack_plan_ledger(n, c, T, levels, flops_by_level, count)
 *     leading-term FLOP ledger of the recursion tree the driver would build:
 *     flops_by_level[l] (l = 0..levels-1) = TRSM (m*k^2) + SYRK (n2^2*k) flops
 *     issued at recursion level l+1, flops_by_level[levels] = base-case flops
 *     (sum c_b^3/3); *count = number of kernel launches in the plan.
 *     Returns the recursion depth, or -1 on bad arguments.
 */
RELAPACK_API int relapack_split_point(int n, int align);
RELAPACK_API int relapack_plan_ledger(int n, int c, int T, int levels, double* flops_by_level, int* count);

/*
 * relapack_plan_schedule(n, c, T, lookahead, ops, max_ops, dep_off, dep_idx,
 *                        max_deps)
 *   host-only view of the single-GPU plan the executor captures (knobs as
 *   arguments; lookahead 0/1 splits every trailing SYRK along the child's
 *   split point).  ops (may be NULL): 16 int64 per kernel launch, in the
 *   serial plan order — (kind, level, c_i, c_j, a_i, a_j, b_i, b_j, m, n, k,
 *   info_base, c_buf, a_buf, b_buf, deferred), L-view coordinates as in
 *   relapack_dist_schedule; deferred = 1 for the lookahead trailing updates.
 *   dep_off (max_ops + 1 ints) / dep_idx (max_deps ints), may be NULL: CSR
 *   list of each launch's direct predecessors in the dependency DAG the
 *   graph is captured with (read/write footprint overlaps, transitively
 *   reduced).  Returns the launch count (the arrays are filled only if they
 *   are large enough; *dep_off[count] = total edges), or -1 on bad arguments.
 */
RELAPACK_API int relapack_plan_schedule(int n, int c, int T, int lookahead, int64_t* ops, int max_ops, int* dep_off,
                                        int* dep_idx, int max_deps);

/*
 * Per-kernel-class profiling (bench.py's roofline line).  While enabled, the
 * executor launches the plan without a CUDA graph and brackets every kernel
 * with CUDA events on the launch stream.  relapack_profile_read(kind, ...)
 * synchronises those events and returns, for kind 0 = base potf2, 1 = base
 * TRSM, 2 = GEMM update, 3 = SYRK update: the summed kernel time (ms), the
 * summed leading-term algorithmic flops and the number of launches recorded
 * since the last relapack_profile_reset().  Return 0, or -1 on a bad kind.
 */
RELAPACK_API int relapack_profile_enable(int on);
RELAPACK_API int relapack_profile_read(int kind, double* ms_total, double* flops_total, int* launches);
RELAPACK_API void relapack_profile_reset(void);
/* Per-launch records since the last reset, 7 doubles each: kind, m, n, k,
 * recursion level, algorithmic flops, milliseconds.  Returns the count. */
RELAPACK_API int relapack_profile_records(int max, double* out);

/*
 * Timeline of the last factorization run with RELAPACK_TRACE=1 in the
 * environment (the captured graph itself, not a serialised replay): every
 * kernel records the %globaltimer of its first CTA's start and its last CTA's
 * end.  Writes up to `max` records of 7 doubles in plan order — op kind
 * (0 potf2, 1 trsm, 2 gemm, 3 syrk, 20/21 copies: -1 times), m, n, k,
 * algorithmic flops, start and end in microseconds from the earliest start
 * (-1 if the op launched no kernel) — and returns the count, 0 when no traced
 * run exists, -1 on a CUDA error.  Synchronises the device.
 */
RELAPACK_API int relapack_trace_read(int max, double* out);

/* ---- the paper's other recursive operations ----
 * Same conventions as relapack_dpotrf: column-major FP64 DEVICE matrices,
 * LAPACK argument order and info codes (-i: the i-th argument is illegal,
 * <= -1000: CUDA failure, see relapack_last_error), work ordered on the
 * calling thread's relapack_set_stream stream, synchronous (info is a host
 * int).  Each call's plan is captured once per (operation, shape, operand
 * pointers) into a CUDA graph (footprint-dependency edges) and replayed.
 * Only the uplo triangle of a triangular / symmetric operand is read or
 * written.  uplo 'U' runs the lower algorithms on L = U^T (as dpotrf).
 *
 * relapack_dtrtri — A := A^{-1} for triangular A (LAPACK dtrtri; the paper's
 *   running example; recursive algorithm: invert A_TL,
 *   A_BL := -A_BL A_TL^{-1} (trmm) and A_BL := A_BR^{-1} A_BL (trsm, the
 *   stable form), invert A_BR; crossover to an unblocked in-SM
 *   kernel at n <= 64).  The default plan issues a level's steps as solve
 *   (with the original A_BR), both inversions, trmm — the same product
 *   -A_BR^{-1} A_BL A_TL^{-1}, the two inversions independent of one another
 *   (R16b; RELAPACK_TRTRI_ORDER=0 keeps the paper's order).  diag 'N'/'U' (unit: the diagonal is neither read nor
 *   written).  Arguments: 1 uplo, 2 diag, 3 n, 4 A, 5 lda.  info = k > 0:
 *   A(k,k) == 0, A is not modified (checked first, as LAPACK).
 * relapack_dtrtri_blocked — the blocked algorithm of P:384-409 / S:287-296
 *   with block size nb (>= 1; argument 6): per step A10 := -A10 A00 (A00
 *   already inverted), A10 := A11^{-1} A10, A11 := A11^{-1} (the unblocked
 *   kernel for nb <= 64, the recursive algorithm for larger diagonal blocks).
 * relapack_dlauum — A := L^T L (uplo 'L') / U U^T (uplo 'U') of the
 *   triangular factor, uplo triangle in place (recursive: lauum(A_TL);
 *   A_TL += A_BL^T A_BL; A_BL := A_BR^T A_BL; lauum(A_BR)).
 *   Arguments: 1 uplo, 2 n, 3 A, 4 lda; info 0.
 * relapack_dpotri — A := A^{-1} of the SPD matrix whose Cholesky factor (from
 *   relapack_dpotrf, same uplo) is in A: dtrtri then dlauum.  info = k > 0:
 *   the factor's k-th diagonal entry is zero.
 * relapack_dpotrs — B := A^{-1} B with the Cholesky factor in A: two
 *   recursive triangular solves (L Y = B, L^T X = Y), run per panel of 256
 *   right-hand sides (independent columns; RELAPACK_POTRS_COLS, 0 = one
 *   panel).  B is a DEVICE n x nrhs
 *   column-major matrix (ldb >= max(1, n)).  Arguments: 1 uplo, 2 n, 3 nrhs,
 *   4 A, 5 lda, 6 B, 7 ldb.
 * relapack_dgetrf — P A = L U with partial pivoting (LAPACK dgetrf; recursive
 *   algorithm: split the columns, factor the left panel, swap and
 *   solve the right panel, update A22, factor it, swap the left panel).  A is
 *   m x n (lda >= max(1, m)); ipiv a DEVICE int array of min(m, n) 1-based row
 *   indices (row i was interchanged with row ipiv[i]).  Pivot = the first
 *   maximum |a_ij| of the current column (LAPACK idamax).  info = k > 0: U(k,k)
 *   is exactly zero (the factorization completes).  Panels of <= 32 columns
 *   run as one cooperative grid.  Arguments: 1 m, 2 n, 3 A, 4 lda, 5 ipiv.
 * relapack_dpotrf_blocked — the blocked right-looking Cholesky with block nb
 *   (per step potrf(A11), A21 := A21 L11^{-T}, A22 -=
 *   A21 A21^T) on the same kernels and executor as relapack_dpotrf, for the
 *   paper's blocked-vs-recursive comparison.  nb in [16, n]; diagonal blocks
 *   above 128 are factored by the recursive algorithm.  Arguments: 1 uplo,
 *   2 n, 3 A, 4 lda, 5 nb.  DEVICE A.
 * relapack_xplan_count — host-only: the launch count of one of these plans
 *   (op 0 trtri, 1 trtri_blocked (nb), 2 lauum, 3 potri, 4 potrs (nrhs = nb),
 *   5 getrf (n x n), 6 getrf with lookahead (n x n, 16-CTA cluster panels,
 *   window nb; -1 if n exceeds the cluster panel's rows)), their kinds (0 gemm,
 *   1 tri, 2 trti2, 3 lauu2, 4 potf2, 5 getf2, 6 laswp, 7 check, 8 perm) and
 *   the summed leading-term flops.
 */
RELAPACK_API void relapack_dtrtri(const char* uplo, const char* diag, const int* n, double* A, const int* lda,
                                  int* info);
RELAPACK_API void relapack_dtrtri_blocked(const char* uplo, const char* diag, const int* n, double* A,
                                          const int* lda, int nb, int* info);
RELAPACK_API void relapack_dlauum(const char* uplo, const int* n, double* A, const int* lda, int* info);
RELAPACK_API void relapack_dpotri(const char* uplo, const int* n, double* A, const int* lda, int* info);
RELAPACK_API void relapack_dpotrs(const char* uplo, const int* n, const int* nrhs, const double* A, const int* lda,
                                  double* B, const int* ldb, int* info);
RELAPACK_API void relapack_dgetrf(const int* m, const int* n, double* A, const int* lda, int* ipiv, int* info);
RELAPACK_API void relapack_dpotrf_blocked(const char* uplo, const int* n, double* A, const int* lda, int nb,
                                          int* info);
RELAPACK_API int relapack_xplan_count(int op, int n, int nb, int* kinds, int max_kinds, double* flops);
/* Per-kind profiling of these plans (bench.py): while enabled, plans run
 * serially in plan order (no graph) with CUDA events around every launch;
 * read returns the summed ms, leading-term flops and launch count of one op
 * kind (as relapack_xplan_count's kinds) since the last reset. */
RELAPACK_API int relapack_xprofile_enable(int on);
RELAPACK_API int relapack_xprofile_read(int kind, double* ms_total, double* flops_total, int* launches);
RELAPACK_API void relapack_xprofile_reset(void);
/* Per-launch records since the last reset, 4 doubles each: kind, recursion
 * level (top split = 1), leading-term flops, milliseconds.  Returns the count. */
RELAPACK_API int relapack_xprofile_records(int max, double* out);

/*
 * Kernel test hooks (synchronous; test infrastructure, not a production API).
 * Each launches ONE kernel of the hot path on caller-provided DEVICE blocks with
 * the size-rule choices forced, so every instantiation the factorization runs
 * can be compared with the oracle's BLAS-3 definitions.
 *
 * relapack_update_test — K3/K4: C(M x N) += alpha A B^T on
 *   the tri part of C (0 all, 1 lower i >= j, 2 upper i <= j; M == N if tri).
 *   Operand X (rows x cols) has element (r, c) at X[r + c*ld] (layout 0) or
 *   X[c + r*ld] (layout 1); A is M x K, B is N x K, C is M x N.  The
 *   factorization uses la = lb = lc and alpha = -1 (C -= A B^T).
 *   tile 0 = size rule, else 32/64/128; ksplit 0 = size rule, 1 = none,
 *   2..16 = forced deterministic split-K; allow_tma 0 forces the plain-load
 *   operand path (it is also taken when a base is not 16-byte aligned or an ld
 *   is odd).  max_ctas > 0 caps the grid: each CTA then processes several
 *   (tile, split) work items in turn (the persistent launch the plan uses for
 *   its deferred updates).  full_items > 0 with a forced ksplit > 1 splits
 *   only the tiles [full_items, ntiles) (the plan's tail split of a big
 *   grid's last partial wave); with ksplit 0 the size rule may choose a tail
 *   split itself.  chosen (host, 3 ints, may be NULL) receives (tile, used TMA,
 *   ksplit).  Returns 0, -1 (bad argument) or <= -1000 (CUDA error).
 * relapack_trsm_test — K5 (§8a a3 base): B(m x t) := B L^{-T} (L the t x t lower
 *   L-view block at L, both in `layout`).  variant 0 = the plan's dispatch,
 *   1 register-slab 32-row CTAs, 2 register-slab 64-row, 3 register-slab 128-row
 *   (t <= 128), 4 / 5 shared-memory-slab 4 / 8 warps (t <= 256), 6 the
 *   row-parallel kernel (t <= 64).
 * relapack_potf2_test — K1 (§8a a2): base-case factorization of the n x n
 *   (n <= 128) L-view block; *info (host) = the kernel's info.
 */
RELAPACK_API int relapack_update_test(int la, int lb, int lc, int tri, int M, int N, int K, double alpha, double* C,
                                      int64_t ldc, const double* A, int64_t lda, const double* B, int64_t ldb, int tile,
                                      int ksplit, int allow_tma, int max_ctas, int full_items,
                                      relapack_stream_t stream, int* chosen);
RELAPACK_API int relapack_trsm_test(int layout, int m, int t, const double* L, int64_t ldl, double* B, int64_t ldb,
                                    int variant, relapack_stream_t stream);
RELAPACK_API int relapack_potf2_test(int layout, int n, double* A, int64_t lda, int* info, relapack_stream_t stream);

/* Library version string (build id). */
RELAPACK_API const char* relapack_version(void);

#ifdef __cplusplus
}
#endif

#endif /* RELAPACK_B200_H_ */
