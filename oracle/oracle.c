/*
 * oracle.c — TEST INFRASTRUCTURE ONLY.  Plain, slow, obviously-correct CPU
 * reference for the recursive-Cholesky hot path of arXiv:1602.06763
 * ("Recursive Algorithms for Dense Linear Algebra: The ReLAPACK Collection").
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library.  The product path
 * (paper_1602_06763_b200/) never links, loads or calls it, and this file
 * shares no code, header, table or helper with the CUDA path.
 *
 * Citation convention: P:a-b = /root/reference/PAPER.md lines a-b,
 * S:a-b = /root/reference/SPEC.md lines a-b.
 *
 * What the method computes: the recursive xpotrf (P:275-307,
 * P:366-370 "dpotrf2 ... used in LAPACK's blocked dpotrf as a replacement for
 * the unblocked dpotf2") reaches exactly, up to rounding order, the unique
 * lower-triangular L with positive diagonal such that A = L*L^T.  The oracle
 * is therefore NOT recursive: it is that definition written out as the
 * textbook left-looking ("jki") triple loop of the unblocked dpotf2
 * (post-condition and NotPositiveDefinite error).
 *
 * Arithmetic rules (reading R7): IEEE double, one subtraction per
 * term in ascending k, true division by the pivot, correctly rounded sqrt;
 * built with -O3 -ffp-contract=off and no fast-math, so no FMA contraction.
 * The per-element operation order does not depend on the OpenMP thread count
 * (threads split the row index i only), so results are bitwise deterministic.
 *
 * The BLAS-3 steps of the recursion (TRSM, SYRK, GEMM; "two BLAS-3
 * invocations surrounded by two recursive applications") are also given here
 * by their plain definitions so the CUDA update kernels can be
 * checked in isolation.
 */
#include <math.h>
#include <stddef.h>
#include <stdint.h>

/* Element (i, j) of the factor being computed.  uplo = 'L': column-major
 * lower triangle, a(i,j) = A[i + j*lda].  uplo = 'U': A = U^T U with U = L^T,
 * so L(i,j) = U(j,i) = A[j + i*lda] (reading R5). */
#define LIDX(i, j) (lower ? ((size_t)(i) + (size_t)(j) * (size_t)lda) \
                          : ((size_t)(j) + (size_t)(i) * (size_t)lda))

/*
 * update_column — a(j:n-1, j) -= sum_{k<j} a(j:n-1, k) * a(j, k), one
 * subtraction per term in ascending k for every element (the "jki" loop of the
 * left-looking algorithm).  Threads own disjoint row ranges; the
 * loop nest is ordered so the innermost index walks contiguous memory (rows
 * for 'L', k for 'U').  The per-element operation sequence is the same in
 * both orders, so the result is bitwise independent of order and threads.
 */
static void update_column(int lower, int n, double* A, int lda, int j) {
  if (lower) {
#pragma omp parallel if (n - j > 512)
    {
      int nt = 1, t = 0;
#ifdef _OPENMP
      extern int omp_get_num_threads(void);
      extern int omp_get_thread_num(void);
      nt = omp_get_num_threads();
      t = omp_get_thread_num();
#endif
      const int rows = n - j;
      const int i0 = j + (int)((long long)rows * t / nt), i1 = j + (int)((long long)rows * (t + 1) / nt);
      double* aj = A + (size_t)j * (size_t)lda;
      for (int k = 0; k < j; ++k) {
        const double* ak = A + (size_t)k * (size_t)lda;
        const double ajk = ak[j];
        for (int i = i0; i < i1; ++i) {
          double p = ak[i] * ajk;
          aj[i] = aj[i] - p;
        }
      }
    }
  } else {
#pragma omp parallel for schedule(static) if (n - j > 512)
    for (int i = j; i < n; ++i) {
      double s = A[LIDX(i, j)];
      for (int k = 0; k < j; ++k) {
        double p = A[LIDX(i, k)] * A[LIDX(j, k)];
        s = s - p;
      }
      A[LIDX(i, j)] = s;
    }
  }
}

/*
 * oracle_dpotrf — unblocked Cholesky, left-looking column form.
 *   for j = 0..n-1:
 *     for k = 0..j-1: for i = j..n-1: a(i,j) = a(i,j) - a(i,k)*a(j,k)
 *     d = a(j,j); if !(d > 0) return j+1            (info, 1-based)
 *     a(j,j) = sqrt(d); for i = j+1..n-1: a(i,j) = a(i,j) / a(j,j)
 * Returns LAPACK info: 0 success, -1 bad uplo, -2 n<0, -4 lda<max(1,n),
 * k>0 leading minor of order k not positive definite (factorization stops;
 * columns < k-1 are final).  Only the uplo triangle is read or written.
 */
int oracle_dpotrf(char uplo, int n, double* A, int lda) {
  int lower;
  if (uplo == 'L' || uplo == 'l') lower = 1;
  else if (uplo == 'U' || uplo == 'u') lower = 0;
  else return -1;
  if (n < 0) return -2;
  if (lda < (n > 1 ? n : 1)) return -4;
  for (int j = 0; j < n; ++j) {
    update_column(lower, n, A, lda, j);
    double d = A[LIDX(j, j)];
    if (!(d > 0.0)) return j + 1; /* catches d <= 0, -0.0 and NaN */
    d = sqrt(d);
    A[LIDX(j, j)] = d;
    for (int i = j + 1; i < n; ++i) A[LIDX(i, j)] = A[LIDX(i, j)] / d;
  }
  return 0;
}

/*
 * oracle_dpotrf_cols — the same loop stopped after the first `ncols` columns
 * (a bounded sample of one factorization, used only by bench.py's
 * cpu_baseline).  Returns info as oracle_dpotrf, restricted to those columns.
 */
int oracle_dpotrf_cols(char uplo, int n, double* A, int lda, int ncols) {
  int lower = (uplo == 'L' || uplo == 'l');
  if (!lower && !(uplo == 'U' || uplo == 'u')) return -1;
  if (n < 0) return -2;
  if (lda < (n > 1 ? n : 1)) return -4;
  if (ncols > n) ncols = n;
  for (int j = 0; j < ncols; ++j) {
    update_column(lower, n, A, lda, j);
    double d = A[LIDX(j, j)];
    if (!(d > 0.0)) return j + 1;
    d = sqrt(d);
    A[LIDX(j, j)] = d;
    for (int i = j + 1; i < n; ++i) A[LIDX(i, j)] = A[LIDX(i, j)] / d;
  }
  return 0;
}

/*
 * oracle_dpotrf_batched — oracle_dpotrf applied to each matrix of a batch
 * (CFG[4]); matrices are independent, so threads split the batch.
 * A_all holds matrix b at offset[b] with leading dimension lda[b].
 */
void oracle_dpotrf_batched(char uplo, int batch, const int* n, double* A_all,
                           const int64_t* offset, const int* lda, int* info) {
#pragma omp parallel for schedule(dynamic, 64)
  for (int b = 0; b < batch; ++b)
    info[b] = oracle_dpotrf(uplo, n[b], A_all + offset[b], lda[b]);
}

/*
 * oracle_dtrsm_rlt — TRSM Right/Lower/Trans/NonUnit, the solve
 * step of the recursion: B (m x k, col-major, ldb) := B * L^{-T}, i.e. solve
 * X * L^T = B for X with L (k x k lower, ldl).  Row r of X:
 *   x(r,j) = (b(r,j) - sum_{p<j} x(r,p) * L(j,p)) / L(j,j), ascending p.
 */
void oracle_dtrsm_rlt(int m, int k, const double* L, int ldl, double* B, int ldb) {
#pragma omp parallel for schedule(static) if (m > 256)
  for (int r = 0; r < m; ++r) {
    for (int j = 0; j < k; ++j) {
      double s = B[(size_t)r + (size_t)j * ldb];
      for (int p = 0; p < j; ++p) {
        double q = B[(size_t)r + (size_t)p * ldb] * L[(size_t)j + (size_t)p * ldl];
        s = s - q;
      }
      B[(size_t)r + (size_t)j * ldb] = s / L[(size_t)j + (size_t)j * ldl];
    }
  }
}

/*
 * oracle_dsyrk_ln — SYRK Lower/NoTrans with alpha = -1, beta = 1,
 * the trailing update of the recursion: C (n x n, ldc) lower triangle only
 *   c(i,j) = c(i,j) - sum_{p<k} a(i,p) * a(j,p),  i >= j, ascending p.
 * The strict upper triangle of C is never read or written.
 */
void oracle_dsyrk_ln(int n, int k, const double* A, int lda, double* C, int ldc) {
#pragma omp parallel for schedule(dynamic, 16) if (n > 128)
  for (int j = 0; j < n; ++j) {
    for (int i = j; i < n; ++i) {
      double s = C[(size_t)i + (size_t)j * ldc];
      for (int p = 0; p < k; ++p) {
        double q = A[(size_t)i + (size_t)p * lda] * A[(size_t)j + (size_t)p * lda];
        s = s - q;
      }
      C[(size_t)i + (size_t)j * ldc] = s;
    }
  }
}

/*
 * oracle_dgemm_nt — GEMM NoTrans/Trans with alpha = -1, beta = 1,
 * the update inside the recursive TRSM: C (m x n) -= A (m x k) * B (n x k)^T.
 */
void oracle_dgemm_nt(int m, int n, int k, const double* A, int lda, const double* B,
                     int ldb, double* C, int ldc) {
#pragma omp parallel for schedule(static) if (n > 64)
  for (int j = 0; j < n; ++j) {
    for (int i = 0; i < m; ++i) {
      double s = C[(size_t)i + (size_t)j * ldc];
      for (int p = 0; p < k; ++p) {
        double q = A[(size_t)i + (size_t)p * lda] * B[(size_t)j + (size_t)p * ldb];
        s = s - q;
      }
      C[(size_t)i + (size_t)j * ldc] = s;
    }
  }
}

/* ========================================================================
 * SURVEY §8(f) rows N1-N4 (the other recursive operations of the paper):
 * each function is the plain definition of what the recursive algorithm
 * reaches (the recursion reorganises a blocked algorithm, "once the
 * traversal direction is fixed, all blocked variants result in the same
 * recursive algorithm"), written out as the unblocked loop.  L-view indexing
 * (LIDX) as above: uplo 'U' works on L = U^T.
 * ======================================================================== */
#include <stdlib.h>
#include <string.h>

static int parse_lower(char uplo) {
  if (uplo == 'L' || uplo == 'l') return 1;
  if (uplo == 'U' || uplo == 'u') return 0;
  return -1;
}

/*
 * oracle_dtrtri — X = L^{-1} in place ("in-place inversion of a
 * lower triangular matrix A := A^{-1}", the paper's running example; SPEC
 * rec_trtri / blocked_trtri S:287-296; LAPACK dtrtri).  Definition
 * L X = I, column j of X by forward substitution (ascending k, one
 * subtraction per term, true division):
 *   x_jj = 1 / l_jj;  x_ij = (0 - sum_{k=j}^{i-1} l_ik x_kj) / l_ii   (i > j)
 * computed as the column-oriented (axpy) sweep with the same per-element
 * operation order.  diag 'U': l_ii = 1 (not referenced).  uplo 'U': U^{-1} =
 * (L^{-1})^T of L = U^T.  Returns 0, -1 uplo, -2 diag, -3 n < 0, -5 lda, or
 * k > 0: l_kk == 0 (singular; A is then not modified, LAPACK's check).
 */
int oracle_dtrtri(char uplo, char diag, int n, double* A, int lda) {
  const int lower = parse_lower(uplo);
  if (lower < 0) return -1;
  const int unit = (diag == 'U' || diag == 'u');
  if (!unit && !(diag == 'N' || diag == 'n')) return -2;
  if (n < 0) return -3;
  if (lda < (n > 1 ? n : 1)) return -5;
  if (!unit)
    for (int k = 0; k < n; ++k)
      if (A[LIDX(k, k)] == 0.0) return k + 1;
  /* dense copy of the L-view: columns of X are computed from the original L */
  double* Lc = (double*)malloc(sizeof(double) * (size_t)n * (size_t)(n > 0 ? n : 1));
  for (int j = 0; j < n; ++j)
    for (int i = j; i < n; ++i) Lc[(size_t)i + (size_t)j * n] = A[LIDX(i, j)];
#pragma omp parallel
  {
    double* x = (double*)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
#pragma omp for schedule(dynamic, 8)
    for (int j = 0; j < n; ++j) {
      for (int i = j; i < n; ++i) x[i] = 0.0;
      x[j] = 1.0;
      for (int k = j; k < n; ++k) {
        /* x_k is complete once its diagonal division is done */
        if (!unit) x[k] = x[k] / Lc[(size_t)k + (size_t)k * n];
        const double xk = x[k];
        const double* lk = Lc + (size_t)k * n;
        for (int i = k + 1; i < n; ++i) {
          double p = lk[i] * xk;
          x[i] = x[i] - p;
        }
      }
      for (int i = j; i < n; ++i)
        if (!(unit && i == j)) A[LIDX(i, j)] = x[i];
    }
    free(x);
  }
  free(Lc);
  return 0;
}

/*
 * oracle_dlauum — the product L^T L of the L-view, lower triangle in place
 * (uplo 'L': A := L^T L; uplo 'U': A := U U^T = the same in the L-view;
 * SPEC rec_lauum S:376-384; the macro list P:125-127).  Definition:
 *   c_ij = sum_{k=i}^{n-1} l_ki l_kj,  i >= j   (ascending k, from 0.0)
 */
void oracle_dlauum(char uplo, int n, double* A, int lda) {
  const int lower = parse_lower(uplo);
  if (lower < 0 || n <= 0) return;
  double* Lc = (double*)malloc(sizeof(double) * (size_t)n * (size_t)n);
  for (int j = 0; j < n; ++j)
    for (int i = j; i < n; ++i) Lc[(size_t)i + (size_t)j * n] = A[LIDX(i, j)];
#pragma omp parallel for schedule(dynamic, 8)
  for (int j = 0; j < n; ++j) {
    const double* lj = Lc + (size_t)j * n;
    for (int i = j; i < n; ++i) {
      const double* li = Lc + (size_t)i * n;
      double s = 0.0;
      for (int k = i; k < n; ++k) {
        double p = li[k] * lj[k];
        s = s + p;
      }
      A[LIDX(i, j)] = s;
    }
  }
  free(Lc);
}

/*
 * oracle_dpotri — inverse of the SPD matrix from its Cholesky factor, in place
 * (LAPACK dpotri = dtrtri then dlauum; §8(f) N3):
 * A^{-1} = L^{-T} L^{-1} (uplo 'L'), U^{-1} U^{-T} (uplo 'U'), uplo triangle.
 * Returns oracle_dtrtri's info.
 */
int oracle_dpotri(char uplo, int n, double* A, int lda) {
  const int info = oracle_dtrtri(uplo, 'N', n, A, lda);
  if (info != 0) return info;
  oracle_dlauum(uplo, n, A, lda);
  return 0;
}

/*
 * oracle_dpotrs — solve A X = B with the Cholesky factor in A (LAPACK dpotrs;
 * §8(f) N3): B (n x nrhs, column-major, ldb) := A^{-1} B by
 *   L Y = B  (forward:  y_i = (b_i - sum_{k<i} l_ik y_k) / l_ii)
 *   L^T X = Y (backward: x_i = (y_i - sum_{k>i} l_ki x_k) / l_ii, i descending)
 * ascending / descending k as written, true division.  uplo 'U': L = U^T.
 */
void oracle_dpotrs(char uplo, int n, int nrhs, const double* A, int lda, double* B, int ldb) {
  const int lower = parse_lower(uplo);
  if (lower < 0 || n <= 0 || nrhs <= 0) return;
#pragma omp parallel for schedule(dynamic, 4)
  for (int c = 0; c < nrhs; ++c) {
    double* b = B + (size_t)c * (size_t)ldb;
    for (int i = 0; i < n; ++i) {
      double s = b[i];
      for (int k = 0; k < i; ++k) {
        double p = A[LIDX(i, k)] * b[k];
        s = s - p;
      }
      b[i] = s / A[LIDX(i, i)];
    }
    for (int i = n - 1; i >= 0; --i) {
      double s = b[i];
      for (int k = i + 1; k < n; ++k) {
        double p = A[LIDX(k, i)] * b[k];
        s = s - p;
      }
      b[i] = s / A[LIDX(i, i)];
    }
  }
}

/*
 * oracle_dgetrf — LU with partial pivoting, P A = L U (SPEC rec_getrf /
 * blocked_getrf S:306-312; §8(f) N4), as the unblocked
 * right-looking getf2 loop (LAPACK order) on the m x n column-major A:
 *   for j = 0 .. min(m,n)-1:
 *     p = first index of max_{i>=j} |a_ij|            (ties: smallest i)
 *     ipiv[j] = p + 1 (1-based);  swap rows j and p over all n columns
 *     if a_jj != 0:  a_ij = a_ij / a_jj  (i > j, true division)
 *     else if info == 0: info = j + 1  (factorization continues)
 *     a_ik = a_ik - a_ij * a_jk  (i > j, k > j)
 * Returns info (0, or the first zero pivot), or -1 m < 0, -2 n < 0, -4 lda.
 */
int oracle_dgetrf(int m, int n, double* A, int lda, int* ipiv) {
  if (m < 0) return -1;
  if (n < 0) return -2;
  if (lda < (m > 1 ? m : 1)) return -4;
  int info = 0;
  const int mn = m < n ? m : n;
  for (int j = 0; j < mn; ++j) {
    double* aj = A + (size_t)j * (size_t)lda;
    int p = j;
    double best = fabs(aj[j]);
    for (int i = j + 1; i < m; ++i) {
      const double v = fabs(aj[i]);
      if (v > best) {
        best = v;
        p = i;
      }
    }
    ipiv[j] = p + 1;
    if (p != j)
      for (int k = 0; k < n; ++k) {
        double* col = A + (size_t)k * (size_t)lda;
        const double t = col[j];
        col[j] = col[p];
        col[p] = t;
      }
    const double piv = aj[j];
    if (piv != 0.0) {
      for (int i = j + 1; i < m; ++i) aj[i] = aj[i] / piv;
    } else if (info == 0) {
      info = j + 1;
    }
#pragma omp parallel for schedule(static) if ((size_t)(m - j) * (size_t)(n - j) > 65536)
    for (int k = j + 1; k < n; ++k) {
      double* col = A + (size_t)k * (size_t)lda;
      const double ujk = col[j];
      for (int i = j + 1; i < m; ++i) {
        double q = aj[i] * ujk;
        col[i] = col[i] - q;
      }
    }
  }
  return info;
}

/* Number of OpenMP threads the oracle will use (for bench reporting). */
int oracle_num_threads(void) {
#ifdef _OPENMP
  extern int omp_get_max_threads(void);
  return omp_get_max_threads();
#else
  return 1;
#endif
}
