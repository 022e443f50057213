"""Oracle pins for the §8(f) rows (N1 trtri, N3 lauum / potri / potrs, N4
getrf): each oracle function is checked against what the paper and the
mathematics fix — exact integer inverses and products, closed forms,
brute force on tiny inputs, the residual bounds the SPEC examples state — so
that a dropped term, a wrong sign or index or a transposed operand fails one
of them.  CPU only (no GPU)."""
import itertools

import numpy as np
import pytest

import oracle
from inputs import gen

EPS = 2.0 ** -52


def F(x):
    return np.asfortranarray(np.array(x, dtype=np.float64))


def unit_lower_int(n, seed, lo=-2, hi=2):
    """Integer unit-lower-triangular L (off-diagonal in {lo..hi}): det 1, so L^{-1} is integer."""
    g = np.random.default_rng(seed)
    L = np.tril(g.integers(lo, hi + 1, size=(n, n)), -1) + np.eye(n, dtype=np.int64)
    return L.astype(np.int64)


def rand_lower(n, seed):
    """Well-conditioned lower-triangular matrix: the Cholesky factor of a seeded SPD matrix."""
    A = F(gen.spd(n, seed))
    assert oracle.dpotrf(A, "L") == 0
    return np.tril(A)


# ------------------------------------------------------------------ N1 trtri
@pytest.mark.parametrize("n", [1, 2, 5, 17, 40])
def test_trtri_integer_exact(n):
    """L integer with det 1 -> L^{-1} integer; every intermediate is an integer
    < 2^53 (entries stay small), so the inverse is exact: X L == I in integers."""
    L = unit_lower_int(n, n, -1, 1)
    X = F(L)
    assert oracle.dtrtri(X, "L", "N") == 0
    Xi = np.rint(X).astype(np.int64)
    assert np.array_equal(X, Xi.astype(np.float64))
    assert np.array_equal(np.tril(Xi) @ L, np.eye(n, dtype=np.int64))
    assert np.array_equal(L @ np.tril(Xi), np.eye(n, dtype=np.int64))


def test_trtri_closed_forms():
    # 2x2: [[a, 0], [b, c]]^{-1} = [[1/a, 0], [-b/(ac), 1/c]]
    a, b, c = 2.0, 3.0, 4.0
    X = F([[a, 0], [b, c]])
    assert oracle.dtrtri(X, "L") == 0
    assert np.array_equal(np.tril(X), np.array([[0.5, 0], [-3.0 / 8.0, 0.25]]))
    # bidiagonal 1 / -1 -> tril(ones)
    n = 9
    L = np.eye(n) - np.eye(n, k=-1)
    X = F(L)
    assert oracle.dtrtri(X, "L") == 0
    assert np.array_equal(np.tril(X), np.tril(np.ones((n, n))))
    # diagonal powers of two -> reciprocals exactly
    d = 2.0 ** np.arange(-3, 5)
    X = F(np.diag(d))
    assert oracle.dtrtri(X, "L") == 0
    assert np.array_equal(np.diag(X), 1.0 / d)
    # n = 1 (SPEC: [[2]] -> [[0.5]])
    X = F([[2.0]])
    assert oracle.dtrtri(X, "L") == 0 and X[0, 0] == 0.5


def test_trtri_upper_and_unit():
    """uplo U: U^{-1} of U = L^T (here the transposed bidiagonal -> triu(ones));
    diag U: the diagonal is neither read nor written."""
    n = 7
    U = np.eye(n) - np.eye(n, k=1)
    X = F(U + np.tril(np.full((n, n), np.nan), -1))  # NaN below: never read
    assert oracle.dtrtri(X, "U") == 0
    assert np.array_equal(np.triu(X), np.triu(np.ones((n, n))))
    assert np.isnan(X[np.tril_indices(n, -1)]).all()
    L = unit_lower_int(6, 3).astype(np.float64)
    X = F(L)
    np.fill_diagonal(X, 7.0)  # garbage on the diagonal: diag 'U' treats it as 1
    assert oracle.dtrtri(X, "L", "U") == 0
    assert np.array_equal(np.diag(X), np.full(6, 7.0))
    Y = F(L)
    oracle.dtrtri(Y, "L", "N")
    assert np.array_equal(np.tril(X, -1), np.tril(Y, -1))


@pytest.mark.parametrize("n", [50, 200])
def test_trtri_residual(n):
    """SPEC rec_trtri example: ||L X - I||_F <= 100 n eps ||L||_F ||X||_F."""
    L = rand_lower(n, 9)
    X = F(L)
    assert oracle.dtrtri(X, "L") == 0
    X = np.tril(X)
    r = np.linalg.norm(L @ X - np.eye(n)) / (np.linalg.norm(L) * np.linalg.norm(X))
    assert r <= 100 * n * EPS
    # and the upper variant on the transposed data gives the transpose
    Y = F(L.T)
    assert oracle.dtrtri(Y, "U") == 0
    assert np.array_equal(np.triu(Y), X.T)


def test_trtri_singular_and_args():
    X = F(np.tril(np.ones((5, 5))))
    X[3, 3] = 0.0
    before = X.copy()
    assert oracle.dtrtri(X, "L") == 4
    assert np.array_equal(X, before)  # not modified
    assert oracle.dtrtri(F(np.eye(2)), "X") == -1
    assert oracle.dtrtri(F(np.eye(2)), "L", "Q") == -2


# ------------------------------------------------------------------ N3 lauum / potri / potrs
@pytest.mark.parametrize("n", [1, 3, 12, 31])
def test_lauum_integer_exact(n):
    g = np.random.default_rng(n)
    L = np.tril(g.integers(-3, 4, size=(n, n)))
    X = F(L)
    oracle.dlauum(X, "L")
    assert np.array_equal(np.tril(X), np.tril((L.T @ L).astype(np.float64)))
    Y = F(L.T)
    oracle.dlauum(Y, "U")  # U U^T with U = L^T
    assert np.array_equal(np.triu(Y), np.triu((L.T @ L).astype(np.float64)))


def test_lauum_closed_forms():
    n = 8
    X = F(np.tril(np.ones((n, n))))  # (L^T L)_ij = n - max(i, j)
    oracle.dlauum(X, "L")
    i, j = np.indices((n, n))
    assert np.array_equal(np.tril(X), np.tril(n - np.maximum(i, j)).astype(np.float64))
    X = F(np.diag([1.0, 2.0, 3.0]))
    oracle.dlauum(X, "L")
    assert np.array_equal(np.diag(X), np.array([1.0, 4.0, 9.0]))
    X = F([[2.0]])
    oracle.dlauum(X, "L")
    assert X[0, 0] == 4.0  # SPEC: [[2]] -> [[4]]


@pytest.mark.parametrize("n", [4, 15, 30])
def test_potri_integer_exact(n):
    """A = L L^T with L integer, det 1: A^{-1} = L^{-T} L^{-1} integer, exact; A A^{-1} = I."""
    L = unit_lower_int(n, 100 + n, -1, 1)
    A = L @ L.T
    X = F(L)
    assert oracle.dpotri(X, "L") == 0
    Xs = np.tril(X) + np.tril(X, -1).T
    Xi = np.rint(Xs).astype(np.int64)
    assert np.array_equal(Xs, Xi.astype(np.float64))
    assert np.array_equal(A @ Xi, np.eye(n, dtype=np.int64))


@pytest.mark.parametrize("uplo", ["L", "U"])
def test_potri_residual(uplo):
    n = 120
    A = gen.spd(n, 4)
    X = F(A)
    assert oracle.dpotrf(X, uplo) == 0
    assert oracle.dpotri(X, uplo) == 0
    T = np.tril(X) if uplo == "L" else np.triu(X)
    Xs = T + T.T - np.diag(np.diag(T))
    r = np.linalg.norm(A @ Xs - np.eye(n)) / (np.linalg.norm(A) * np.linalg.norm(Xs))
    assert r <= 100 * n * EPS


def test_potri_diagonal():
    d = np.array([4.0, 16.0, 0.25])
    X = F(np.diag(np.sqrt(d)))
    assert oracle.dpotri(X, "L") == 0
    assert np.array_equal(np.diag(X), 1.0 / d)


@pytest.mark.parametrize("uplo", ["L", "U"])
def test_potrs_integer_exact(uplo):
    """L integer unit diagonal, X integer: B = L L^T X integer; both solves exact."""
    n, nrhs = 20, 5
    L = unit_lower_int(n, 7, -1, 1)
    Xtrue = np.random.default_rng(1).integers(-5, 6, size=(n, nrhs))
    B = F(L @ L.T @ Xtrue)
    Af = F(L if uplo == "L" else L.T)
    oracle.dpotrs(Af, B, uplo)
    assert np.array_equal(B, Xtrue.astype(np.float64))


def test_potrs_residual():
    n, nrhs = 150, 7
    A = gen.spd(n, 8)
    Lf = F(A)
    assert oracle.dpotrf(Lf, "L") == 0
    B0 = np.random.default_rng(2).uniform(-1, 1, size=(n, nrhs))
    X = F(B0)
    oracle.dpotrs(Lf, X, "L")
    r = np.linalg.norm(A @ X - B0) / (np.linalg.norm(A) * np.linalg.norm(X))
    assert r <= 100 * n * EPS


# ------------------------------------------------------------------ N4 getrf
def apply_ipiv(A, ipiv):
    """P A for LAPACK-style 1-based sequential row interchanges."""
    A = A.copy()
    for j, p in enumerate(ipiv):
        A[[j, p - 1]] = A[[p - 1, j]]
    return A


def lu_parts(F_, m, n):
    k = min(m, n)
    L = np.tril(F_[:, :k], -1) + np.eye(m, k)
    U = np.triu(F_[:k, :])
    return L, U


def test_getrf_identity_and_permutation():
    n = 7
    X = F(np.eye(n))
    info, ipiv = oracle.dgetrf(X)
    assert info == 0 and list(ipiv) == list(range(1, n + 1)) and np.array_equal(X, np.eye(n))
    # a permutation matrix: L = U = I, the pivots reproduce the permutation
    perm = np.random.default_rng(3).permutation(n)
    P = np.eye(n)[perm]
    X = F(P)
    info, ipiv = oracle.dgetrf(X)
    assert info == 0
    assert np.array_equal(X, np.eye(n))
    assert np.array_equal(apply_ipiv(P, ipiv), np.eye(n))


def test_getrf_exact_no_pivoting():
    """A = L U with |l_ij| < 1 dyadic and an integer U: partial pivoting keeps
    the diagonal (|u_jj| > |l_ij u_jj|), all arithmetic is exact -> L, U back."""
    n = 10
    g = np.random.default_rng(5)
    L = np.tril(g.choice([-0.5, -0.25, 0.0, 0.25, 0.5], size=(n, n)), -1) + np.eye(n)
    U = np.triu(g.integers(-4, 5, size=(n, n)).astype(np.float64), 1) + np.diag(g.choice([8.0, -8.0, 16.0], n))
    X = F(L @ U)
    info, ipiv = oracle.dgetrf(X)
    assert info == 0 and list(ipiv) == list(range(1, n + 1))
    Lg, Ug = lu_parts(X, n, n)
    assert np.array_equal(Lg, L) and np.array_equal(Ug, U)


def test_getrf_2x2_closed_form():
    a, b, c, d = 1.0, 2.0, 4.0, 3.0  # |c| > |a|: swap
    X = F([[a, b], [c, d]])
    info, ipiv = oracle.dgetrf(X)
    assert info == 0 and list(ipiv) == [2, 2]
    assert np.array_equal(X, np.array([[c, d], [a / c, b - (a / c) * d]]))


def test_getrf_ties_take_first():
    X = F([[1.0, 0.0], [-1.0, 1.0]])  # |a00| == |a10|: idamax's first index
    info, ipiv = oracle.dgetrf(X)
    assert list(ipiv) == [1, 2]


def test_getrf_brute_force_tiny():
    """400 random 3x3 matrices with entries in {-2..2}: the same elimination
    done in exact rationals (fractions) gives the same pivots (first maximum
    of the current Schur column), the same info and, to rounding, the same
    L and U."""
    from fractions import Fraction

    vals = [-2, -1, 0, 1, 2]
    rng = np.random.default_rng(0)
    for _ in range(400):
        M = rng.choice(vals, size=(3, 3)).astype(np.float64)
        X = F(M)
        info, ipiv = oracle.dgetrf(X)
        # exact rational partial pivoting
        S = [[Fraction(int(v)) for v in row] for row in M]
        rinfo, rpiv = 0, []
        for j in range(3):
            col = [abs(S[i][j]) for i in range(j, 3)]
            # first index of the maximum (exact)
            mx = max(col)
            p = j + next(i for i, c in enumerate(col) if c == mx)
            rpiv.append(p + 1)
            S[j], S[p] = S[p], S[j]
            if S[j][j] == 0:
                rinfo = rinfo or j + 1
                continue
            for i in range(j + 1, 3):
                S[i][j] = S[i][j] / S[j][j]
                for k in range(j + 1, 3):
                    S[i][k] -= S[i][j] * S[j][k]
        assert info == rinfo
        assert list(ipiv) == rpiv
        for i in range(3):
            for k in range(3):
                assert abs(X[i, k] - float(S[i][k])) <= 1e-14 * 8


@pytest.mark.parametrize("m,n", [(100, 100), (130, 70), (60, 90)])
def test_getrf_residual(m, n):
    """SPEC rec_getrf example: ||P A - L U||_F <= 100 n eps ||A||_F, |l_ij| <= 1."""
    A = np.random.default_rng(m * n).uniform(-1, 1, size=(m, n))
    X = F(A)
    info, ipiv = oracle.dgetrf(X)
    assert info == 0
    L, U = lu_parts(X, m, n)
    assert np.max(np.abs(L)) <= 1.0
    r = np.linalg.norm(apply_ipiv(A, ipiv) - L @ U) / np.linalg.norm(A)
    assert r <= 100 * max(m, n) * EPS


def test_getrf_singular_continues():
    n = 6
    A = np.random.default_rng(9).uniform(-1, 1, size=(n, n))
    A[:, 2] = 0.0  # column 2 zero: the pivot search finds 0 at j = 2
    X = F(A)
    info, ipiv = oracle.dgetrf(X)
    assert info == 3
    L, U = lu_parts(X, n, n)
    assert np.linalg.norm(apply_ipiv(A, ipiv) - L @ U) <= 100 * n * EPS * np.linalg.norm(A)
