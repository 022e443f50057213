"""Pins for the oracle: the oracle is checked against what
the paper and the mathematics fix, never against itself or the CUDA path.

P1 exact integer recovery (north_star)      P5 special cases (n=0,1,2, diagonal, identity)
P2 closed form A_ij = min(i,j)+1            P6 invariants (backward error, log det, row norms)
P3 Pascal closed form (n <= 29)             P7 constructed failure (negated diagonal -> info)
P4 brute force n <= 8 (exact minors)        P8 LAPACK cross-check (numpy.linalg.cholesky)
plus the SPEC examples under tests/golden/ and the TRSM/SYRK/GEMM definitions.
"""
import itertools
import math
import os
from fractions import Fraction

import numpy as np
import pytest

import oracle
from inputs import gen
from tests.metrics import backward_error, floored_rel_err, lower_of, sym_from

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def fortran(a):
    return np.asfortranarray(np.array(a, dtype=np.float64))


def run(A, uplo="L"):
    F = fortran(A)
    info = oracle.dpotrf(F, uplo)
    return F, info


# ---------------------------------------------------------------- exact helpers
def exact_det(M):
    """Determinant by fraction-exact Gaussian elimination (independent of Cholesky)."""
    M = [[Fraction(x) for x in row] for row in M]
    n = len(M)
    det = Fraction(1)
    for c in range(n):
        p = next((r for r in range(c, n) if M[r][c] != 0), None)
        if p is None:
            return Fraction(0)
        if p != c:
            M[c], M[p] = M[p], M[c]
            det = -det
        det *= M[c][c]
        for r in range(c + 1, n):
            f = M[r][c] / M[c][c]
            if f:
                for k in range(c, n):
                    M[r][k] -= f * M[c][k]
    return det


def minors_factor(A):
    """L_ij = det(A[{0..j-1,i},{0..j}]) / sqrt(D_j D_{j+1}) with exact minors."""
    A = [[Fraction(float(x)) for x in row] for row in np.asarray(A)]
    n = len(A)
    D = [Fraction(1)] + [exact_det([r[:k] for r in A[:k]]) for k in range(1, n + 1)]
    L = np.zeros((n, n))
    for j in range(n):
        for i in range(j, n):
            rows = list(range(j)) + [i]
            sub = [[A[r][c] for c in range(j + 1)] for r in rows]
            N = exact_det(sub)
            r2 = N * N / (D[j] * D[j + 1])
            L[i, j] = math.copysign(math.sqrt(float(r2)), float(N)) if N != 0 else 0.0
    return L, D


def sylvester_info(A):
    """info = smallest k with det(A[:k,:k]) <= 0 (Sylvester's criterion), 0 if none."""
    n = len(A)
    for k in range(1, n + 1):
        if exact_det([list(r[:k]) for r in A[:k]]) <= 0:
            return k
    return 0


# ---------------------------------------------------------------- golden SPEC examples
def _parse_potf2_cases():
    cases, cur, section = [], None, None
    for line in open(os.path.join(GOLDEN, "potf2_spec_examples.txt")):
        line = line.strip()
        if not line or line.startswith("#"):
            continue
        if line.startswith("case"):
            parts = dict(p.split("=") for p in line.split()[2:])
            cur = dict(name=line.split()[1], n=int(parts["n"]), info=int(parts["info"]), A=[], L=[])
            cases.append(cur)
            section = "A"
        elif line == "L":
            section = "L"
        else:
            cur[section].append([float("nan") if t == "*" else float(t) for t in line.split()])
    return cases


@pytest.mark.parametrize("case", _parse_potf2_cases(), ids=lambda c: c["name"])
@pytest.mark.parametrize("uplo", ["L", "U"])
def test_golden_potf2_spec_examples(case, uplo):
    A = np.array(case["A"])
    if uplo == "U":
        A = A.T  # '*' entries move to the strict lower triangle: never referenced
    F, info = run(A, uplo)
    assert info == case["info"]
    if case["info"] == 0:
        L = np.array(case["L"])
        assert np.array_equal(lower_of(F, uplo), L)
        # the opposite strict triangle (NaN '*' sentinels) is untouched
        other = np.triu(np.ones_like(A, dtype=bool), 1) if uplo == "L" else np.tril(np.ones_like(A, dtype=bool), -1)
        assert np.array_equal(np.isnan(F[other]), np.isnan(A[other]))


def test_golden_trsm_spec_example():
    sec, data = None, {}
    for line in open(os.path.join(GOLDEN, "trsm_spec_example.txt")):
        line = line.strip()
        if not line or line.startswith("#"):
            continue
        if line in ("L", "B", "X"):
            sec = line
            data[sec] = []
        else:
            data[sec].append([float(t) for t in line.split()])
    Lm, B = fortran(data["L"]), fortran(data["B"])
    oracle.dtrsm_rlt(Lm, B)
    assert np.array_equal(B, np.array(data["X"]))


def test_golden_syrk_spec_example():
    sec, data = None, {}
    for line in open(os.path.join(GOLDEN, "syrk_spec_example.txt")):
        line = line.strip()
        if not line or line.startswith("#"):
            continue
        if line in ("A", "C_lower_expected"):
            sec = line
            data[sec] = []
        else:
            data[sec].append([float("nan") if t == "*" else float(t) for t in line.split()])
    A = fortran(data["A"])
    C = np.asfortranarray(np.zeros((2, 2)))
    C[0, 1] = np.nan  # strict upper: must stay untouched
    oracle.dsyrk_ln(A, C)
    exp = np.array(data["C_lower_expected"])
    assert np.array_equal(np.tril(C), np.tril(np.nan_to_num(exp)))
    assert np.isnan(C[0, 1])


# ---------------------------------------------------------------- P1 exact integer recovery
@pytest.mark.parametrize("uplo", ["L", "U"])
def test_P1_integer_L_exact_n8(uplo):
    for seed in range(1, 101):
        A, L = gen.integer_L(8, seed)
        F, info = run(A, uplo)
        assert info == 0
        assert np.array_equal(lower_of(F, uplo), L), f"seed {seed}"


@pytest.mark.parametrize("n", [64, 256])
def test_P1_integer_L_exact_larger(n):
    A, L = gen.integer_L(n, 5)
    assert np.abs(A).max() < 2**53
    F, info = run(A, "L")
    assert info == 0
    assert np.array_equal(np.tril(F), L)


# ---------------------------------------------------------------- P2 min(i,j)+1 closed form
@pytest.mark.parametrize("n", [1, 2, 17, 300])
@pytest.mark.parametrize("uplo", ["L", "U"])
def test_P2_min_matrix(n, uplo):
    F, info = run(gen.min_matrix(n), uplo)
    assert info == 0
    assert np.array_equal(lower_of(F, uplo), np.tril(np.ones((n, n))))


# ---------------------------------------------------------------- P3 Pascal closed form
@pytest.mark.parametrize("n", [5, 12, 29])
def test_P3_pascal(n):
    F, info = run(gen.pascal(n), "L")
    assert info == 0
    exp = np.array([[float(math.comb(i, j)) if i >= j else 0.0 for j in range(n)] for i in range(n)])
    assert np.array_equal(np.tril(F), exp)


# ---------------------------------------------------------------- P4 brute force n <= 8
@pytest.mark.parametrize("n", [1, 2, 3, 5, 8])
def test_P4_minor_formula_random_spd(n):
    for seed in range(3):
        A = gen.spd(n, seed)
        F, info = run(A, "L")
        assert info == 0
        Lm, _ = minors_factor(A)
        assert floored_rel_err(np.tril(F), Lm, A) <= 1e-13


def test_P4_minor_formula_integer():
    for seed in range(10):
        A, L = gen.integer_L(6, 100 + seed)
        Lm, _ = minors_factor(A)
        assert np.max(np.abs(Lm - L)) <= 1e-12  # the minor formula itself reproduces L
        F, info = run(A, "L")
        assert np.array_equal(np.tril(F), L)


def test_P4_exhaustive_3x3_info():
    """All 5^6 symmetric 3x3 matrices with entries in {-2..2}: info == Sylvester's criterion
    except where a leading minor is exactly 0 (rounding decides; DESIGN reading R4)."""
    vals = range(-2, 3)
    checked = 0
    for a00, a10, a11, a20, a21, a22 in itertools.product(vals, repeat=6):
        A = [[a00, a10, a20], [a10, a11, a21], [a20, a21, a22]]
        minors = [exact_det([r[:k] for r in A[:k]]) for k in (1, 2, 3)]
        exp = sylvester_info(A)
        # skip exactly-zero minors at or before the first failure (several correct infos)
        upto = exp if exp else 3
        if any(m == 0 for m in minors[:upto]):
            continue
        F = fortran(A)
        info = oracle.dpotrf(F, "L")
        assert info == exp, (A, info, exp)
        if exp == 0:
            Lm, _ = minors_factor(A)
            assert floored_rel_err(np.tril(F), Lm, np.array(A, float)) <= 1e-14
        checked += 1
    assert checked > 5000


# ---------------------------------------------------------------- P5 special cases
def test_P5_n0_noop():
    A = np.full((1, 1), 7.0, order="F")
    assert oracle.dpotrf_raw("L", 0, A.reshape(-1), 1) == 0
    assert A[0, 0] == 7.0


def test_P5_n1_sqrt():
    for a in (1.0, 2.0, 1e-300, 1e300, 0.25):
        F, info = run([[a]])
        assert info == 0 and F[0, 0] == math.sqrt(a)
    for a in (0.0, -0.0, -1.0, float("nan")):
        F, info = run([[a]])
        assert info == 1


def test_P5_n2_closed_form():
    a, b, c = 9.0, 3.0, 5.0
    F, info = run([[a, b], [b, c]])
    l00 = math.sqrt(a)
    l10 = b / l00
    l11 = math.sqrt(c - l10 * l10)
    assert info == 0
    assert F[0, 0] == l00 and F[1, 0] == l10 and F[1, 1] == l11


def test_P5_diagonal_and_identity():
    d = np.array([4.0, 9.0, 2.0, 1e-8, 1e8])
    F, info = run(np.diag(d))
    assert info == 0
    assert np.array_equal(np.diag(F), np.sqrt(d))
    assert np.array_equal(np.tril(F, -1), np.zeros((5, 5)))
    F, info = run(np.eye(33), "U")
    assert info == 0 and np.array_equal(F, np.eye(33))


def test_P5_argument_errors():
    buf = np.zeros(16)
    assert oracle.dpotrf_raw("X", 2, buf, 2) == -1
    assert oracle.dpotrf_raw("L", -1, buf, 2) == -2
    assert oracle.dpotrf_raw("L", 4, buf, 3) == -4
    assert oracle.dpotrf_raw("L", 0, buf, 0) == -4  # lda >= max(1, n)


# ---------------------------------------------------------------- P6 invariants
@pytest.mark.parametrize("n,dist", [(64, "uniform"), (300, "uniform"), (257, "normal")])
@pytest.mark.parametrize("uplo", ["L", "U"])
def test_P6_invariants(n, dist, uplo):
    A = gen.spd(n, 3, dist)
    F, info = run(A, uplo)
    assert info == 0
    L = lower_of(F, uplo)
    S = sym_from(A, uplo)
    assert backward_error(S, L) <= 10.0
    assert np.all(np.diag(L) > 0)
    # sum_j L_ij^2 = A_ii to rounding
    assert np.allclose((L * L).sum(axis=1), np.diag(S), rtol=1e-13, atol=0)
    sign, logdet = np.linalg.slogdet(S)
    assert sign == 1.0
    assert abs(2.0 * np.log(np.diag(L)).sum() - logdet) <= 1e-10 * abs(logdet)


def test_P6_other_triangle_untouched_with_nan_sentinels():
    n = 40
    A = gen.spd(n, 9)
    for uplo in ("L", "U"):
        X = np.array(A, order="F")
        mask = np.triu(np.ones((n, n), bool), 1) if uplo == "L" else np.tril(np.ones((n, n), bool), -1)
        X[mask] = np.nan
        info = oracle.dpotrf(X, uplo)
        assert info == 0
        assert np.all(np.isnan(X[mask]))
        assert not np.any(np.isnan(X[~mask]))


def test_P6_lda_padding_untouched():
    n, lda = 50, 53
    A = gen.spd(n, 4, lda=lda)
    X = np.array(A, order="F")
    info = oracle.dpotrf(X, "L", n=n)
    assert info == 0
    assert np.all(np.isnan(X[n:, :]))
    Lo = np.tril(X[:n, :])
    assert backward_error(A[:n, :], Lo) <= 10


# ---------------------------------------------------------------- P7 constructed failure
@pytest.mark.parametrize("uplo", ["L", "U"])
def test_P7_negated_diagonal_info(uplo):
    n = 300
    A = gen.spd(n, 2)
    for k in (0, 1, 37, 150, n - 1):
        F, info = run(gen.indefinite(A, k), uplo)
        assert info == k + 1


def test_P7_spec_shifted_indefinite():
    """gen_spd(64) - 3n I is not positive definite -> info in 1..n."""
    n = 64
    A = gen.spd(n, 1) - 3.0 * n * np.eye(n)
    F, info = run(np.asfortranarray(A))
    assert 1 <= info <= n


# ---------------------------------------------------------------- P8 LAPACK cross-check
@pytest.mark.parametrize("n,dist", [(1, "uniform"), (31, "uniform"), (256, "uniform"), (400, "normal")])
def test_P8_lapack_crosscheck(n, dist):
    A = gen.spd(n, 11, dist)
    F, info = run(A, "L")
    assert info == 0
    Ll = np.linalg.cholesky(A)
    assert floored_rel_err(np.tril(F), Ll, A) <= 1e-12


# ---------------------------------------------------------------- BLAS-3 definitions
def test_trsm_integer_exact_and_reconstruction():
    g = gen.philox(3, 5)
    m, k = 37, 21
    L = np.tril(g.integers(-3, 4, size=(k, k))).astype(np.float64)
    L[np.diag_indices(k)] = g.choice([1.0, 2.0, 4.0], size=k)
    X = g.integers(-5, 6, size=(m, k)).astype(np.float64)
    B = fortran(X.astype(np.int64) @ L.T.astype(np.int64))
    oracle.dtrsm_rlt(fortran(L), B)
    assert np.array_equal(B, X)
    # random well-conditioned case: X L^T reproduces B (independent numpy matmul)
    L2 = np.tril(g.random((k, k)) - 0.5) + np.diag(k + g.random(k))
    B0 = g.random((m, k)) - 0.5
    B2 = fortran(B0)
    oracle.dtrsm_rlt(fortran(L2), B2)
    assert np.allclose(B2 @ L2.T, B0, rtol=0, atol=1e-13)


def test_syrk_gemm_integer_exact():
    g = gen.philox(4, 5)
    n, k, m = 29, 13, 17
    A = g.integers(-9, 10, size=(n, k))
    C = g.integers(-99, 100, size=(n, n))
    Cf = fortran(C)
    Cf[np.triu_indices(n, 1)] = np.nan
    oracle.dsyrk_ln(fortran(A), Cf)
    exp = C - A @ A.T
    assert np.array_equal(np.tril(Cf), np.tril(exp).astype(float))
    assert np.all(np.isnan(Cf[np.triu_indices(n, 1)]))
    Am = g.integers(-9, 10, size=(m, k))
    Bn = g.integers(-9, 10, size=(n, k))
    C2 = g.integers(-99, 100, size=(m, n))
    C2f = fortran(C2)
    oracle.dgemm_nt(fortran(Am), fortran(Bn), C2f)
    assert np.array_equal(C2f, (C2 - Am @ Bn.T).astype(float))


# ---------------------------------------------------------------- batched
def test_batched_oracle_info_closed_form():
    b = gen.batched_spd(400, 3)
    assert int((b["expected_info"] > 0).sum()) == 4
    buf = b["buf"].copy()
    info = oracle.dpotrf_batched("L", b["ns"], buf, b["offsets"], b["ldas"])
    assert np.array_equal(info, b["expected_info"])
    # successful matrices satisfy the backward-error bound
    for i in np.nonzero(info == 0)[0][:50]:
        nb, off = int(b["ns"][i]), int(b["offsets"][i])
        A = b["buf"][off: off + nb * nb].reshape(nb, nb).T
        L = np.tril(buf[off: off + nb * nb].reshape(nb, nb).T)
        assert backward_error(sym_from(A, "L"), L) <= 10


def test_dpotrf_cols_prefix_bitwise():
    """The bench's bounded sample (first c columns) is bitwise the full factor's prefix."""
    n, c = 200, 57
    A = gen.spd(n, 8)
    F1 = np.array(A, order="F")
    F2 = np.array(A, order="F")
    assert oracle.dpotrf(F1, "L") == 0
    assert oracle.dpotrf_cols(F2, "L", c) == 0
    assert np.array_equal(np.tril(F1)[:, :c], np.tril(F2)[:, :c])


def test_oracle_thread_count_independent(tmp_path):
    """Per-element order is fixed, so the result does not depend on the thread count."""
    import json
    import subprocess
    import sys

    n = 700
    path = str(tmp_path / "A.npy")
    np.save(path, gen.spd(n, 1))  # same input bits for every child (BLAS threading may vary the generator)
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = (
        "import numpy as np, sys, json, hashlib; sys.path.insert(0, %r); import oracle;"
        "A = np.asfortranarray(np.load(%r)); info = oracle.dpotrf(A, 'L');"
        "print(json.dumps([info, hashlib.sha256(np.tril(A).tobytes()).hexdigest()]))"
    ) % (root, path)
    outs = []
    for t in ("1", "4"):
        env = dict(os.environ, OMP_NUM_THREADS=t)
        outs.append(json.loads(subprocess.check_output([sys.executable, "-c", code], env=env)))
    assert outs[0] == outs[1]


def test_dpotrf_cols_panel_matches_full():
    """The column-panel binding (used by the full-size GPU parity test) gives
    bitwise the first J columns of the whole-matrix left-looking loop."""
    n, J = 300, 64
    A = gen.spd(n, 21)
    full = np.array(A, order="F", copy=True)
    assert oracle.dpotrf(full, "L") == 0
    panel = np.asfortranarray(A[:, :J])
    assert oracle.dpotrf_cols_panel(panel, J) == 0
    assert np.array_equal(np.tril(panel), np.tril(full[:, :J]))
