"""GPU parity of the §8(f) rows (N1 dtrtri + blocked dtrtri, N2 blocked
dpotrf, N3 dlauum / dpotri / dpotrs, N4 dgetrf) through the C ABI against the
oracle (oracle.c, pinned in tests/test_oracle_next.py) on the same seeded
inputs, element by element.

Tolerances (derived):
* products (lauum): the dot-product bound |Cg - Co| <= 2 (n + 2) u (|L|^T |L|).
* inverses and solves of the well-conditioned test matrices (Cholesky factors
  of the kappa ~ 2.3 SPD recipe): per-column normwise
  max_i |Xg - Xo|_ij / max_i |Xo|_ij <= 1e-11 (both sides are backward
  stable; forward error <~ n u kappa; measured ~1e-14), plus the SPEC
  residual ||A X - I|| <= 100 n eps ||A|| ||X||.
* getrf: identical pivots (exact), per-column normwise factor error <= 1e-9
  (random Uniform(-1,1) matrices: growth and kappa ~ n), residual
  ||P A - L U||_F <= 100 n eps ||A||_F.
* blocked dpotrf: the factorization's own bound (floored relative 1e-10, R8).
"""
import numpy as np
import pytest
import torch

import oracle
import paper_1602_06763_b200 as rl
from inputs import gen
from tests.metrics import floored_rel_err

pytestmark = pytest.mark.gpu

EPS = 2.0 ** -52
U = 2.0 ** -53


def to_dev(A: np.ndarray) -> torch.Tensor:
    """Column-major device copy of a Fortran-ordered numpy matrix."""
    return torch.from_numpy(np.ascontiguousarray(A.T)).cuda().t()


def chol_factor(n, seed, uplo="L"):
    """The Cholesky factor of the SPD recipe, in the uplo triangle; NaN in the other one."""
    A = gen.spd(n, seed)
    F = np.array(A, order="F")
    assert oracle.dpotrf(F, uplo) == 0
    nan = np.full((n, n), np.nan)
    T = np.tril(F) + np.triu(nan, 1) if uplo == "L" else np.triu(F) + np.tril(nan, -1)
    return np.asfortranarray(T), A


def tri_part(X, uplo):
    return np.tril(X) if uplo == "L" else np.triu(X)


def colnorm_err(G, O):
    den = np.maximum(np.max(np.abs(O), axis=0, keepdims=True), 1e-300)
    return float(np.max(np.abs(G - O) / den))


def other_mask(n, uplo):
    return np.triu(np.ones((n, n), bool), 1) if uplo == "L" else np.tril(np.ones((n, n), bool), -1)


# ------------------------------------------------------------------ N1 trtri
@pytest.mark.parametrize("uplo", ["L", "U"])
@pytest.mark.parametrize("n", [1, 7, 64, 65, 100, 300, 1031, 2048])
def test_trtri(n, uplo):
    T, _ = chol_factor(n, n, uplo)
    dT = to_dev(T)
    assert rl.dtrtri(dT, uplo, "N") == 0
    G = dT.cpu().numpy()
    R = np.array(T, order="F")
    assert oracle.dtrtri(R, uplo, "N") == 0
    e = colnorm_err(tri_part(G, uplo), tri_part(R, uplo))
    assert e <= 1e-11, e
    assert np.isnan(G[other_mask(n, uplo)]).all()  # the other triangle never written
    Lm, X = tri_part(np.nan_to_num(T), uplo), tri_part(G, uplo)
    r = np.linalg.norm(Lm @ X - np.eye(n)) / (np.linalg.norm(Lm) * np.linalg.norm(X))
    assert r <= 100 * n * EPS


@pytest.mark.parametrize("uplo", ["L", "U"])
def test_trtri_unit_and_integer(uplo):
    """Integer unit-lower L (det 1): the inverse is an exact integer matrix;
    diag 'U' ignores (and keeps) a garbage diagonal."""
    n = 200
    g = np.random.default_rng(4)
    L = np.tril(g.integers(-1, 2, size=(n, n)), -1).astype(np.float64) * (g.random((n, n)) < 0.05) + np.eye(n)
    T = L if uplo == "L" else L.T
    X = np.asfortranarray(T.copy())
    np.fill_diagonal(X, 3.0)
    dX = to_dev(X)
    assert rl.dtrtri(dX, uplo, "U") == 0
    G = dX.cpu().numpy()
    R = np.array(X, order="F")
    assert oracle.dtrtri(R, uplo, "U") == 0
    assert np.array_equal(tri_part(G, uplo), tri_part(R, uplo))  # exact integers
    assert np.array_equal(np.diag(G), np.full(n, 3.0))


def test_trtri_singular():
    T, _ = chol_factor(300, 3)
    T[150, 150] = 0.0
    dT = to_dev(T)
    before = dT.clone()
    assert rl.dtrtri(dT, "L") == 151
    assert torch.equal(torch.nan_to_num(dT, 7.0), torch.nan_to_num(before, 7.0))  # not modified
    assert rl.dtrtri(dT, "X") == -1


@pytest.mark.parametrize("nb", [64, 128, 256])
@pytest.mark.parametrize("n", [300, 1031])
def test_trtri_blocked(n, nb):
    T, _ = chol_factor(n, 2, "L")
    dT = to_dev(T)
    assert rl.dtrtri_blocked(dT, nb, "L") == 0
    G = dT.cpu().numpy()
    R = np.array(T, order="F")
    assert oracle.dtrtri(R, "L") == 0
    assert colnorm_err(np.tril(G), np.tril(R)) <= 1e-11


# ------------------------------------------------------------------ N3 lauum / potri / potrs
@pytest.mark.parametrize("uplo", ["L", "U"])
@pytest.mark.parametrize("n", [1, 33, 64, 65, 200, 1031, 2048])
def test_lauum(n, uplo):
    T, _ = chol_factor(n, 5 + n, uplo)
    dT = to_dev(T)
    assert rl.dlauum(dT, uplo) == 0
    G = dT.cpu().numpy()
    R = np.array(T, order="F")
    oracle.dlauum(R, uplo)
    Lm = np.tril(np.nan_to_num(T)) if uplo == "L" else np.tril(np.nan_to_num(T).T)
    bound = 2 * (n + 2) * U * (np.abs(Lm).T @ np.abs(Lm))
    Gl = np.tril(G) if uplo == "L" else np.tril(G.T)
    Rl = np.tril(R) if uplo == "L" else np.tril(R.T)
    mask = np.tril(np.ones((n, n), bool))
    assert np.all(np.abs(Gl - Rl)[mask] <= bound[mask])
    assert np.isnan(G[other_mask(n, uplo)]).all()


@pytest.mark.parametrize("uplo", ["L", "U"])
@pytest.mark.parametrize("n", [5, 64, 129, 500, 1500])
def test_potri(n, uplo):
    T, A = chol_factor(n, 9, uplo)
    dT = to_dev(T)
    assert rl.dpotri(dT, uplo) == 0
    G = dT.cpu().numpy()
    R = np.array(T, order="F")
    assert oracle.dpotri(R, uplo) == 0
    assert colnorm_err(tri_part(G, uplo), tri_part(R, uplo)) <= 1e-11
    Xt = tri_part(G, uplo)
    Xs = Xt + Xt.T - np.diag(np.diag(Xt))
    r = np.linalg.norm(A @ Xs - np.eye(n)) / (np.linalg.norm(A) * np.linalg.norm(Xs))
    assert r <= 100 * n * EPS


def test_potri_after_potrf_on_gpu():
    """The LAPACK chain dpotrf -> dpotri on the device (same uplo), against A^{-1} of the oracle."""
    n = 777
    A = np.asfortranarray(gen.spd(n, 12))
    dA = to_dev(A)
    assert rl.dpotrf(dA, "U") == 0
    assert rl.dpotri(dA, "U") == 0
    R = np.array(A, order="F")
    assert oracle.dpotrf(R, "U") == 0 and oracle.dpotri(R, "U") == 0
    assert colnorm_err(np.triu(dA.cpu().numpy()), np.triu(R)) <= 1e-11


@pytest.mark.parametrize("uplo", ["L", "U"])
@pytest.mark.parametrize("n,nrhs", [(1, 1), (65, 7), (300, 1), (1031, 130), (2048, 64)])
def test_potrs(n, nrhs, uplo):
    T, A = chol_factor(n, 13, uplo)
    B0 = np.asfortranarray(np.random.default_rng(n + nrhs).uniform(-1, 1, size=(n, nrhs)))
    dT, dB = to_dev(T), to_dev(B0)
    assert rl.dpotrs(dT, dB, uplo) == 0
    X = dB.cpu().numpy()
    R = np.array(B0, order="F")
    oracle.dpotrs(np.nan_to_num(T), R, uplo)
    assert colnorm_err(X, R) <= 1e-11
    r = np.linalg.norm(A @ X - B0) / (np.linalg.norm(A) * np.linalg.norm(X))
    assert r <= 100 * n * EPS
    assert np.isnan(dT.cpu().numpy()[other_mask(n, uplo)]).all()


def padded_dev(A, extra):
    """Column-major device view of A inside a (n + extra)-row buffer whose
    padding rows hold NaN (an odd lda: no 16-byte-aligned columns, the plain-load
    paths of the kernels)."""
    m, n = A.shape
    buf = np.full((m + extra, n), np.nan)
    buf[:m] = A
    d = torch.from_numpy(np.ascontiguousarray(buf.T)).cuda().t()
    return d[:m], d


@pytest.mark.parametrize("uplo", ["L", "U"])
def test_next_ops_padded_lda(uplo):
    """trtri, lauum, potrs and getrf on a matrix with lda = n + 3: the same
    parity, and the lda padding (NaN) bitwise untouched."""
    n = 301
    T, A = chol_factor(n, 31, uplo)
    for op in ("trtri", "lauum"):
        dT, full = padded_dev(T, 3)
        assert (rl.dtrtri(dT, uplo, "N") if op == "trtri" else rl.dlauum(dT, uplo)) == 0
        G = dT.cpu().numpy()
        R = np.array(T, order="F")
        if op == "trtri":
            assert oracle.dtrtri(R, uplo, "N") == 0
            assert colnorm_err(tri_part(G, uplo), tri_part(R, uplo)) <= 1e-11
        else:
            oracle.dlauum(R, uplo)
            assert colnorm_err(tri_part(G, uplo), tri_part(R, uplo)) <= 1e-11
        assert np.isnan(full.cpu().numpy()[n:]).all()
        assert np.isnan(G[other_mask(n, uplo)]).all()
    B0 = np.asfortranarray(np.random.default_rng(5).uniform(-1, 1, size=(n, 37)))
    dT, _ = padded_dev(T, 3)
    dB, fullB = padded_dev(B0, 5)
    assert rl.dpotrs(dT, dB, uplo) == 0
    R = np.array(B0, order="F")
    oracle.dpotrs(np.nan_to_num(T), R, uplo)
    assert colnorm_err(dB.cpu().numpy(), R) <= 1e-11
    assert np.isnan(fullB.cpu().numpy()[n:]).all()
    if uplo == "L":
        M = np.asfortranarray(np.random.default_rng(9).uniform(-1, 1, size=(n, n)))
        dM, fullM = padded_dev(M, 3)
        ipiv = torch.zeros(n, dtype=torch.int32, device="cuda")
        assert rl.dgetrf(dM, ipiv) == 0
        R = np.array(M, order="F")
        rinfo, rpiv = oracle.dgetrf(R)
        assert rinfo == 0 and np.array_equal(ipiv.cpu().numpy(), rpiv)
        assert colnorm_err(dM.cpu().numpy(), R) <= 1e-9
        assert np.isnan(fullM.cpu().numpy()[n:]).all()


# ------------------------------------------------------------------ N4 getrf
def apply_ipiv(A, ipiv):
    A = A.copy()
    for j, p in enumerate(ipiv):
        A[[j, p - 1]] = A[[p - 1, j]]
    return A


@pytest.mark.parametrize("m,n", [(1, 1), (5, 5), (32, 32), (33, 33), (100, 100), (300, 300), (1031, 1031),
                                 (2048, 2048), (1500, 700), (700, 1500), (4096, 64), (16384, 48)])
def test_getrf(m, n):
    A = np.asfortranarray(np.random.default_rng(m * 7 + n).uniform(-1, 1, size=(m, n)))
    dA = to_dev(A)
    ipiv = torch.zeros(min(m, n), dtype=torch.int32, device="cuda")
    assert rl.dgetrf(dA, ipiv) == 0
    G = dA.cpu().numpy()
    R = np.array(A, order="F")
    rinfo, rpiv = oracle.dgetrf(R)
    assert rinfo == 0
    assert np.array_equal(ipiv.cpu().numpy(), rpiv), "pivot sequence differs from the oracle's"
    e = colnorm_err(G, R)
    assert e <= 1e-9, e
    k = min(m, n)
    L = np.tril(G[:, :k], -1) + np.eye(m, k)
    Uf = np.triu(G[:k, :])
    r = np.linalg.norm(apply_ipiv(A, ipiv.cpu().numpy()) - L @ Uf) / np.linalg.norm(A)
    assert r <= 100 * max(m, n) * EPS


def test_getrf_singular_and_identity():
    n = 300
    A = np.asfortranarray(np.random.default_rng(3).uniform(-1, 1, size=(n, n)))
    A[:, 100] = 0.0
    dA = to_dev(A)
    ipiv = torch.zeros(n, dtype=torch.int32, device="cuda")
    info = rl.dgetrf(dA, ipiv)
    R = np.array(A, order="F")
    rinfo, rpiv = oracle.dgetrf(R)
    assert info == rinfo == 101
    assert np.array_equal(ipiv.cpu().numpy(), rpiv)
    I = np.asfortranarray(np.eye(77))
    dI = to_dev(I)
    ip = torch.zeros(77, dtype=torch.int32, device="cuda")
    assert rl.dgetrf(dI, ip) == 0
    assert torch.equal(dI.cpu(), torch.eye(77, dtype=torch.float64))
    assert ip.cpu().tolist() == list(range(1, 78))


@pytest.mark.parametrize("cluster", ["16", "8", "poll"])
def test_getrf_panel_variants(cluster):
    """The getrf panels on one thread-block cluster of 16 / 8 CTAs (opt-in
    RELAPACK_GETF2_CLUSTER; narrower leaves for tall panels, interchanges by
    k_permute) and the cooperative panels with the epoch-stamped exchange
    (opt-in RELAPACK_GETF2_POLL) — the knobs are read once per process, so each
    variant runs in a subprocess."""
    import os
    import subprocess
    import sys
    from pathlib import Path

    code = ("from tests.test_gpu_next import test_getrf, test_getrf_singular_and_identity\n"
            "for mn in [(33, 33), (300, 300), (1031, 1031), (1500, 700), (700, 1500), (4096, 64), (16384, 48)]:\n"
            "    test_getrf(*mn)\n"
            "test_getrf_singular_and_identity()\nprint('variant ok')\n")
    env = dict(os.environ, **({"RELAPACK_GETF2_POLL": "1"} if cluster == "poll" else {"RELAPACK_GETF2_CLUSTER": cluster}))
    r = subprocess.run([sys.executable, "-c", code], cwd=Path(__file__).resolve().parents[1], env=env,
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0 and "variant ok" in r.stdout, r.stdout[-2000:] + r.stderr[-4000:]


@pytest.mark.parametrize("window", ["64", "256"])
def test_getrf_lookahead_variant(window):
    """The lookahead getrf plan (RELAPACK_GETRF_LA=1: panel-only cluster
    leaves, each level's P1 laswp / solve / update issued as column pieces,
    deferred pieces serialized at low priority, P2 laswp after the right
    recursion) against the oracle — identical pivots, same factor tolerances;
    window 64 puts the lookahead pieces and the multi-chunk laswp into every
    size here.  In a subprocess (knobs read per plan key)."""
    import os
    import subprocess
    import sys
    from pathlib import Path

    code = ("from tests.test_gpu_next import test_getrf, test_getrf_singular_and_identity\n"
            "for mn in [(33, 33), (300, 300), (1031, 1031), (2048, 2048), (1500, 700), (700, 1500), (4096, 64),"
            " (16384, 48)]:\n"
            "    test_getrf(*mn)\n"
            "test_getrf_singular_and_identity()\nprint('variant ok')\n")
    env = dict(os.environ, RELAPACK_GETRF_LA="1", RELAPACK_GETRF_WINDOW=window)
    r = subprocess.run([sys.executable, "-c", code], cwd=Path(__file__).resolve().parents[1], env=env,
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0 and "variant ok" in r.stdout, r.stdout[-2000:] + r.stderr[-4000:]


def test_tri_leaf_row_kernel_variant():
    """The triangular leaves on the row-per-thread kernel (RELAPACK_TRI_MMA=0)
    instead of the DMMA one: the same parity checks of every operation that
    uses them (trtri L/U and unit, lauum, potri, potrs, getrf), in a subprocess
    (the knob is read once per process)."""
    import os
    import subprocess
    import sys
    from pathlib import Path

    code = ("import tests.test_gpu_next as t\n"
            "for n in (65, 300, 1031):\n"
            "    for u in 'LU':\n"
            "        t.test_trtri(n, u); t.test_lauum(n, u)\n"
            "t.test_trtri_unit_and_integer('L'); t.test_trtri_unit_and_integer('U')\n"
            "t.test_getrf(300, 300); t.test_getrf(1500, 700)\n"
            "print('variant ok')\n")
    env = dict(os.environ, RELAPACK_TRI_MMA="0")
    r = subprocess.run([sys.executable, "-c", code], cwd=Path(__file__).resolve().parents[1], env=env,
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0 and "variant ok" in r.stdout, r.stdout[-2000:] + r.stderr[-4000:]


@pytest.mark.parametrize("cols,rows", [("16", "64"), ("48", "200")])
def test_panel_split_variant(cols, rows):
    """potrs with the right-hand sides in column panels (RELAPACK_POTRS_COLS:
    each panel its own pair of recursive solves) and trtri / lauum / potri with
    the rows of each level's TRMM / TRSM operand in panels (RELAPACK_TRI_ROWS):
    the same parity checks, incl. the untouched other triangle, with panel
    sizes small enough that every size here splits (ragged last panels, panel
    bounds rounded to 8).  In a subprocess (knobs are part of the plan key)."""
    import os
    import subprocess
    import sys
    from pathlib import Path

    code = ("import tests.test_gpu_next as t\n"
            "for u in 'LU':\n"
            "    for n, r in [(65, 7), (300, 100), (1031, 130), (2048, 301)]:\n"
            "        t.test_potrs(n, r, u)\n"
            "    for n in (65, 300, 1031, 2048):\n"
            "        t.test_trtri(n, u); t.test_lauum(n, u)\n"
            "    t.test_potri(1500, u); t.test_trtri_unit_and_integer(u)\n"
            "t.test_trtri_blocked(1031, 128)\n"
            "print('variant ok')\n")
    env = dict(os.environ, RELAPACK_POTRS_COLS=cols, RELAPACK_TRI_ROWS=rows)
    r = subprocess.run([sys.executable, "-c", code], cwd=Path(__file__).resolve().parents[1], env=env,
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0 and "variant ok" in r.stdout, r.stdout[-2000:] + r.stderr[-4000:]


@pytest.mark.parametrize("order", ["0", "1"])
def test_trtri_order_variant(order):
    """trtri in the paper's step order (RELAPACK_TRTRI_ORDER=0: trtri(A_TL),
    trmm, trsm, trtri(A_BR) — one chain) and with the level's solve first (1,
    the default: A_BL := A_BR^{-1} A_BL with the original A_BR, both recursive
    calls side by side in the DAG, then A_BL := -A_BL A_TL^{-1}): the same
    inverse up to rounding order — the same parity checks against the oracle
    (which keeps the paper's order), the exact integer / unit cases, singular
    info, potri.  In a subprocess with the knob set explicitly."""
    import os
    import subprocess
    import sys
    from pathlib import Path

    code = ("import tests.test_gpu_next as t\n"
            "for u in 'LU':\n"
            "    for n in (1, 7, 64, 65, 100, 300, 1031, 2048):\n"
            "        t.test_trtri(n, u)\n"
            "    t.test_potri(1500, u); t.test_trtri_unit_and_integer(u)\n"
            "t.test_trtri_singular(); t.test_potri_after_potrf_on_gpu()\n"
            "print('variant ok')\n")
    env = dict(os.environ, RELAPACK_TRTRI_ORDER=order)
    r = subprocess.run([sys.executable, "-c", code], cwd=Path(__file__).resolve().parents[1], env=env,
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0 and "variant ok" in r.stdout, r.stdout[-2000:] + r.stderr[-4000:]


# ------------------------------------------------------------------ N2 blocked dpotrf
@pytest.mark.parametrize("uplo", ["L", "U"])
@pytest.mark.parametrize("nb", [64, 128, 256])
@pytest.mark.parametrize("n", [300, 1031, 2048])
def test_potrf_blocked(n, nb, uplo):
    A = np.asfortranarray(gen.spd(n, 21))
    dA = to_dev(A)
    assert rl.dpotrf_blocked(dA, nb, uplo) == 0
    G = dA.cpu().numpy()
    R = np.array(A, order="F")
    assert oracle.dpotrf(R, uplo) == 0
    Lg = np.tril(G) if uplo == "L" else np.tril(G.T)
    Lo = np.tril(R) if uplo == "L" else np.tril(R.T)
    assert floored_rel_err(Lg, Lo, A) <= 1e-10


def test_potrf_blocked_info():
    n = 700
    A = np.asfortranarray(gen.spd(n, 22))
    A[400, 400] = -A[400, 400]
    dA = to_dev(A)
    assert rl.dpotrf_blocked(dA, 128, "L") == 401
