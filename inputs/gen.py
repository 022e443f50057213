"""Seeded synthetic inputs for the recursive Cholesky hot path.

Recipe (BASELINE.json configs; SURVEY §8c.3 #10-#12,
§8d):

* random SPD  A = tril(B B^T) mirrored + n I, B i.i.d. Uniform(-1, 1) or N(0, 1)
  drawn from numpy's counter-based Philox generator keyed by (seed, stream).
  The matrix is exactly symmetric (the upper triangle is a bitwise mirror of
  the lower one) so uplo='L' and uplo='U' see identical values.  kappa(A) is
  about 2.3 (uniform) / 5 (normal); every pivot is >= n.
* integer case (CFG[0]): L integer lower-triangular, diag U{1..4}, off-diag
  U{-2..2}; A = L L^T computed exactly in int64.
* batched (CFG[4]): sizes U{16,32,48,64}; 1 % of the matrices (a seeded
  choice) get one diagonal entry negated, A_kk <- -A_kk, which makes info =
  k+1 exactly.

Large products B B^T are computed on the GPU with torch (cuBLAS) when a CUDA
device is requested: input construction is test/bench harness, not the
product path.  Whatever produced A, the same A bits are handed to both the
oracle and the CUDA path.
"""
from __future__ import annotations

import numpy as np

__all__ = [
    "philox",
    "draw_B",
    "spd",
    "spd_torch",
    "integer_L",
    "min_matrix",
    "pascal",
    "indefinite",
    "batched_spd",
    "BATCH_SIZES",
]

BATCH_SIZES = (16, 32, 48, 64)


def philox(seed: int, stream: int = 0) -> np.random.Generator:
    """Counter-based generator keyed by (seed, stream): independent, reproducible streams."""
    return np.random.Generator(np.random.Philox(key=[int(seed) & (2**64 - 1), int(stream) & (2**64 - 1)]))


def draw_B(n: int, seed: int, dist: str = "uniform", m: int | None = None, stream: int = 0) -> np.ndarray:
    """n x m (default n x n) matrix of i.i.d. Uniform(-1,1) or N(0,1) draws."""
    m = n if m is None else m
    g = philox(seed, stream)
    if dist == "uniform":
        return 2.0 * g.random((n, m)) - 1.0
    if dist == "normal":
        return g.standard_normal((n, m))
    raise ValueError(f"unknown distribution {dist!r}")


def _symmetrize_lower(M: np.ndarray) -> np.ndarray:
    """Exactly symmetric copy built from the lower triangle of M (Fortran order)."""
    L = np.tril(M)
    A = L + np.tril(L, -1).T  # x + 0.0 == x exactly
    return np.asfortranarray(A)


def spd(n: int, seed: int, dist: str = "uniform", lda: int | None = None, device=None):
    """A = B B^T + n I (exactly symmetric), column-major float64.

    Returns a numpy Fortran-ordered (lda x n) array when device is None, else a
    torch tensor on `device` with column-major strides (1, lda).
    """
    if device is not None:
        return spd_torch(n, seed, dist=dist, lda=lda, device=device)
    lda = n if lda is None else lda
    B = draw_B(n, seed, dist)
    A = _symmetrize_lower(B @ B.T)
    A[np.diag_indices(n)] += float(n)
    if lda == n:
        return A
    out = np.full((lda, n), np.nan, dtype=np.float64, order="F")
    out[:n, :] = A
    return out


def spd_torch(n: int, seed: int, dist: str = "uniform", lda: int | None = None, device="cuda"):
    """Same recipe, product on the device (for n >= 4096).  Column-major (1, lda) strides."""
    import torch

    lda = n if lda is None else lda
    panel = 4096  # B is drawn in row panels, panel p from Philox stream 1 + p (any panel is independent)
    B = torch.empty((n, n), dtype=torch.float64, device=device)
    for p, r0 in enumerate(range(0, n, panel)):
        r1 = min(n, r0 + panel)
        B[r0:r1] = torch.from_numpy(draw_B(r1 - r0, seed, dist, m=n, stream=1 + p)).to(device)
    M = B @ B.T
    del B
    # exact symmetry: mirror the lower triangle onto the upper one, tile by tile (in place)
    for i0 in range(0, n, panel):
        for j0 in range(i0 + panel, n, panel):
            M[i0:i0 + panel, j0:j0 + panel] = M[j0:j0 + panel, i0:i0 + panel].T
        blk = M[i0:i0 + panel, i0:i0 + panel]
        blk.copy_(torch.tril(blk) + torch.tril(blk, -1).T)
    M.diagonal().add_(float(n))
    # M is symmetric, so its row-major storage equals the column-major one.
    if lda == n:
        return M.T  # strides (1, n): column-major view
    out = torch.full((n, lda), float("nan"), dtype=torch.float64, device=device)
    out[:, :n] = M
    return out.T[:n, :]  # (n, n) with strides (1, lda)


def integer_L(n: int, seed: int):
    """(A, L): L integer lower-triangular (diag U{1..4}, off-diag U{-2..2}), A = L L^T exact."""
    g = philox(seed, 7)
    L = np.tril(g.integers(-2, 3, size=(n, n), dtype=np.int64), -1)
    L[np.diag_indices(n)] = g.integers(1, 5, size=n, dtype=np.int64)
    A = L @ L.T  # exact in int64
    return np.asfortranarray(A.astype(np.float64)), np.asfortranarray(L.astype(np.float64))


def min_matrix(n: int) -> np.ndarray:
    """A_ij = min(i, j) + 1, whose Cholesky factor is tril(ones) exactly."""
    i = np.arange(n)
    return np.asfortranarray(np.minimum.outer(i, i).astype(np.float64) + 1.0)


def pascal(n: int) -> np.ndarray:
    """Symmetric Pascal matrix S_ij = C(i+j, i); Cholesky factor L_ij = C(i, j)."""
    from math import comb

    S = np.empty((n, n), dtype=np.float64, order="F")
    for i in range(n):
        for j in range(n):
            S[i, j] = float(comb(i + j, i))
    return S


def indefinite(A: np.ndarray, k: int) -> np.ndarray:
    """Copy of A with A_kk negated: for the configs' SPD matrices info = k+1 exactly."""
    B = np.array(A, order="F", copy=True)
    B[k, k] = -B[k, k]
    return B


def batched_spd(count: int, seed: int, sizes=BATCH_SIZES, frac_indefinite: float = 0.01):
    """CFG[4] batch, packed back to back with lda = n_b.

    Returns dict(ns, offsets, buf, bad_index, expected_info):
      buf        flat float64 buffer, matrix b column-major at offsets[b]
      bad_index  per-matrix negated diagonal index k, or -1
      expected_info  k+1 for the indefinite ones, 0 otherwise (closed form)
    """
    g = philox(seed, 11)
    ns = g.choice(np.asarray(sizes, dtype=np.int32), size=count).astype(np.int32)
    offsets = np.zeros(count, dtype=np.int64)
    if count:
        offsets[1:] = np.cumsum(ns.astype(np.int64) ** 2)[:-1]
    total = int((ns.astype(np.int64) ** 2).sum())
    buf = np.empty(total, dtype=np.float64)
    for nb in sorted(set(int(x) for x in ns)):
        idx = np.nonzero(ns == nb)[0]
        gb = philox(seed, 1000 + nb)
        Bs = 2.0 * gb.random((len(idx), nb, nb)) - 1.0
        M = Bs @ np.transpose(Bs, (0, 2, 1))
        Lt = np.tril(M)
        A = Lt + np.transpose(np.tril(Lt, -1), (0, 2, 1))
        A[:, np.arange(nb), np.arange(nb)] += float(nb)
        # column-major: element (i, j) at i + j*nb -> store A^T row-major == A (symmetric)
        for t, b in enumerate(idx):
            buf[offsets[b]: offsets[b] + nb * nb] = A[t].T.reshape(-1)
    nbad = int(round(frac_indefinite * count))
    bad = np.full(count, -1, dtype=np.int64)
    chosen = g.permutation(count)[:nbad]
    for b in chosen:
        nb = int(ns[b])
        k = int(g.integers(0, nb))
        bad[b] = k
        buf[offsets[b] + k + k * nb] = -buf[offsets[b] + k + k * nb]
    expected = np.where(bad >= 0, bad + 1, 0).astype(np.int32)
    return dict(ns=ns, offsets=offsets, buf=buf, bad_index=bad, expected_info=expected, ldas=ns.copy())
