"""Kernel-level parity: every instantiation of the
update kernel (K3 GEMM / K4 SYRK) and every TRSM base variant (K5) the plan can
launch, called once through the C-ABI test hooks with the size-rule choices
forced (CTA tile 32/64/128, TMA or plain-load operands, split-K), against the
oracle's BLAS-3 definitions (oracle_dgemm_nt / dsyrk_ln / dtrsm_rlt)
on the same seeded inputs, element by element.

Tolerances (derived):
* GEMM/SYRK: both sides compute c + alpha * sum_k a_ik b_jk in FP64 with a
  different summation order; the standard dot-product bound gives
  |Cg - Co| <= 2 (K + 2) u (|C0| + |A| |B|^T), u = 2^-53, elementwise.
* TRSM: x = b L^{-T} with L the Cholesky factor of a kappa ~ 2.3 SPD matrix;
  forward error <= kappa(L) t u per row scale: max_j |Xg - Xo|_ij /
  max_j |Xo|_ij <= 1e-12 (measured ~1e-15).
Elements outside the updated part (the other triangle, ld padding) must be
bitwise unchanged.
"""
import itertools

import numpy as np
import pytest
import torch

import oracle
import paper_1602_06763_b200 as rl
from inputs import gen

pytestmark = pytest.mark.gpu

U = 2.0 ** -53


def _operand(X: np.ndarray, layout: int, pad: int = 0, odd_offset: bool = False) -> torch.Tensor:
    """Device tensor with the values of X in the given layout (0 column-major,
    1 row-major), leading dimension padded by `pad` (NaN padding), optionally
    starting one element into its allocation (base not 16-byte aligned)."""
    r, c = X.shape
    off = 1 if odd_offset else 0
    if layout == 0:
        ld = r + pad
        buf = torch.full((ld * max(c, 1) + off,), float("nan"), dtype=torch.float64, device="cuda")
        T = buf[off:off + ld * c].view(c, ld).t()[:r, :] if c > 0 else buf[:0].view(r, 0)
    else:
        ld = c + pad
        buf = torch.full((ld * max(r, 1) + off,), float("nan"), dtype=torch.float64, device="cuda")
        T = buf[off:off + ld * r].view(r, ld)[:, :c] if r > 0 else buf[:0].view(0, c)
    T.copy_(torch.from_numpy(X))
    return T, buf


def _rand(shape, seed, stream):
    g = gen.philox(seed, stream)
    return g.uniform(-1.0, 1.0, size=shape)


def _run_update(M, N, K, la, lb, lc, tri, tile, tma, ksplit, alpha=-1.0, pad=0, odd=False, seed=7, ctas=0, full=0):
    A = _rand((M, K), seed, 1)
    B = A.copy() if (tri and seed % 2 == 0 and M == N) else _rand((N, K), seed, 2)
    C0 = _rand((M, N), seed, 3) * 4.0
    tA, _ = _operand(A, la, pad, odd)
    tB, _ = _operand(B, lb, pad)
    tC, bufC = _operand(C0, lc, pad)
    before = bufC.clone()
    chosen = rl.update_test(tC, tA, tB, alpha=alpha, tri=tri, tile=tile, ksplit=ksplit, tma=tma, ctas=ctas, full=full)
    torch.cuda.synchronize()
    Cg = tC.cpu().numpy()
    # oracle: C -= A' B^T with A' = -alpha A (alpha a power of two: exact scaling)
    Co = np.asfortranarray(C0.copy())
    oracle.dgemm_nt(np.asfortranarray(-alpha * A), np.asfortranarray(B), Co)
    bound = 2 * (K + 2) * U * (np.abs(C0) + np.abs(alpha) * (np.abs(A) @ np.abs(B).T))
    if tri == 1:
        keep = np.tril(np.ones((M, N), dtype=bool))
    elif tri == 2:
        keep = np.triu(np.ones((M, N), dtype=bool))
    else:
        keep = np.ones((M, N), dtype=bool)
    err = np.abs(Cg - Co)
    bad = keep & ~(err <= bound)
    assert not bad.any(), (
        f"update M={M} N={N} K={K} la={la} lb={lb} lc={lc} tri={tri} tile={tile} tma={tma} ks={ksplit}: "
        f"{int(bad.sum())} elements outside the bound, max err/bound {float(np.max(err[keep] / np.maximum(bound[keep], 1e-300))):.3g}")
    # the other triangle bitwise untouched, and the padding too
    assert np.array_equal(Cg[~keep], C0[~keep])
    after = bufC.cpu().numpy()
    pad_mask = np.isnan(before.cpu().numpy())
    assert np.isnan(after[pad_mask]).all(), "padding written"
    return chosen


SIZES = (1, 7, 63, 65, 129)
HOT = ((0, 0, 0), (1, 1, 1))  # the factorization's (la, lb, lc) for uplo L / U


@pytest.mark.parametrize("lay", HOT)
@pytest.mark.parametrize("tma", (True, False))
@pytest.mark.parametrize("full,ksplit,ctas", [(10, 2, 0), (13, 3, 0), (1, 4, 0), (9, 2, 4)])
def test_update_tail_split(lay, tma, full, ksplit, ctas):
    """Tail split: tiles [0, full) whole, the rest split ksplit ways (the plan's
    last-partial-wave split), also under a CTA cap; GEMM (16 tiles) and SYRK
    (10 lower tiles) on ragged 128-tiles."""
    la, lb, lc = lay
    for tri in (0, 1):
        M = N = 3 * 128 + 17
        f = full if tri == 0 else min(full, 9)  # 16 GEMM tiles, 10 SYRK tiles
        chosen = _run_update(M, N, 300, la, lb, lc, tri, 128, tma, ksplit, ctas=ctas, full=f, seed=21 + tri)
        assert chosen[0] == 128 and chosen[2] == ksplit


@pytest.mark.parametrize("lay", HOT)
def test_update_tail_split_size_rule(lay):
    """The size rule's own tail split: 169 tiles of 128 = one wave of 148 plus
    21, split 4 ways (K = 512: 8 k-tiles a piece)."""
    la, lb, lc = lay
    chosen = _run_update(13 * 128, 13 * 128, 512, la, lb, lc, 0, 128, True, 0, seed=5)
    assert chosen[0] == 128 and chosen[2] == 4


@pytest.mark.parametrize("lay", HOT)
@pytest.mark.parametrize("tile", (64, 128))
@pytest.mark.parametrize("tma", (True, False))
@pytest.mark.parametrize("ctas,ksplit", [(3, 1), (7, 1), (5, 3)])
def test_update_persistent_ctas(lay, tile, tma, ctas, ksplit):
    """Persistent CTAs (the plan's CTA-capped deferred updates): each CTA runs
    several (tile, split) items through the same shared-memory ring, the TMA of
    an item writing the bytes the previous item's fragment reads and epilogue
    staging used (generic -> async proxy, fenced).  GEMM and SYRK."""
    la, lb, lc = lay
    for tri in (0, 1):
        M = N = 3 * tile + 17
        chosen = _run_update(M, N, 200, la, lb, lc, tri, tile, tma, ksplit, ctas=ctas, seed=11 + tri)
        assert chosen[0] == tile and chosen[2] == ksplit


@pytest.mark.parametrize("lay", HOT)
@pytest.mark.parametrize("tile", (32, 64, 128))
@pytest.mark.parametrize("tma", (True, False))
def test_update_hot_instantiations(lay, tile, tma):
    """Every k_update<layout, tma, tile> the factorization launches: GEMM and
    SYRK (tri 1), ragged M/N/K across several tiles, with and without split-K."""
    la, lb, lc = lay
    cases = [(300, 260, 129, 0, 1), (260, 260, 65, 1, 1), (200, 130, 7, 0, 1), (129, 129, 1, 1, 1),
             (300, 300, 2049, 1, 4), (300, 140, 2049, 0, 3), (65, 63, 63, 0, 2)]
    for M, N, K, tri, ks in cases:
        ch = _run_update(M, N, K, la, lb, lc, tri, tile, tma, ks)
        assert ch[0] == tile and ch[2] == ks
        # TMA needs even leading dimensions (layout 0: ld = rows, 1: ld = K)
        even = (K % 2 == 0) if la == 1 else (M % 2 == 0 and N % 2 == 0)
        assert bool(ch[1]) == (tma and even), f"TMA path expected {tma and even}, got {ch}"


@pytest.mark.parametrize("lay", HOT)
def test_update_size_rule(lay):
    """The plan's own choices (tile / split-K by size rule) on the shapes of the
    n = 16384 plan's top levels, scaled down to oracle-friendly K."""
    la, lb, lc = lay
    for M, N, K, tri in ((2048, 2048, 256, 1), (2048, 1024, 384, 0), (512, 512, 1024, 1), (4096, 128, 128, 0),
                         (1536, 1536, 64, 1)):
        _run_update(M, N, K, la, lb, lc, tri, 0, True, 0)


@pytest.mark.parametrize("M,N,K", list(itertools.product(SIZES, SIZES, (1, 65))) + [(129, 129, 2049)])
def test_update_shapes_sweep(M, N, K):
    """Ragged shape sweep (m, n, k in {1, 7, 63, 65, 129}), both hot layouts, size-rule tiles."""
    for la in (0, 1):
        _run_update(M, N, K, la, la, la, 0, 0, True, 0, seed=M * 1000 + N)
        if M == N:
            _run_update(M, N, K, la, la, la, 1, 0, True, 0, seed=M * 1000 + N + 1)


def test_update_odd_ld_and_misaligned():
    """Odd leading dimension and a base off 16-byte alignment fall back to the plain-load path."""
    for la in (0, 1):
        # odd ld: layout 0 has ld = rows + pad (200 + 1, 170 + 1), layout 1 ld = K + pad (129 + 2)
        ch = _run_update(200, 170, 129, la, la, la, 0, 0, True, 1, pad=1 if la == 0 else 2)
        assert ch[1] == 0
        ch = _run_update(200, 170, 129, la, la, la, 0, 0, True, 1, odd=True)
        assert ch[1] == 0
        ch = _run_update(170, 170, 129, la, la, la, 1, 0, True, 1, pad=2 if la == 0 else 1)
        assert ch[1] == 1


@pytest.mark.parametrize("lay", [(0, 1, 0), (1, 0, 0), (1, 1, 0), (0, 0, 1), (0, 1, 1), (1, 0, 1)])
@pytest.mark.parametrize("tri", (0, 1, 2))
def test_update_mixed_layouts(lay, tri):
    """Mixed operand layouts (used by trtri / lauum / potrs / getrf), alpha = +-1, +-0.5,
    lower / upper triangle, every tile, TMA and plain loads."""
    la, lb, lc = lay
    for tile in (32, 64, 128):
        for tma in (True, False):
            for alpha in (-1.0, 1.0, -0.5):
                M = N = 150 if tri else 150
                _run_update(M, N if tri else 97, 70, la, lb, lc, tri, tile, tma, 1, alpha=alpha, seed=tile + int(tma))
    _run_update(300, 300, 2049, la, lb, lc, tri, 0, True, 0)


# ------------------------------------------------------------------ K5 TRSM base
def _chol_factor(t, seed):
    A = gen.spd(t, seed)
    L = np.array(A, order="F")
    assert oracle.dpotrf(L, "L") == 0
    return np.tril(L)


def _run_trsm(m, t, layout, variant, seed=3):
    L = _chol_factor(t, seed)
    B = _rand((m, t), seed, 5)
    # device blocks: layout 0 = column-major (uplo L), 1 = row-major L-view (uplo U)
    full = L + np.triu(np.full((t, t), np.nan), 1)  # NaN above the diagonal: must never be read
    tL, _ = _operand(full, layout)
    tB, _ = _operand(B, layout)
    rl.trsm_test(tL, tB, variant)
    torch.cuda.synchronize()
    Xg = tB.cpu().numpy()
    Xo = np.asfortranarray(B.copy())
    oracle.dtrsm_rlt(np.asfortranarray(L), Xo)
    if m == 0:
        return
    scale = np.maximum(np.max(np.abs(Xo), axis=1, keepdims=True), 1e-300)
    e = float(np.max(np.abs(Xg - Xo) / scale))
    assert np.isfinite(Xg).all() and e <= 1e-12, f"trsm m={m} t={t} layout={layout} variant={variant}: {e:.3e}"


@pytest.mark.parametrize("layout", (0, 1))
@pytest.mark.parametrize("variant", (0, 1, 2, 3, 4, 5))
def test_trsm_variants(layout, variant):
    ts = (8, 17, 64, 100, 128) + ((200, 256) if variant in (4, 5) else ())
    for t in ts:
        for m in (1, 7, 65, 2049):
            _run_trsm(m, t, layout, variant)


@pytest.mark.parametrize("layout", (0, 1))
def test_trsm_rowparallel(layout):
    for t in (1, 8, 33, 64):
        for m in (1, 33, 130, 2047, 4100):
            _run_trsm(m, t, layout, 6)


def test_trsm_tall_panel():
    """The panel height of the n = 16384 plan's top TRSM bases (8192 rows) on the 64-row CTAs."""
    for layout in (0, 1):
        _run_trsm(8192, 128, layout, 0)


# ------------------------------------------------------------------ K1 base case
@pytest.mark.parametrize("layout", (0, 1))
def test_potf2_kernel_sizes(layout):
    for n in (1, 2, 31, 32, 33, 64, 65, 100, 127, 128):
        A = gen.spd(n, n)
        full = np.tril(A) + np.triu(np.full((n, n), np.nan), 1) if layout == 0 else np.triu(A) + np.tril(
            np.full((n, n), np.nan), -1)
        tA, _ = _operand(full, 0)
        info = rl.potf2_test(tA if layout == 0 else tA.t())
        assert info == 0
        R = np.array(A, order="F")
        assert oracle.dpotrf(R, "L" if layout == 0 else "U") == 0
        G = tA.cpu().numpy()
        Lg = np.tril(G) if layout == 0 else np.tril(G.T)
        Lo = np.tril(R) if layout == 0 else np.tril(R.T)
        floor = 1e-4 * np.sqrt(np.diag(A))[:, None]
        e = float(np.max(np.tril(np.abs(Lg - Lo) / np.maximum(np.abs(Lo), floor))))
        assert e <= 1e-10
        other = np.triu(G, 1) if layout == 0 else np.tril(G, -1)
        assert np.isnan(other[np.triu(np.ones((n, n), bool), 1) if layout == 0 else np.tril(np.ones((n, n), bool), -1)]).all()
