"""Host-only checks of the §8(f) launch plans (no GPU): the getrf lookahead
plan is the same recursion with its right-part work issued as
column pieces, so its leading-term flops equal the plain recursion's and the
closed form m n^2 - n^3/3 (square: 2 n^3 / 3); its row interchanges are the
P1 / P2 laswp calls of the levels above the windows and the per-leaf
permutations inside them."""
import pytest

import paper_1602_06763_b200 as rl

GETF2, LASWP, PERM = rl.XKINDS["getf2"], rl.XKINDS["laswp"], rl.XKINDS["perm"]


@pytest.mark.parametrize("n", [1, 100, 512, 1031, 4096, 16384])
@pytest.mark.parametrize("window", [0, 64, 256])
def test_getrf_lookahead_plan_flops(n, window):
    c5, k5, f5 = rl.xplan_count("getrf", n)
    c6, k6, f6 = rl.xplan_count("getrf_la", n, window)
    assert f6 == pytest.approx(f5, rel=1e-12)
    assert f6 == pytest.approx(2.0 * n ** 3 / 3.0, rel=1e-12)
    # leaves: 16 columns while the panel has > 8192 rows (16-CTA cluster), else 32
    assert k6.count(GETF2) == k5.count(GETF2) or n > 8192
    w = window or 256
    if n <= w:
        assert LASWP not in k6  # one window: eager interchanges only
    else:
        assert k6.count(LASWP) > 0


def test_getrf_lookahead_plan_bounds():
    with pytest.raises(ValueError):
        rl.xplan_count("getrf_la", 16 * 2048 + 16)  # beyond the 16-CTA cluster panel's rows


@pytest.mark.parametrize("op,n,nb", [("potrs", 4096, 1000), ("potrs", 1031, 130), ("trtri", 4096, 0),
                                     ("lauum", 1031, 0), ("potri", 2048, 0)])
def test_panel_split_plan_flops(op, n, nb, monkeypatch):
    """Right-hand-side panels (potrs) / operand-row panels (trtri, lauum) are
    the same recursion on independent rows: the plan's leading-term flops do not
    change (potrs: 2 n^2 nrhs; trtri, lauum: n^3 / 3 each) and the launch count grows."""
    monkeypatch.setenv("RELAPACK_POTRS_COLS", "0")
    monkeypatch.setenv("RELAPACK_TRI_ROWS", "0")
    c0, _, f0 = rl.xplan_count(op, n, nb)
    monkeypatch.setenv("RELAPACK_POTRS_COLS", "64")
    monkeypatch.setenv("RELAPACK_TRI_ROWS", "128")
    c1, _, f1 = rl.xplan_count(op, n, nb)
    assert f1 == pytest.approx(f0, rel=1e-12)
    closed = {"potrs": 2.0 * n * n * nb, "trtri": n ** 3 / 3.0, "lauum": n ** 3 / 3.0, "potri": 2 * n ** 3 / 3.0}[op]
    assert f0 == pytest.approx(closed, rel=1e-12)
    assert c1 > c0


@pytest.mark.parametrize("n", [65, 1031, 4096])
def test_trtri_solve_first_plan(n, monkeypatch):
    """RELAPACK_TRTRI_ORDER=1 reorders a level's four steps; the launches and their flops are the same multiset."""
    monkeypatch.setenv("RELAPACK_TRTRI_ORDER", "0")
    c0, k0, f0 = rl.xplan_count("trtri", n)
    monkeypatch.setenv("RELAPACK_TRTRI_ORDER", "1")
    c1, k1, f1 = rl.xplan_count("trtri", n)
    assert c1 == c0 and sorted(k1) == sorted(k0) and f1 == pytest.approx(f0, rel=1e-12)
    assert k1 != k0 or n <= 64
