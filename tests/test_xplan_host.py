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
