"""CPU-only checks of the boundary and the host recursion driver (no GPU):
the C-ABI library loads and exports every symbol include/relapack.h declares,
argument errors follow LAPACK, and the plan the driver builds has the split
rule and FLOP-share ladder the paper fixes."""
import ctypes
import os

import numpy as np
import pytest

import paper_1602_06763_b200 as rl

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module", autouse=True)
def built():
    from paper_1602_06763_b200 import build

    build.build()


def test_library_exports_every_declared_symbol():
    syms = rl.declared_symbols()
    assert len(syms) >= 15
    L = rl.lib()
    for s in syms:
        assert hasattr(L, s), s


def test_product_library_does_not_link_oracle():
    data = open(rl.library_path, "rb").read()
    assert b"oracle_dpotrf" not in data


def test_split_point_spec_examples():
    for line in open(os.path.join(GOLDEN, "split_point_spec_examples.txt")):
        if line.startswith("#") or not line.strip():
            continue
        n, n1, n2 = map(int, line.split())
        assert rl.split_point(n, 8) == n1
        assert n - rl.split_point(n, 8) == n2


def test_split_point_invariants():
    for align in (8, 16, 64):
        for n in range(2, 600):
            n1 = rl.split_point(n, align)
            assert 1 <= n1 <= n - 1
            assert n1 <= n // 2 + 0  # rounding down keeps the second call the larger one
            if n >= 2 * align:
                assert n1 % align == 0
            elif n >= 16:
                assert n1 % 8 == 0
    assert rl.split_point(1, 8) == -1


def _ladder():
    rows = []
    for line in open(os.path.join(GOLDEN, "flop_share_ladder.txt")):
        if line.startswith("#") or not line.strip():
            continue
        lvl, exact, printed = line.split()
        rows.append((int(lvl), float(exact), float(printed)))
    return rows


@pytest.mark.parametrize("n,c", [(2048, 64), (4096, 64), (16384, 128), (1024, 32), (65536, 64)])
def test_flop_share_ladder_matches_paper(n, c):
    """level-l share of the two BLAS-3 calls is 3/4^l (75, 18.8, 4.69, 1.17 %)."""
    total = n**3 / 3.0
    depth, by_level, base, launches = rl.plan_ledger(n, c, 64, 12)
    assert depth == int(np.log2(n // c))
    for lvl, exact, printed in _ladder():
        share = by_level[lvl - 1] / total
        assert share == pytest.approx(exact, rel=1e-12)
        assert round(100 * share, 2 if printed < 10 else 1) == pytest.approx(printed, abs=0.011)
    assert base / total == pytest.approx(c * c / n**2, rel=1e-12)
    assert (sum(by_level) + base) / total == pytest.approx(1.0, rel=1e-12)
    # > 99.6 % of the flops in BLAS-3 for c < 100
    if c < 100:
        assert sum(by_level) / total > 0.996


def test_ledger_crossover_invariance():
    """total flops do not depend on the crossover (leading-term model)."""
    tot = []
    for c in (16, 32, 64, 128):
        _, by_level, base, _ = rl.plan_ledger(1024, c, 64, 12)
        tot.append(sum(by_level) + base)
    assert max(tot) - min(tot) <= 1e-6 * tot[0]


def test_launch_count_scales():
    _, _, _, k4096 = rl.plan_ledger(4096, 64, 64, 12)
    _, _, _, k256 = rl.plan_ledger(256, 64, 64, 12)
    assert k256 < k4096


def test_argument_errors_without_gpu():
    """LAPACK info codes for bad arguments are returned before any device work."""
    buf = np.zeros(16)
    p = buf.ctypes.data
    assert rl.dpotrf_raw("X", 2, p, 2) == -1
    assert rl.dpotrf_raw("L", -1, p, 2) == -2
    assert rl.dpotrf_raw("L", 2, 0, 2) == -3
    assert rl.dpotrf_raw("L", 4, p, 3) == -4
    assert rl.dpotrf_raw("U", 0, p, 0) == -4
    assert rl.dpotrf_raw("u", 0, p, 1) == 0  # quick return


def test_knobs():
    old = rl.get_crossover()
    assert old == 128  # default: the in-CTA 128-node base case (256-node kernel opt-in)
    with pytest.raises(ValueError):
        rl.set_crossover(8)
    with pytest.raises(ValueError):
        rl.set_split_tile(48)
    with pytest.raises(ValueError):
        rl.set_crossover(300)  # the base case lives in one SM's shared memory: c <= 256
    rl.set_crossover(48)
    assert rl.get_crossover() == 48
    rl.set_crossover(old)
