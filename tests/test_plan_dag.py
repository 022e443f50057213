"""CPU checks of the dependency DAG the executor captures its CUDA graph with
(driver.cu capture_dag, plan.cpp compute_deps): the graph may run any
topological order of the plan's launches, so

  * every pair of launches whose footprints conflict (write/write,
    write/read, read/write) must be ordered by a path in the DAG, and
  * executing the launches in random topological orders (numpy, the plan's
    own block operations: P:366-370 potf2 / trsm / syrk, P:292-295 the TRSM
    recursion's GEMM) must give the Cholesky factor.

Footprints are re-derived here from the launch fields, not taken from C++."""
import random

import numpy as np
import pytest
import scipy.linalg as sla

import paper_1602_06763_b200 as rl
from inputs.gen import spd


@pytest.fixture(scope="module", autouse=True)
def built():
    from paper_1602_06763_b200 import build

    build.build()


def footprint(op):
    """(written rect, [read rects]) as (r0, r1, c0, c1) in L-view coordinates."""
    k, ci, cj, ai, aj, bi, bj = op["kind"], op["c_i"], op["c_j"], op["a_i"], op["a_j"], op["b_i"], op["b_j"]
    m, n, kk = op["m"], op["n"], op["k"]
    if k == "potf2":
        return (ci, ci + n, cj, cj + n), []
    if k == "trsm":
        return (ci, ci + m, cj, cj + kk), [(ai, ai + kk, aj, aj + kk)]
    if k == "gemm":
        return (ci, ci + m, cj, cj + n), [(ai, ai + m, aj, aj + kk), (bi, bi + n, bj, bj + kk)]
    if k == "syrk":
        return (ci, ci + n, cj, cj + n), [(ai, ai + n, aj, aj + kk)]
    raise AssertionError(k)


def overlap(a, b):
    return a[0] < b[1] and b[0] < a[1] and a[2] < b[3] and b[2] < a[3]


def ancestors(deps):
    anc = []
    for j, d in enumerate(deps):
        s = set()
        for i in d:
            assert i < j
            s.add(i)
            s |= anc[i]
        anc.append(s)
    return anc


CASES = [(300, 32, 16, True), (777, 64, 64, True), (1234, 64, 64, False), (1234, 48, 32, True), (2048, 64, 64, True)]


@pytest.mark.parametrize("n,c,T,la", CASES)
def test_dag_orders_every_conflict(n, c, T, la):
    ops, deps = rl.plan_schedule(n, c, T, la)
    assert len(ops) == len(deps) > 0
    fp = [footprint(o) for o in ops]
    anc = ancestors(deps)
    for j in range(len(ops)):
        wj, rj = fp[j]
        for i in range(j):
            wi, ri = fp[i]
            conflict = overlap(wi, wj) or any(overlap(wi, r) for r in rj) or any(overlap(r, wj) for r in ri)
            if conflict:
                assert i in anc[j], (i, j, ops[i], ops[j])
    # direct edges are real conflicts (no spurious serialisation) and reduced
    for j, d in enumerate(deps):
        for i in d:
            wi, ri = fp[i]
            wj, rj = fp[j]
            assert overlap(wi, wj) or any(overlap(wi, r) for r in rj) or any(overlap(r, wj) for r in ri)
            assert not any(i in anc[q] for q in d if q != i), "edge implied by another predecessor"


def test_lookahead_marks_deferred_trailing_updates():
    ops, _ = rl.plan_schedule(4096, 64, 64, True)
    deferred = [o for o in ops if o["deferred"]]
    assert deferred and all(o["kind"] in ("gemm", "syrk") for o in deferred)
    ops0, _ = rl.plan_schedule(4096, 64, 64, False)
    assert not any(o["deferred"] for o in ops0)
    # same total leading-term work either way: sum of trailing-update flops
    def upd_flops(os_):
        f = 0
        for o in os_:
            if o["kind"] == "syrk":
                f += o["n"] ** 2 * o["k"]
            elif o["kind"] == "gemm":
                f += 2 * o["m"] * o["n"] * o["k"]
        return f

    assert upd_flops(ops) == upd_flops(ops0)


def run_order(A, ops, order):
    """Execute the plan's launches on the lower-triangle L-view of A (in place)."""
    for q in order:
        o = ops[q]
        k = o["kind"]
        if k == "potf2":
            i, n = o["c_i"], o["n"]
            blk = np.tril(A[i:i + n, i:i + n])
            blk = blk + np.tril(blk, -1).T
            A[i:i + n, i:i + n] = np.linalg.cholesky(blk)
        elif k == "trsm":
            L = np.tril(A[o["a_i"]:o["a_i"] + o["k"], o["a_j"]:o["a_j"] + o["k"]])
            B = A[o["c_i"]:o["c_i"] + o["m"], o["c_j"]:o["c_j"] + o["k"]]
            A[o["c_i"]:o["c_i"] + o["m"], o["c_j"]:o["c_j"] + o["k"]] = sla.solve_triangular(L, B.T, lower=True).T
        elif k == "gemm":
            Aa = A[o["a_i"]:o["a_i"] + o["m"], o["a_j"]:o["a_j"] + o["k"]]
            Bb = A[o["b_i"]:o["b_i"] + o["n"], o["b_j"]:o["b_j"] + o["k"]]
            A[o["c_i"]:o["c_i"] + o["m"], o["c_j"]:o["c_j"] + o["n"]] -= Aa @ Bb.T
        elif k == "syrk":
            Aa = A[o["a_i"]:o["a_i"] + o["n"], o["a_j"]:o["a_j"] + o["k"]]
            C = A[o["c_i"]:o["c_i"] + o["n"], o["c_j"]:o["c_j"] + o["n"]]
            C -= np.tril(Aa @ Aa.T)


def random_topo(deps, rng):
    n = len(deps)
    succ = [[] for _ in range(n)]
    indeg = [len(d) for d in deps]
    for j, d in enumerate(deps):
        for i in d:
            succ[i].append(j)
    ready = [j for j in range(n) if indeg[j] == 0]
    order = []
    while ready:
        j = ready.pop(rng.randrange(len(ready)))
        order.append(j)
        for s in succ[j]:
            indeg[s] -= 1
            if indeg[s] == 0:
                ready.append(s)
    assert len(order) == n
    return order


@pytest.mark.parametrize("n,c,T,la", [(300, 32, 16, True), (777, 64, 64, True), (1234, 48, 32, True)])
def test_random_topological_orders_factor(n, c, T, la):
    ops, deps = rl.plan_schedule(n, c, T, la)
    A0 = spd(n, seed=11)
    Lref = np.linalg.cholesky(A0)
    rng = random.Random(n)
    for _ in range(3):
        A = np.tril(A0).copy()
        run_order(A, ops, random_topo(deps, rng))
        err = np.abs(np.tril(A) - Lref).max() / np.abs(Lref).max()
        assert err < 1e-12, err
