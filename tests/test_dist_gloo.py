"""Multi-GPU schedule exercised on CPU with world_size 2 and 3
`gloo` processes: every rank takes ITS step list from the C library's
schedule builder (relapack_dist_schedule, the same code the NCCL executor
runs), executes the compute steps with the oracle / numpy on its own copy of
the matrix and the collectives with torch.distributed.all_gather.  Ownership
(snake row-block-cyclic, block nb) and the packed-row layout are re-derived
here independently.  Every rank must end with the oracle's factor and the same info.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def owner_of_row(i, nranks, nb):
    """Snake (boustrophedon) block-cyclic owner of L-view row i."""
    b = i // nb
    q, p = divmod(b, nranks)
    return nranks - 1 - p if q % 2 else p


def owned_rows(lo, hi, rank, nranks, nb):
    return [i for i in range(lo, hi) if owner_of_row(i, nranks, nb) == rank]


def simulate(rank, nranks, A, nb, dist_min, c):
    import sys

    sys.path.insert(0, ROOT)
    import oracle
    import paper_1602_06763_b200 as rl

    n = A.shape[0]
    M = np.array(np.tril(A), order="F")  # L-view working copy (lower triangle is all that is read)
    info = 0
    sched = rl.dist_schedule(n, rank, nranks, nb=nb, dist_min=dist_min, c=c)
    send = None
    recv = None
    geom = None  # (lo, hi, c0, ncols, rows_pad)

    def buf(b):
        return M if b == 0 else send

    for op in sched:
        k = op["kind"]
        if info:
            # after a failure every rank skips compute but keeps the collectives in step
            if k not in ("pack", "allgather", "unpack"):
                continue
        if k == "potf2":
            o, nn = op["c_i"], op["n"]
            blk = np.array(M[o:o + nn, o:o + nn], order="F")
            r = oracle.dpotrf(blk, "L")
            M[o:o + nn, o:o + nn] = np.tril(blk) + np.triu(M[o:o + nn, o:o + nn], 1)
            if r and not info:
                info = op["info_base"] + r
        elif k == "trsm":
            lo_, kk, m = op["a_i"], op["k"], op["m"]
            L = np.array(np.tril(M[lo_:lo_ + kk, lo_:lo_ + kk]), order="F")
            X = buf(op["c_buf"])
            B = np.array(X[op["c_i"]:op["c_i"] + m, op["c_j"]:op["c_j"] + kk], order="F")
            oracle.dtrsm_rlt(L, B)
            X[op["c_i"]:op["c_i"] + m, op["c_j"]:op["c_j"] + kk] = B
        elif k == "gemm":
            C = buf(op["c_buf"])
            Aop = buf(op["a_buf"])[op["a_i"]:op["a_i"] + op["m"], op["a_j"]:op["a_j"] + op["k"]]
            Bop = buf(op["b_buf"])[op["b_i"]:op["b_i"] + op["n"], op["b_j"]:op["b_j"] + op["k"]]
            C[op["c_i"]:op["c_i"] + op["m"], op["c_j"]:op["c_j"] + op["n"]] -= Aop @ Bop.T
        elif k == "syrk":
            nn, kk = op["n"], op["k"]
            Aop = buf(op["a_buf"])[op["a_i"]:op["a_i"] + nn, op["a_j"]:op["a_j"] + kk]
            C = buf(op["c_buf"])
            blk = C[op["c_i"]:op["c_i"] + nn, op["c_j"]:op["c_j"] + nn]
            blk -= np.tril(Aop @ Aop.T)
        elif k == "pack":
            lo, hi, c0, ncols = op["c_i"], op["c_i"] + op["m"], op["c_j"], op["k"]
            rows_max = max(len(owned_rows(lo, hi, s, nranks, nb)) for s in range(nranks))
            rows_pad = (rows_max + 7) // 8 * 8
            send = np.zeros((rows_pad, ncols))
            for r, g in enumerate(owned_rows(lo, hi, rank, nranks, nb)):
                send[r] = M[g, c0:c0 + ncols]
            geom = (lo, hi, c0, ncols, rows_pad)
        elif k == "allgather":
            t = torch.from_numpy(np.ascontiguousarray(send))
            parts = [torch.empty_like(t) for _ in range(nranks)]
            dist.all_gather(parts, t)
            recv = [p.numpy() for p in parts]
        elif k == "unpack":
            lo, hi, c0, ncols, rows_pad = geom
            for s in range(nranks):
                for r, g in enumerate(owned_rows(lo, hi, s, nranks, nb)):
                    M[g, c0:c0 + ncols] = recv[s][r]
        else:
            raise AssertionError(k)
    return np.tril(M), info


def _worker(rank, nranks, port, A, nb, dist_min, c, outq):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=nranks)
    try:
        L, info = simulate(rank, nranks, A, nb, dist_min, c)
        outq.put((rank, L, info))
    finally:
        dist.destroy_process_group()


def _run(nranks, A, nb, dist_min, c=32):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, nranks, port, A, nb, dist_min, c, q)) for r in range(nranks)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(nranks):
        r, L, info = q.get(timeout=300)
        res[r] = (L, info)
    for p in procs:
        p.join(timeout=60)
    return res


@pytest.fixture(scope="module", autouse=True)
def built():
    from paper_1602_06763_b200 import build

    build.build()


def _oracle_factor(A):
    import oracle

    R = np.array(A, order="F")
    info = oracle.dpotrf(R, "L")
    return np.tril(R), info


@pytest.mark.parametrize("nranks,n,nb,dist_min", [(2, 520, 64, 128), (3, 700, 64, 200)])
def test_dist_schedule_gloo_matches_oracle(nranks, n, nb, dist_min):
    from inputs import gen
    from tests.metrics import floored_rel_err

    A = gen.spd(n, 21)
    Lo, oinfo = _oracle_factor(A)
    res = _run(nranks, A, nb, dist_min)
    for r in range(nranks):
        L, info = res[r]
        assert info == oinfo == 0
        assert floored_rel_err(L, Lo, A) <= 1e-10, f"rank {r}"
    # every rank holds the same factor
    for r in range(1, nranks):
        assert np.array_equal(res[r][0], res[0][0])


def test_dist_schedule_gloo_indefinite_same_info():
    from inputs import gen

    n, k = 520, 300
    A = gen.indefinite(gen.spd(n, 5), k)
    res = _run(2, A, 64, 128)
    assert res[0][1] == res[1][1] == k + 1


def test_dist_schedule_structure():
    """Host logic: collectives appear in the same order on every rank; every
    owned row block of every distributed node is updated by exactly one rank."""
    import paper_1602_06763_b200 as rl

    n, P, nb, dmin = 4096, 4, 256, 1024
    scheds = [rl.dist_schedule(n, r, P, nb=nb, dist_min=dmin, c=64) for r in range(P)]
    colls = [[(o["kind"], o["m"], o["k"]) for o in s if o["kind"] == "allgather"] for s in scheds]
    assert all(c == colls[0] for c in colls)
    # SYRK row blocks of the top node: union over ranks covers [n1, n) exactly once
    n1 = rl.split_point(n, 64)
    covered = []
    for s in scheds:
        for o in s:
            if o["kind"] == "syrk" and o["level"] == 1:
                covered.extend(range(o["c_i"], o["c_i"] + o["n"]))
    assert sorted(covered) == list(range(n1, n))
    # flops balance of the top-level updates within 2 row blocks
    per = []
    for s in scheds:
        per.append(sum(2.0 * o["m"] * o["n"] * o["k"] if o["kind"] == "gemm" else o["n"] ** 2 * o["k"]
                       for o in s if o["kind"] in ("gemm", "syrk") and o["level"] == 1 and o["c_buf"] == 0))
    assert max(per) / min(per) < 1.35


# ---------------------------------------------------------------- batched split (CFG[4] across GPUs)
def _batch_worker(rank, nranks, port, count, q):
    import sys

    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=nranks)
    import oracle
    import paper_1602_06763_b200 as rl
    from inputs import gen

    b = gen.batched_spd(count, 5)
    bounds = rl.batch_split(b["ns"], nranks)
    lo, hi = bounds[rank], bounds[rank + 1]
    # this rank's range: the oracle stands in for relapack_dpotrf_batched on CPU
    ns = b["ns"][lo:hi]
    offs = b["offsets"][lo:hi] - (b["offsets"][lo] if hi > lo else 0)
    end = int(b["offsets"][hi - 1] + int(b["ns"][hi - 1]) ** 2) if hi > lo else int(b["offsets"][lo]) if lo < count else 0
    sub = b["buf"][int(b["offsets"][lo]) if hi > lo else 0:end].copy() if hi > lo else np.zeros(0)
    info = oracle.dpotrf_batched("L", ns, sub, offs, ns) if hi > lo else np.zeros(0, np.int32)
    # gather every rank's infos (the optional info gather of §8e) and range sizes
    sizes = [None] * nranks
    dist.all_gather_object(sizes, (lo, hi, info.tolist(), float((ns.astype(np.float64) ** 3).sum())))
    if rank == 0:
        q.put(sizes)
    dist.destroy_process_group()


@pytest.mark.parametrize("nranks", [2, 3])
def test_batched_split_gloo(nranks):
    """Each rank takes its contiguous range from the library's split, factors it
    (oracle on CPU), and the gathered per-matrix infos equal the closed form for
    the whole batch; the ranges partition the batch and balance sum n^3."""
    from inputs import gen

    count = 3000
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_batch_worker, args=(r, nranks, port, count, q)) for r in range(nranks)]
    for p in procs:
        p.start()
    sizes = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    b = gen.batched_spd(count, 5)
    los = [s[0] for s in sizes]
    his = [s[1] for s in sizes]
    assert los[0] == 0 and his[-1] == count and all(his[r] == los[r + 1] for r in range(nranks - 1))
    infos = np.concatenate([np.array(s[2], dtype=np.int32) for s in sizes])
    assert np.array_equal(infos, b["expected_info"])
    work = [s[3] for s in sizes]
    assert max(work) / (sum(work) / nranks) < 1.01  # balanced within 1 %
