"""GPU parity tests: the CUDA path (through the C ABI) against the oracle on the
same seeded inputs.  Tolerances (north_star, readings R8/R9):
floored elementwise relative error <= 1e-10, backward error <= 10, identical
info; bitwise for the exact-integer pins and for the untouched triangle.
"""
import numpy as np
import pytest
import torch

import oracle
import paper_1602_06763_b200 as rl
from inputs import gen
from tests.metrics import backward_error, floored_rel_err, lower_of, sym_from

pytestmark = pytest.mark.gpu

TOL = 1e-10


def to_dev(A: np.ndarray) -> torch.Tensor:
    """Column-major device copy of a Fortran-ordered numpy matrix (same bits, same lda)."""
    lda, n = A.shape
    buf = torch.from_numpy(np.ascontiguousarray(A.T)).cuda()  # (n, lda) row-major == column-major (lda, n)
    return buf.t()[:lda, :n] if lda == n else buf.t()[:n, :]


def dev_full(dA: torch.Tensor, lda: int) -> np.ndarray:
    """The whole lda x n column-major buffer behind a device view, as Fortran numpy."""
    n = dA.shape[1]
    base = torch.as_strided(dA, (lda, n), (1, lda))
    return np.asfortranarray(base.cpu().numpy())


def run_both(A, uplo, n=None):
    """(gpu_result_full, gpu_info, oracle_result_full, oracle_info)."""
    lda = A.shape[0]
    n = A.shape[1] if n is None else n
    dA = to_dev(A)
    info = rl.dpotrf(dA, uplo)
    torch.cuda.synchronize()
    G = dev_full(dA, lda)
    R = np.array(A, order="F", copy=True)
    rinfo = oracle.dpotrf(R, uplo, n=n)
    return G, info, R, rinfo


def check_spd(A, uplo, tol=TOL):
    n = A.shape[1]
    G, info, R, rinfo = run_both(A, uplo)
    assert info == rinfo == 0
    Lg, Lo = lower_of(G[:n], uplo), lower_of(R[:n], uplo)
    err = floored_rel_err(Lg, Lo, A[:n])
    assert err <= tol, f"n={n} uplo={uplo} floored rel err {err:.3e}"
    assert backward_error(sym_from(A[:n], uplo), Lg) <= 10.0
    # the opposite strict triangle and the lda padding are bitwise untouched
    other = np.triu(np.ones((n, n), bool), 1) if uplo == "L" else np.tril(np.ones((n, n), bool), -1)
    assert np.array_equal(G[:n][other].view(np.uint64), A[:n][other].view(np.uint64))
    if A.shape[0] > n:
        assert np.array_equal(G[n:].view(np.uint64), A[n:].view(np.uint64))
    return err


# ---------------------------------------------------------------- base case (n <= c)
@pytest.mark.parametrize("n", [1, 2, 3, 8, 31, 33, 64])
@pytest.mark.parametrize("uplo", ["L", "U"])
def test_base_case_random(n, uplo):
    check_spd(gen.spd(n, n), uplo)


@pytest.mark.parametrize("uplo", ["L", "U"])
def test_P1_integer_n8_bitwise(uplo):
    for seed in range(1, 51):
        A, L = gen.integer_L(8, seed)
        G, info, _, _ = run_both(A, uplo)
        assert info == 0
        assert np.array_equal(lower_of(G, uplo), L)


# ---------------------------------------------------------------- recursion
@pytest.mark.parametrize("n", [65, 100, 127, 128, 129, 200, 256, 300, 513, 1000, 1031])
@pytest.mark.parametrize("uplo", ["L", "U"])
def test_recursive_random(n, uplo):
    check_spd(gen.spd(n, 7 + n), uplo)


@pytest.mark.parametrize("n", [256, 1024])
def test_recursive_normal_dist(n):
    check_spd(gen.spd(n, 3, "normal"), "U")


@pytest.mark.parametrize("n", [256, 1000])
@pytest.mark.parametrize("uplo", ["L", "U"])
def test_P1_integer_recursive_bitwise(n, uplo):
    A, L = gen.integer_L(n, 11)
    G, info, _, _ = run_both(A, uplo)
    assert info == 0
    assert np.array_equal(lower_of(G, uplo), L)


@pytest.mark.parametrize("n", [777, 2048])
def test_P2_min_matrix_exact(n):
    A = gen.min_matrix(n)
    dA = to_dev(A)
    assert rl.dpotrf(dA, "L") == 0
    assert torch.equal(torch.tril(dA), torch.tril(torch.ones(n, n, dtype=torch.float64, device="cuda")))


@pytest.mark.parametrize("n,lda", [(300, 304), (257, 300), (300, 301), (129, 131)])
@pytest.mark.parametrize("uplo", ["L", "U"])
def test_lda_padding_and_odd_lda(n, lda, uplo):
    """Odd lda takes the non-TMA fallback loader; padding rows stay untouched."""
    A = gen.spd(n, 5, lda=lda)
    check_spd(A, uplo)


@pytest.mark.parametrize("uplo", ["L", "U"])
def test_nan_sentinels_other_triangle(uplo):
    n = 333
    A = gen.spd(n, 2)
    other = np.triu(np.ones((n, n), bool), 1) if uplo == "L" else np.tril(np.ones((n, n), bool), -1)
    A = np.array(A, order="F")
    A[other] = np.nan
    G, info, R, rinfo = run_both(A, uplo)
    assert info == rinfo == 0
    assert np.all(np.isnan(G[other]))
    assert not np.any(np.isnan(G[~other]))


# ---------------------------------------------------------------- info
@pytest.mark.parametrize("uplo", ["L", "U"])
@pytest.mark.parametrize("k", [0, 1, 63, 64, 65, 100, 255, 256, 499])
def test_P7_indefinite_info(uplo, k):
    n = 500
    A = gen.indefinite(gen.spd(n, 4), k)
    G, info, R, rinfo = run_both(A, uplo)
    assert rinfo == k + 1
    assert info == rinfo
    # the leading (k x k) block holds the factor of the leading minor of order k
    # (dpotrf2 semantics; the recursion skips the updates after the failure, so
    # rows below the failing diagonal block are left unspecified)
    if k > 0:
        Lg, Lo = lower_of(G, uplo)[:k, :k], lower_of(R, uplo)[:k, :k]
        floor = 1e-4 * np.sqrt(np.abs(np.diag(A)))[:k, None]
        assert np.max(np.abs(Lg - Lo) / np.maximum(np.abs(Lo), floor)) <= TOL


def test_nan_pivot_info():
    n = 200
    A = np.array(gen.spd(n, 1), order="F")
    A[150, 150] = np.nan
    _, info, _, rinfo = run_both(A, "L")
    assert info == rinfo == 151


def test_repeat_calls_use_cached_graph():
    n = 700
    A = gen.spd(n, 9)
    dA = to_dev(A)
    for _ in range(3):
        dA.copy_(to_dev(A))
        assert rl.dpotrf(dA, "L") == 0
    R = np.array(A, order="F")
    oracle.dpotrf(R, "L")
    assert floored_rel_err(np.tril(dA.cpu().numpy()), np.tril(R), A) <= TOL


def test_graphs_off_same_bits():
    n = 600
    A = gen.spd(n, 10)
    d1, d2 = to_dev(A), to_dev(A)
    rl.set_graphs(True)
    assert rl.dpotrf(d1, "L") == 0
    rl.set_graphs(False)
    try:
        assert rl.dpotrf(d2, "L") == 0
    finally:
        rl.set_graphs(True)
    assert torch.equal(d1, d2)  # same kernels, same order: deterministic


@pytest.mark.parametrize("c", [16, 24, 32, 48, 96, 128])
def test_crossover_values(c):
    old = rl.get_crossover()
    rl.set_crossover(c)
    try:
        check_spd(gen.spd(517, c), "L")
    finally:
        rl.set_crossover(old)


# ---------------------------------------------------------------- other entry points
@pytest.mark.parametrize("uplo", ["L", "U"])
@pytest.mark.parametrize("pinned,n", [(False, 450), (True, 450), (True, 2600)])
def test_host_matrix_path(uplo, pinned, n):
    """relapack_dpotrf with a HOST pointer stages the triangle through the GPU;
    a pinned matrix takes the overlapped path (copies are nodes of the DAG)."""
    lda = n + 2
    A = gen.spd(n, 12, lda=lda)
    R = np.array(A, order="F", copy=True)
    rinfo = oracle.dpotrf(R, uplo, n=n)
    H_full = torch.from_numpy(np.array(A.T, order="C", copy=True)).t()  # own CPU buffer (lda x n), column-major
    if pinned:
        H_full = H_full.t().contiguous().pin_memory().t()
        assert H_full.is_pinned()
    H = H_full[:n, :]  # (n, n) view with lda
    for rep in range(2):  # second call replays the cached plan
        if rep:
            H_full.copy_(torch.from_numpy(np.array(A.T, order="C", copy=True)).t())
        info = rl.dpotrf(H, uplo)
        assert info == rinfo == 0
        G = np.asfortranarray(H_full.numpy())
        assert floored_rel_err(lower_of(G[:n], uplo), lower_of(R[:n], uplo), A[:n]) <= TOL
        other = np.triu(np.ones((n, n), bool), 1) if uplo == "L" else np.tril(np.ones((n, n), bool), -1)
        assert np.array_equal(G[:n][other], A[:n][other])
        assert np.all(np.isnan(G[n:]))


def test_async_entry_point():
    n = 640
    A = gen.spd(n, 13)
    dA = to_dev(A)
    d_info = torch.full((1,), -7, dtype=torch.int32, device="cuda")
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        assert rl.dpotrf_async(dA, d_info, "L", stream=s) == 0
    s.synchronize()
    assert int(d_info.item()) == 0
    R = np.array(A, order="F")
    oracle.dpotrf(R, "L")
    assert floored_rel_err(np.tril(dA.cpu().numpy()), np.tril(R), A) <= TOL
    B = gen.indefinite(A, 321)
    dB = to_dev(B)
    assert rl.dpotrf_async(dB, d_info, "L") == 0
    torch.cuda.synchronize()
    assert int(d_info.item()) == 322


def test_argument_errors_on_device():
    d = torch.zeros(16, dtype=torch.float64, device="cuda")
    assert rl.dpotrf_raw("Q", 2, d.data_ptr(), 2) == -1
    assert rl.dpotrf_raw("L", 4, d.data_ptr(), 2) == -4


# ---------------------------------------------------------------- batched (CFG[4] shape)
@pytest.mark.parametrize("uplo", ["L", "U"])
def test_batched_parity(uplo):
    b = gen.batched_spd(3000, 5)
    buf = torch.from_numpy(b["buf"]).cuda()
    ptrs = (buf.data_ptr() + 8 * torch.from_numpy(b["offsets"])).cuda()
    ns = torch.from_numpy(b["ns"]).cuda()
    ldas = torch.from_numpy(b["ldas"]).cuda()
    infos = torch.full((len(b["ns"]),), -99, dtype=torch.int32, device="cuda")
    assert rl.dpotrf_batched(ns, ptrs, ldas, infos, uplo) == 0
    torch.cuda.synchronize()
    ref = b["buf"].copy()
    rinfo = oracle.dpotrf_batched(uplo, b["ns"], ref, b["offsets"], b["ldas"])
    ginfo = infos.cpu().numpy()
    assert np.array_equal(ginfo, rinfo)
    assert np.array_equal(ginfo, b["expected_info"])
    G = buf.cpu().numpy()
    worst = 0.0
    for i in np.nonzero(rinfo == 0)[0]:
        nb, off = int(b["ns"][i]), int(b["offsets"][i])
        A = b["buf"][off: off + nb * nb].reshape(nb, nb).T
        g = G[off: off + nb * nb].reshape(nb, nb).T
        r = ref[off: off + nb * nb].reshape(nb, nb).T
        worst = max(worst, floored_rel_err(lower_of(g, uplo), lower_of(r, uplo), A))
        other = np.triu(np.ones((nb, nb), bool), 1) if uplo == "L" else np.tril(np.ones((nb, nb), bool), -1)
        assert np.array_equal(g[other], A[other])
    assert worst <= TOL


def _batched_case(count, seed):
    b = gen.batched_spd(count, seed)
    buf = torch.from_numpy(b["buf"]).cuda()
    ptrs = (buf.data_ptr() + 8 * torch.from_numpy(b["offsets"])).cuda()
    ns = torch.from_numpy(b["ns"]).cuda()
    ldas = torch.from_numpy(b["ldas"]).cuda()
    infos = torch.full((len(b["ns"]),), -99, dtype=torch.int32, device="cuda")
    return b, buf, ptrs, ns, ldas, infos


def _batched_check(b, buf, infos):
    ref = b["buf"].copy()
    rinfo = oracle.dpotrf_batched("L", b["ns"], ref, b["offsets"], b["ldas"])
    assert np.array_equal(infos.cpu().numpy(), rinfo)
    G = buf.cpu().numpy()
    for i in np.nonzero(rinfo == 0)[0]:
        nb, off = int(b["ns"][i]), int(b["offsets"][i])
        A = b["buf"][off: off + nb * nb].reshape(nb, nb).T
        g = G[off: off + nb * nb].reshape(nb, nb).T
        r = ref[off: off + nb * nb].reshape(nb, nb).T
        assert floored_rel_err(lower_of(g, "L"), lower_of(r, "L"), A) <= TOL


def test_batched_two_streams():
    """Back-to-back batched calls on two streams share the library's bucketing
    workspace: the second must not overwrite it while the first still runs."""
    cases = [_batched_case(4000, 21), _batched_case(3000, 22)]
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    for (b, buf, ptrs, ns, ldas, infos), s in zip(cases, (s1, s2)):
        with torch.cuda.stream(s):
            assert rl.dpotrf_batched(ns, ptrs, ldas, infos, "L") == 0
    torch.cuda.synchronize()
    for b, buf, ptrs, ns, ldas, infos in cases:
        _batched_check(b, buf, infos)


def test_batched_graph_capture():
    """The batched call (bucketing + size classes on forked streams) captured
    into a CUDA graph and replayed gives the same factors."""
    b, buf, ptrs, ns, ldas, infos = _batched_case(2000, 23)
    pristine = buf.clone()
    assert rl.dpotrf_batched(ns, ptrs, ldas, infos, "L") == 0  # sizes the workspace outside capture
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        rl.dpotrf_batched(ns, ptrs, ldas, infos, "L", stream=s)
    for _ in range(2):
        buf.copy_(pristine)
        infos.fill_(-99)
        g.replay()
        torch.cuda.synchronize()
        _batched_check(b, buf, infos)


def test_batched_graph_replay_after_regrow():
    """a graph captured with no library workspace in place, an eager
    call that (re)grows the library workspace, then replays of the graph
    concurrent with eager calls on another stream — the replay owns its own
    (graph-allocated) workspace, so all results stay right."""
    rl.finalize()  # no library workspace exists: the capture must not allocate one
    b, buf, ptrs, ns, ldas, infos = _batched_case(1500, 31)
    pristine = buf.clone()
    s = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        rl.dpotrf_batched(ns, ptrs, ldas, infos, "L", stream=s)
    big = _batched_case(6000, 32)  # eager: grows the library workspace
    assert rl.dpotrf_batched(big[3], big[2], big[4], big[5], "L") == 0
    torch.cuda.synchronize()
    _batched_check(big[0], big[1], big[5])
    other = _batched_case(5000, 33)
    other_pristine = other[1].clone()
    s2 = torch.cuda.Stream()
    for _ in range(3):
        buf.copy_(pristine)
        infos.fill_(-99)
        other[1].copy_(other_pristine)
        other[5].fill_(-99)
        torch.cuda.synchronize()
        g.replay()
        with torch.cuda.stream(s2):
            assert rl.dpotrf_batched(other[3], other[2], other[4], other[5], "L", stream=s2) == 0
        torch.cuda.synchronize()
        _batched_check(b, buf, infos)
    _batched_check(other[0], other[1], other[5])


def test_set_stream_is_per_thread():
    """relapack_set_stream is a per-thread setting — two threads each
    factor on their own stream, interleaving set_stream and the call."""
    import threading

    n = 700
    errs = []

    def work(seed):
        try:
            s = torch.cuda.Stream()
            for it in range(5):
                A = np.asfortranarray(gen.spd(n, seed + it))
                with torch.cuda.stream(s):
                    dA = to_dev(A)
                    info = rl.dpotrf(dA, "L", stream=s)
                s.synchronize()
                R = np.array(A, order="F")
                assert info == oracle.dpotrf(R, "L") == 0
                G = dA.cpu().numpy()
                assert floored_rel_err(np.tril(G), np.tril(R), A) <= TOL
        except Exception as e:  # pragma: no cover - reported below
            errs.append(e)

    ts = [threading.Thread(target=work, args=(100 * k,)) for k in range(3)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errs, errs


def test_batched_bad_sizes():
    n_ok = 16
    buf = torch.from_numpy(np.asfortranarray(gen.spd(n_ok, 1)).T.copy().reshape(-1)).cuda()
    ns = torch.tensor([n_ok, 65, -1, 16, 0], dtype=torch.int32, device="cuda")
    ldas = torch.tensor([16, 65, 1, 8, 1], dtype=torch.int32, device="cuda")
    ptrs = torch.tensor([buf.data_ptr()] * 5, dtype=torch.int64, device="cuda")
    infos = torch.zeros(5, dtype=torch.int32, device="cuda")
    assert rl.dpotrf_batched(ns, ptrs, ldas, infos, "L") == 0
    torch.cuda.synchronize()
    assert infos.cpu().tolist() == [0, -2, -2, -4, 0]


@pytest.mark.parametrize("uplo", ["L", "U"])
def test_batched_ragged_layouts(uplo):
    """Every n in 1..64 (odd n take the plain-load path), lda > n for some,
    bases that are only 8-byte aligned for some; NaN sentinels in the other
    triangle and the lda padding must stay bitwise untouched."""
    rng = np.random.default_rng(123)
    ns, ldas, offs, mats = [], [], [], []
    off = 1  # first matrix starts at an odd double: not 16-byte aligned
    for k in range(400):
        n = int(k % 64) + 1
        lda = n + (3 if k % 5 == 0 else (1 if k % 7 == 0 else 0))
        A = np.full((lda, n), np.nan)
        A[:n, :n] = gen.spd(n, 100 + k)
        if k % 3 == 0:
            kk = int(rng.integers(0, n))
            A[kk, kk] = -A[kk, kk]
        ns.append(n)
        ldas.append(lda)
        offs.append(off)
        mats.append(A)
        off += lda * n + (1 if k % 4 == 0 else 0)
    buf = np.full(off, np.nan)
    for A, o in zip(mats, offs):
        lda, n = A.shape
        buf[o:o + lda * n] = A.T.reshape(-1)
    ns, ldas, offs = np.array(ns, np.int32), np.array(ldas, np.int32), np.array(offs, np.int64)
    dbuf = torch.from_numpy(buf).cuda()
    ptrs = (dbuf.data_ptr() + 8 * torch.from_numpy(offs)).cuda()
    infos = torch.full((len(ns),), -99, dtype=torch.int32, device="cuda")
    assert rl.dpotrf_batched(torch.from_numpy(ns).cuda(), ptrs, torch.from_numpy(ldas).cuda(), infos, uplo) == 0
    torch.cuda.synchronize()
    ref = buf.copy()
    rinfo = oracle.dpotrf_batched(uplo, ns, ref, offs, ldas)
    ginfo = infos.cpu().numpy()
    assert np.array_equal(ginfo, rinfo)
    G = dbuf.cpu().numpy()
    outside = np.ones(off, bool)
    for i in range(len(ns)):
        n, lda, o = int(ns[i]), int(ldas[i]), int(offs[i])
        g = G[o:o + lda * n].reshape(n, lda).T
        r = ref[o:o + lda * n].reshape(n, lda).T
        A0 = mats[i]
        tri = np.tril(np.ones((n, n), bool)) if uplo == "L" else np.triu(np.ones((n, n), bool))
        untouched = np.ones((lda, n), bool)
        untouched[:n, :n] = ~tri
        assert np.array_equal(g[untouched], A0[untouched], equal_nan=True), i
        if rinfo[i] == 0:
            assert floored_rel_err(lower_of(g[:n, :n], uplo), lower_of(r[:n, :n], uplo), A0[:n, :n]) <= TOL, i
        outside[o:o + lda * n] = False
    assert np.all(np.isnan(G[outside]))


def test_batched_integer_exact():
    """P1 through the batched kernel: integer L (diag 1..4, off-diagonal -2..2),
    A = L L^T, every size class; the factor comes back bitwise."""
    ns, offs, mats, Ls = [], [], [], []
    off = 0
    for k, n in enumerate([8, 13, 16, 24, 32, 40, 48, 56, 64] * 3):
        A, L = gen.integer_L(n, 200 + k)
        ns.append(n)
        offs.append(off)
        mats.append(A)
        Ls.append(L)
        off += n * n
    buf = np.zeros(off)
    for A, o in zip(mats, offs):
        n = A.shape[0]
        buf[o:o + n * n] = np.asfortranarray(A).T.reshape(-1)
    ns, offs = np.array(ns, np.int32), np.array(offs, np.int64)
    dbuf = torch.from_numpy(buf).cuda()
    ptrs = (dbuf.data_ptr() + 8 * torch.from_numpy(offs)).cuda()
    infos = torch.full((len(ns),), -99, dtype=torch.int32, device="cuda")
    dn = torch.from_numpy(ns).cuda()
    assert rl.dpotrf_batched(dn, ptrs, dn, infos, "L") == 0
    torch.cuda.synchronize()
    G = dbuf.cpu().numpy()
    assert infos.cpu().numpy().tolist() == [0] * len(ns)
    for i in range(len(ns)):
        n, o = int(ns[i]), int(offs[i])
        g = G[o:o + n * n].reshape(n, n).T
        assert np.array_equal(np.tril(g), Ls[i]), (i, n)


# ---------------------------------------------------------------- 64 < n <= 128 base case (in-CTA node)
@pytest.mark.parametrize("n", [65, 72, 100, 127, 128])
@pytest.mark.parametrize("uplo", ["L", "U"])
def test_node128_base_case(n, uplo):
    old = rl.get_crossover()
    rl.set_crossover(128)
    try:
        check_spd(gen.spd(n, 40 + n), uplo)
        A, L = gen.integer_L(n, 3 + n)
        G, info, _, _ = run_both(A, uplo)
        assert info == 0
        assert np.array_equal(lower_of(G, uplo), L)  # exact: integer factor, perfect-square pivots
    finally:
        rl.set_crossover(old)


@pytest.mark.parametrize("k", [5, 63, 64, 90, 127])
def test_node128_info(k):
    """A negated diagonal at k makes pivot k the first failure (closed form R11)."""
    n = 128
    A = np.array(gen.spd(n, 9), order="F")
    A[k, k] = -A[k, k]
    old = rl.get_crossover()
    rl.set_crossover(128)
    try:
        _, info, _, rinfo = run_both(A, "L")
    finally:
        rl.set_crossover(old)
    assert info == rinfo == k + 1


# ---------------------------------------------------------------- 128 < n <= 256 base case (in-CTA 256-node)
@pytest.mark.parametrize("n", [129, 136, 160, 191, 192, 200, 255, 256])
@pytest.mark.parametrize("uplo", ["L", "U"])
def test_node256_base_case(n, uplo):
    """The 256-node kernel (A11 node, register TRSM, K-halved SYRK, A22 node in one CTA)."""
    old = rl.get_crossover()
    rl.set_crossover(256)
    try:
        check_spd(gen.spd(n, 70 + n), uplo)
        A, L = gen.integer_L(n, 5 + n)
        G, info, _, _ = run_both(A, uplo)
        assert info == 0
        assert np.array_equal(lower_of(G, uplo), L)  # exact: integer factor, perfect-square pivots
    finally:
        rl.set_crossover(old)


@pytest.mark.parametrize("n,lda", [(256, 259), (200, 203), (250, 256), (129, 130)])
@pytest.mark.parametrize("uplo", ["L", "U"])
def test_node256_lda(n, lda, uplo):
    """Odd / padded lda (element copies instead of 16-byte pairs); padding untouched."""
    old = rl.get_crossover()
    rl.set_crossover(256)
    try:
        check_spd(gen.spd(n, 17, lda=lda), uplo)
    finally:
        rl.set_crossover(old)


@pytest.mark.parametrize("k", [0, 5, 64, 127, 128, 129, 191, 200, 255])
@pytest.mark.parametrize("uplo", ["L", "U"])
def test_node256_info(k, uplo):
    """A negated diagonal at k is the first failed pivot (closed form R11), in A11's
    or in A22's half of the node."""
    n = 256
    A = np.array(gen.spd(n, 9), order="F")
    A[k, k] = -A[k, k]
    old = rl.get_crossover()
    rl.set_crossover(256)
    try:
        _, info, _, rinfo = run_both(A, uplo)
    finally:
        rl.set_crossover(old)
    assert info == rinfo == k + 1


@pytest.mark.parametrize("n", [256, 1000, 2048])
def test_node256_vs_node128_plans(n):
    """Crossover 256 (one launch per 256-node) and 128 (node-128, TRSM, SYRK,
    node-128) factor the same matrix to within the parity tolerance of each other."""
    A = gen.spd(n, 77)
    old = rl.get_crossover()
    try:
        out = []
        for c in (128, 256):
            rl.set_crossover(c)
            dA = to_dev(A)
            assert rl.dpotrf(dA, "L") == 0
            out.append(np.tril(dA.cpu().numpy()))
    finally:
        rl.set_crossover(old)
    assert floored_rel_err(out[1], out[0], A) <= TOL


# ---------------------------------------------------------------- extreme exponents
@pytest.mark.parametrize("uplo", ["L", "U"])
@pytest.mark.parametrize("n", [100, 300, 1031])
@pytest.mark.parametrize("e2", [1000, -1000])
def test_scaled_inputs(n, uplo, e2):
    """A * 2^e2 (exact scaling): entries near 2^1010 / 2^-990, pivots and factors
    far from 1.  Compared after scaling back by 2^(-e2/2) (exact), so the norms
    of the metric stay finite."""
    A0 = gen.spd(n, 11)
    A = np.asfortranarray(A0 * 2.0 ** e2)
    G, info, R, rinfo = run_both(A, uplo)
    assert info == rinfo == 0
    s = 2.0 ** (-e2 // 2)
    Lg, Lo = lower_of(G[:n], uplo) * s, lower_of(R[:n], uplo) * s
    assert np.isfinite(Lg).all()
    err = floored_rel_err(Lg, Lo, A0)
    assert err <= TOL, f"scaled 2^{e2} n={n} {uplo}: {err:.3e}"


@pytest.mark.parametrize("uplo", ["L", "U"])
@pytest.mark.parametrize("n,k", [(1, 0), (2, 1), (64, 40), (128, 127), (300, 200), (1031, 700)])
def test_subnormal_pivot(n, k, uplo):
    """A positive subnormal pivot (d = 2^-1060): DESIGN.md reading R15 — the GPU
    path follows the flush-to-zero semantics of its FP64 rsqrt and reports the
    pivot through info (= k + 1, as for d <= 0) instead of returning inf / NaN
    factors with info = 0; the leading k x k factor is final and matches the
    oracle (which keeps IEEE gradual underflow and continues: a documented
    deviation outside every BASELINE config, whose pivots are >= n)."""
    A = np.asfortranarray(gen.spd(n, 5))
    A[k, :] = 0.0
    A[:, k] = 0.0
    A[k, k] = 2.0 ** -1060
    G, info, R, rinfo = run_both(A, uplo)
    assert rinfo == 0
    assert info == k + 1
    if k > 0:
        Lg, Lo = lower_of(G[:n], uplo)[:k, :k], lower_of(R[:n], uplo)[:k, :k]
        assert np.isfinite(Lg).all()
        assert floored_rel_err(Lg, Lo, A[:k, :k]) <= TOL
    # the smallest normal pivot is accepted (2^-1022 -> l_kk = 2^-511 exactly)
    A[k, k] = 2.0 ** -1022
    G, info, R, rinfo = run_both(A, uplo)
    assert info == rinfo == 0
    assert lower_of(G[:n], uplo)[k, k] == 2.0 ** -511


@pytest.mark.parametrize("uplo", ["L", "U"])
def test_graph_reuse_across_matrices(uplo):
    """One captured graph per (n, lda, uplo) serves every matrix and info
    pointer (pointer-independent plan: offsets + a per-run base, TMA descriptors
    rebased by the graph's first node): three matrices of the same shape and two
    info words, interleaved, each result against the oracle; then a matrix
    whose base is only 8-byte aligned (its own plan, no TMA)."""
    n = 1500
    As = [np.asfortranarray(gen.spd(n, 40 + k)) for k in range(3)]
    infos = [torch.full((1,), -7, dtype=torch.int32, device="cuda") for _ in range(2)]
    for it in range(6):
        k = it % 3
        dA = to_dev(As[k])
        d_info = infos[it % 2]
        assert rl.dpotrf_async(dA, d_info, uplo) == 0
        torch.cuda.synchronize()
        assert int(d_info.item()) == 0
        R = np.array(As[k], order="F")
        assert oracle.dpotrf(R, uplo) == 0
        G = dA.cpu().numpy()
        assert floored_rel_err(lower_of(G, uplo), lower_of(R, uplo), As[k]) <= TOL
    # 8-byte aligned base
    buf = torch.empty(n * n + 1, dtype=torch.float64, device="cuda")
    dA = buf[1:].view(n, n).t()
    dA.copy_(torch.from_numpy(np.ascontiguousarray(As[0].T)).cuda().t())
    assert rl.dpotrf(dA, uplo) == 0
    R = np.array(As[0], order="F")
    oracle.dpotrf(R, uplo)
    assert floored_rel_err(lower_of(dA.cpu().numpy(), uplo), lower_of(R, uplo), As[0]) <= TOL
    # a failing matrix through the same graph: info identical to the oracle's
    Bad = gen.indefinite(As[1], 900)
    dB = to_dev(np.asfortranarray(Bad))
    assert rl.dpotrf(dB, uplo) == 901
