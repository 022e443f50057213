"""GPU tests of the multi-GPU mode on the one GPU available:

* loopback: P virtual ranks on one GPU run the real kernels, pack/unpack and
  schedule; collectives are device copies between the ranks' buffers and the
  ranks run one after another between collectives (no kernel waits on another
  rank).  Every rank must hold the oracle's factor and the same info.
* NCCL with world size 1: the real communicator path end to end.
"""
import numpy as np
import pytest
import torch

import oracle
import paper_1602_06763_b200 as rl
from inputs import gen
from tests.metrics import floored_rel_err, lower_of

pytestmark = pytest.mark.gpu


def to_dev(A):
    return torch.from_numpy(np.array(A.T, order="C", copy=True)).cuda().t()


def oracle_factor(A, uplo):
    R = np.array(A, order="F", copy=True)
    info = oracle.dpotrf(R, uplo)
    return R, info


@pytest.mark.parametrize("nranks", [2, 3, 4])
@pytest.mark.parametrize("uplo", ["L", "U"])
def test_loopback_matches_oracle(nranks, uplo):
    n = 1100
    A = gen.spd(n, 31)
    R, rinfo = oracle_factor(A, uplo)
    As = [to_dev(A) for _ in range(nranks)]
    infos = rl.dpotrf_dist_loopback(As, uplo, nb=64, dist_min=256)
    torch.cuda.synchronize()
    assert infos == [rinfo] * nranks == [0] * nranks
    G0 = None
    for s in range(nranks):
        G = As[s].cpu().numpy()
        assert floored_rel_err(lower_of(G, uplo), lower_of(R, uplo), A) <= 1e-10, f"rank {s}"
        other = np.triu(np.ones((n, n), bool), 1) if uplo == "L" else np.tril(np.ones((n, n), bool), -1)
        assert np.array_equal(G[other], A[other])
        if G0 is None:
            G0 = G
        else:
            assert np.array_equal(G, G0)  # replicated factor, bitwise identical


def test_loopback_indefinite_info_identical():
    n, k = 900, 700
    A = gen.indefinite(gen.spd(n, 3), k)
    As = [to_dev(A) for _ in range(3)]
    infos = rl.dpotrf_dist_loopback(As, "L", nb=64, dist_min=256)
    assert infos == [k + 1] * 3


def test_nccl_world_size_one():
    n = 800
    A = gen.spd(n, 2)
    R, _ = oracle_factor(A, "L")
    uid = rl.Comm.unique_id()
    comm = rl.Comm(uid, 1, 0, torch.cuda.current_device())
    try:
        dA = to_dev(A)
        info = rl.dpotrf_dist(dA, comm, "L", nb=64, dist_min=256)
        torch.cuda.synchronize()
        assert info == 0
        assert floored_rel_err(np.tril(dA.cpu().numpy()), np.tril(R), A) <= 1e-10
    finally:
        comm.close()
