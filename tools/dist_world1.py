"""The multi-GPU executor on one GPU (world size 1, real NCCL communicator):
relapack_dpotrf_dist (the distributed plan — pack, TRSM on packed rows,
ncclAllGather, unpack, owned-row updates, replicated leaves — captured as one
graph with the NCCL calls as nodes) against the single-GPU relapack_dpotrf on
the same matrix, same box.  CUDA events around each call; A restored between
calls (untimed).

  python tools/dist_world1.py [n] [dist_min] [nb]     (default 16384 8192 512)
"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1602_06763_b200 as rl
from inputs import gen

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
dist_min = int(sys.argv[2]) if len(sys.argv) > 2 else 8192
nb = int(sys.argv[3]) if len(sys.argv) > 3 else 512
uplo = "U"
P = gen.spd_torch(n, 1, dist="normal")
W = torch.empty_like(P.t()).t()
st = torch.cuda.current_stream()
comm = rl.Comm(rl.Comm.unique_id(), 1, 0, torch.cuda.current_device())
d_info = torch.zeros(1, dtype=torch.int32, device="cuda")


def timed(fn, reps=5):
    out = []
    for i in range(reps + 2):
        W.copy_(P)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        info = fn()
        e1.record(st)
        torch.cuda.synchronize()
        assert info == 0, info
        if i >= 2:
            out.append(e0.elapsed_time(e1))
    return out


def single():
    rl.dpotrf_async(W, d_info, uplo, stream=st)
    return 0


def dist():
    return rl.dpotrf_dist(W, comm, uplo, nb=nb, dist_min=dist_min, stream=st)


ts = timed(single)
td = timed(dist)
W.copy_(P)
assert rl.dpotrf_dist(W, comm, uplo, nb=nb, dist_min=dist_min) == 0
R = W.clone()
W.copy_(P)
rl.dpotrf_async(W, d_info, uplo)
torch.cuda.synchronize()
diff = float(torch.max(torch.abs(torch.triu(R) - torch.triu(W))) / torch.max(torch.abs(torch.triu(W))))
comm.close()
ms_s, ms_d = sum(ts) / len(ts), sum(td) / len(td)
fl = n ** 3 / 3.0
print(f"n={n} uplo={uplo} world=1 dist_min={dist_min} nb={nb}")
print(f"single-GPU relapack_dpotrf_async: {ms_s:.3f} ms ({fl / ms_s / 1e9:.1f} GFLOP/s)  {['%.3f' % t for t in ts]}")
print(f"relapack_dpotrf_dist (NCCL, world 1): {ms_d:.3f} ms ({fl / ms_d / 1e9:.1f} GFLOP/s)  {['%.3f' % t for t in td]}")
print(f"ratio dist / single = {ms_d / ms_s:.4f}; max |L_dist - L_single| / max |L| = {diff:.2e}")
