"""Repeat the bench's n = 16384 U factorization (captured graph, replayed) and
check every result by backward error on the GPU (plain torch matmuls,
test-only): a nondeterministic race shows up as some replays failing.
  python tools/race_check.py [reps] [n] [uplo]
"""
import sys

import torch

sys.path.insert(0, ".")
import paper_1602_06763_b200 as rl
from inputs import gen
from tests.metrics import EPS

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
n = int(sys.argv[2]) if len(sys.argv) > 2 else 16384
uplo = sys.argv[3] if len(sys.argv) > 3 else "U"
P = gen.spd_torch(n, 1, dist="normal" if uplo == "U" else "uniform")
W = torch.empty_like(P.t()).t()
d_info = torch.zeros(1, dtype=torch.int32, device="cuda")
den = float(torch.linalg.norm(P))
bad = 0
ref = None
for r in range(reps):
    W.copy_(P)
    rl.dpotrf_async(W, d_info, uplo)
    torch.cuda.synchronize()
    L = (W if uplo == "L" else W.t()).tril()
    num = 0.0
    for r0 in range(0, n, 4096):
        R = P[r0:r0 + 4096, :] - L[r0:r0 + 4096, :] @ L.t()
        num += float(torch.sum(R * R))
    be = num ** 0.5 / (n * EPS * den)
    same = ref is None or bool(torch.equal(L, ref))
    if ref is None:
        ref = L.clone()
    bad += be > 10
    print(f"rep {r}: info {int(d_info.item())} backward error {be:.3f} bitwise-equal-to-first {same}", flush=True)
print(f"{bad} of {reps} replays failed")
