"""Two factorizations of one config (the first captures the graph): a short
command for ncu launch lists / captures.  python tools/ncu_step.py n uplo"""
import sys

import torch

sys.path.insert(0, ".")
import paper_1602_06763_b200 as rl
from inputs import gen

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
uplo = sys.argv[2] if len(sys.argv) > 2 else "U"
P = gen.spd_torch(n, 1, dist="normal" if uplo == "U" else "uniform", device="cuda")
W = torch.empty_like(P.t()).t()
d_info = torch.zeros(1, dtype=torch.int32, device="cuda")
for _ in range(2):
    W.copy_(P)
    torch.cuda.synchronize()
    rl.dpotrf_async(W, d_info, uplo)
    torch.cuda.synchronize()
assert int(d_info.item()) == 0
print("ok", n, uplo)
