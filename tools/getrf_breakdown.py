"""Serial per-launch breakdown of the getrf plan at n (default 16384): time per
op kind and per recursion level of the panels (xprofile_records: the plan
replayed one launch at a time with CUDA events on the launch stream).  Knobs
(RELAPACK_GETRF_LA, _WINDOW, RELAPACK_GETF2_CLUSTER) from the environment."""
import sys
from collections import defaultdict

import torch

import paper_1602_06763_b200 as rl

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
g = torch.Generator(device="cuda").manual_seed(1)
A = (torch.rand(n, n, device="cuda", dtype=torch.float64, generator=g) * 2 - 1).t()  # column-major view
P = A.clone()
ipiv = torch.zeros(n, dtype=torch.int32, device="cuda")
rl.dgetrf(A, ipiv)  # plan + warm-up
A.copy_(P)
torch.cuda.synchronize()
recs = rl.xprofile_records(lambda: rl.dgetrf(A, ipiv))
by = defaultdict(lambda: [0.0, 0.0, 0])
lv = defaultdict(lambda: [0.0, 0])
for r in recs:
    b = by[r["kind"]]
    b[0] += r["ms"]; b[1] += r["flops"]; b[2] += 1
    if r["kind"] == "getf2":
        lv[r["level"]][0] += r["ms"]; lv[r["level"]][1] += 1
tot = sum(v[0] for v in by.values())
print(f"n={n} launches={len(recs)} serial total {tot:.1f} ms")
for k, (ms, fl, c) in sorted(by.items(), key=lambda x: -x[1][0]):
    print(f"  {k:6s} {ms:9.2f} ms  {c:6d} launches  {fl / max(ms, 1e-9) / 1e9:8.2f} TF" if fl else f"  {k:6s} {ms:9.2f} ms  {c:6d} launches")
print("  getf2 by level:", {k: (round(v[0], 2), v[1]) for k, v in sorted(lv.items())})
