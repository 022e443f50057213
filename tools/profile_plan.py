"""Per-launch breakdown of one factorization (profile mode: events around every kernel)."""
import collections
import json
import sys

import torch

sys.path.insert(0, ".")
import paper_1602_06763_b200 as rl
from inputs import gen

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
uplo = sys.argv[2] if len(sys.argv) > 2 else "U"
P = gen.spd_torch(n, 1, dist="normal", device="cuda")
W = torch.empty_like(P.t()).t()
d_info = torch.zeros(1, dtype=torch.int32, device="cuda")
rl.profile_enable(True)
for it in range(2):
    W.copy_(P)
    torch.cuda.synchronize()
    rl.profile_reset()
    rl.dpotrf_async(W, d_info, uplo)
    torch.cuda.synchronize()
recs = rl.profile_records()
rl.profile_enable(False)
agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
for r in recs:
    if r["kind"] in ("gemm", "syrk"):
        key = (r["kind"], r["m"], r["n"], r["k"])
    else:
        key = (r["kind"], r["m"], r["n"], r["k"])
    a = agg[key]
    a[0] += 1
    a[1] += r["ms"]
    a[2] += r["flops"]
tot = sum(a[1] for a in agg.values())
print(f"n={n} uplo={uplo} total profiled {tot:.3f} ms, {len(recs)} launches")
for key, (c, ms, fl) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:60]:
    print(f"{key[0]:6s} m={key[1]:6d} n={key[2]:6d} k={key[3]:6d} x{c:5d} {ms:9.3f} ms ({100*ms/tot:5.1f}%) "
          f"{fl/ms/1e9 if ms else 0:8.2f} TF/s  {1000*ms/c:8.2f} us/launch")
json.dump(recs, open(f"gpurun_out/profile_plan_{n}_{uplo}.json", "w"))
