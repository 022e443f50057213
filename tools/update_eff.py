"""In-graph efficiency of the update launches by CTA tile (RELAPACK_TRACE=1).

For every GEMM/SYRK launch of one captured-graph factorization: algorithmic
flops / (last CTA end - first CTA start), grouped by the tile the size rule
picks (update_tile_for, replicated here for the report), with the time-weighted
mean TFLOP/s per group and the largest launches listed.
  RELAPACK_TRACE=1 python tools/update_eff.py [n] [uplo]
"""
import collections
import os
import sys

import torch

sys.path.insert(0, ".")
import paper_1602_06763_b200 as rl
from inputs import gen

assert os.environ.get("RELAPACK_TRACE") == "1", "run with RELAPACK_TRACE=1"
n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
uplo = sys.argv[2] if len(sys.argv) > 2 else "U"
P = gen.spd_torch(n, 1, dist="normal" if uplo == "U" else "uniform", device="cuda")
W = torch.empty_like(P.t()).t()
d_info = torch.zeros(1, dtype=torch.int32, device="cuda")
for _ in range(3):
    W.copy_(P)
    torch.cuda.synchronize()
    rl.dpotrf_async(W, d_info, uplo)
    torch.cuda.synchronize()
recs = rl.trace_records()
ops, _ = rl.plan_schedule(n, rl.get_crossover(), 64, True)
assert len(ops) == len(recs)


def tile_for(M, N, K, tri):
    def tiles(t):
        tm, tn = (M + t - 1) // t, (N + t - 1) // t
        return tm * (tm + 1) // 2 if tri else tm * tn
    if tiles(128) >= 148:
        return 128
    return 64 if tiles(64) >= 32 else 32


grp = collections.defaultdict(lambda: [0, 0.0, 0.0])
rows = []
for o, r in zip(ops, recs):
    if o["kind"] not in ("gemm", "syrk") or r["t1_us"] < 0:
        continue
    tri = o["kind"] == "syrk"
    M, N, K = o["m"], (o["m"] if tri else o["n"]), o["k"]
    fl = M * M * K if tri else 2.0 * M * N * K
    dt = (r["t1_us"] - r["t0_us"]) * 1e-6
    t = tile_for(M, N, K, tri)
    g = grp[t]
    g[0] += 1
    g[1] += fl
    g[2] += dt
    rows.append((fl / dt / 1e12, dt * 1e3, o["kind"], M, N, K, t, o["deferred"]))
print(f"n={n} uplo={uplo}: update launches by tile (flops / launch span, in the graph)")
for t, (c, fl, dt) in sorted(grp.items()):
    print(f"  tile {t:3d}: {c:4d} launches {fl / 1e12:7.3f} TFLOP in {dt * 1e3:8.2f} ms of spans -> {fl / dt / 1e12:6.2f} TF/s")
rows.sort(key=lambda x: -x[1])
for x in rows[:25]:
    print("  %6.2f TF/s %8.3f ms %s M=%d N=%d K=%d tile=%d deferred=%d" % x)
