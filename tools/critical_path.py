"""Critical path of the captured plan DAG from per-launch serial durations.

Runs the factorization once in profile mode (serial launches, CUDA events
around each), then walks the dependency DAG of the same plan
(relapack_plan_schedule) to report: the serial sum, the DAG critical path
(longest chain of measured durations), and the ops on that path grouped by
kind.  The graph replay time lies between the two.
  python tools/critical_path.py [n] [uplo]
"""
import collections
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
# graph replay time
for _ in range(3):
    W.copy_(P)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    rl.dpotrf_async(W, d_info, uplo)
    e1.record()
    torch.cuda.synchronize()
graph_ms = e0.elapsed_time(e1)
rl.profile_enable(True)
for it in range(2):
    W.copy_(P)
    torch.cuda.synchronize()
    rl.profile_reset()
    rl.dpotrf_async(W, d_info, uplo)
    torch.cuda.synchronize()
recs = rl.profile_records()
rl.profile_enable(False)
ops, deps = rl.plan_schedule(n, rl.get_crossover(), 64, True)
assert len(ops) == len(recs), (len(ops), len(recs))
fin = [0.0] * len(ops)
pred = [-1] * len(ops)
for i, r in enumerate(recs):
    best, bp = 0.0, -1
    for d in deps[i]:
        if fin[d] > best:
            best, bp = fin[d], d
    fin[i] = best + r["ms"]
    pred[i] = bp
end = max(range(len(ops)), key=lambda i: fin[i])
path = []
while end >= 0:
    path.append(end)
    end = pred[end]
path.reverse()
serial = sum(r["ms"] for r in recs)
flops = sum(r["flops"] for r in recs)
print(f"n={n} uplo={uplo} ops={len(ops)} graph={graph_ms:.3f} ms serial_sum={serial:.3f} ms "
      f"critical_path={fin[path[-1]]:.3f} ms ({len(path)} ops)  ideal@37TF={flops/37e9:.3f} ms")
agg = collections.defaultdict(lambda: [0, 0.0])
for i in path:
    r = recs[i]
    key = (r["kind"], r["m"] if r["kind"] != "potf2" else r["n"], r["n"], r["k"])
    agg[key][0] += 1
    agg[key][1] += r["ms"]
print("critical path by (kind, m, n, k):")
for key, (c, ms) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:40]:
    print(f"  {key[0]:6s} m={key[1]:6d} n={key[2]:6d} k={key[3]:6d} x{c:4d} {ms:8.3f} ms  {1000*ms/c:8.2f} us each")
kinds = collections.defaultdict(float)
for i in path:
    kinds[recs[i]["kind"]] += recs[i]["ms"]
print("critical path by kind:", {k: round(v, 3) for k, v in kinds.items()})
