"""Kernel timeline of one captured-graph factorization (RELAPACK_TRACE=1).

Reports the real span, per-kind busy time and kernel-level concurrency, the
critical path through the plan DAG using the traced start/end times (the chain
of ops where each waits for its latest-finishing predecessor), and the gaps on
that path (time between a predecessor's end and the op's start: launch/
scheduling latency or SM contention).
  RELAPACK_TRACE=1 python tools/trace_timeline.py [n] [uplo] [out.json]
"""
import collections
import json
import os
import sys

import torch

sys.path.insert(0, ".")
import paper_1602_06763_b200 as rl
from inputs import gen

assert os.environ.get("RELAPACK_TRACE") == "1", "run with RELAPACK_TRACE=1"
n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
uplo = sys.argv[2] if len(sys.argv) > 2 else "L"
P = gen.spd_torch(n, 1, dist="normal" if uplo == "U" else "uniform", device="cuda")
W = torch.empty_like(P.t()).t()
d_info = torch.zeros(1, dtype=torch.int32, device="cuda")
for _ in range(3):
    W.copy_(P)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    rl.dpotrf_async(W, d_info, uplo)
    e1.record()
    torch.cuda.synchronize()
graph_ms = e0.elapsed_time(e1)
recs = rl.trace_records()
ops, deps = rl.plan_schedule(n, rl.get_crossover(), 64, True)
assert len(ops) == len(recs)
span = max(r["t1_us"] for r in recs)
busy = collections.defaultdict(float)
for r in recs:
    if r["t1_us"] >= 0:
        busy[r["kind"]] += r["t1_us"] - r["t0_us"]
# concurrency histogram (kernels in flight over time)
ev = sorted([(r["t0_us"], 1) for r in recs if r["t1_us"] >= 0] + [(r["t1_us"], -1) for r in recs if r["t1_us"] >= 0])
conc, last, acc = 0, 0.0, collections.defaultdict(float)
for t, d in ev:
    acc[conc] += t - last
    conc += d
    last = t
# critical path: from the last-finishing op back through the latest-finishing predecessor
end = max(range(len(recs)), key=lambda i: recs[i]["t1_us"])
path = []
i = end
while i >= 0:
    path.append(i)
    ps = [d for d in deps[i] if recs[d]["t1_us"] >= 0]
    i = max(ps, key=lambda d: recs[d]["t1_us"]) if ps else -1
path.reverse()
on_path = collections.defaultdict(lambda: [0, 0.0, 0.0])  # kind: count, run us, wait us
prev_end = 0.0
for i in path:
    r = recs[i]
    a = on_path[r["kind"]]
    a[0] += 1
    a[1] += r["t1_us"] - r["t0_us"]
    a[2] += max(0.0, r["t0_us"] - prev_end)
    prev_end = r["t1_us"]
print(f"n={n} uplo={uplo} graph={graph_ms:.3f} ms traced span={span / 1e3:.3f} ms ops={len(recs)}")
print("kernel busy time by kind (us, summed over launches):", {k: round(v, 1) for k, v in busy.items()})
print("time by #kernels in flight (us):", {k: round(v, 1) for k, v in sorted(acc.items())})
tot_run = sum(a[1] for a in on_path.values())
tot_wait = sum(a[2] for a in on_path.values())
print(f"critical path: {len(path)} ops, running {tot_run / 1e3:.3f} ms + waiting {tot_wait / 1e3:.3f} ms")
for k, (c, run, wait) in sorted(on_path.items(), key=lambda kv: -kv[1][1]):
    print(f"  {k:6s} x{c:4d} running {run / 1e3:8.3f} ms  waiting before start {wait / 1e3:8.3f} ms")
if os.environ.get("CP_DETAIL") == "1":
    prev_end = 0.0
    for i in path:
        r, o = recs[i], ops[i]
        print(f"    {r['kind']:5s} m={o['m']:5d} n={o['n']:5d} k={o['k']:5d} lvl={o['level']} defer={o['deferred']} "
              f"wait {max(0.0, r['t0_us'] - prev_end):7.1f} run {r['t1_us'] - r['t0_us']:7.1f} us")
        prev_end = r["t1_us"]
if len(sys.argv) > 3:
    json.dump({"recs": recs, "path": path}, open(sys.argv[3], "w"))
