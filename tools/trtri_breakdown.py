"""B200 analogue of the paper's Fig. recursive_breakdown: the
recursive dtrtri's flops and efficiency per recursion level.  The paper: the
two BLAS-3 calls (trmm + trsm) of level 1 cover 3/4 of the n^3/3 flops at
~86 % efficiency, level 2 18.8 % at 79 %, level 3 4.69 % at 68 %, level 4
1.17 % at 57 % (one Ivy Bridge core, OpenBLAS).  Here every launch of the
plan is timed on its own (serial replay with CUDA events, the xprofile hook),
its leading-term flops attributed to the recursion level that issued it.

  python tools/trtri_breakdown.py [n]      (default 16384)
"""
import collections
import sys

import torch

sys.path.insert(0, ".")
import paper_1602_06763_b200 as rl
from inputs import gen

PEAK = 37.0
n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
P = gen.spd_torch(n, 1, dist="uniform")
assert rl.dpotrf(P, "L") == 0
W = torch.empty_like(P.t()).t()
W.copy_(P)
torch.cuda.synchronize()
recs = rl.xprofile_records(lambda: rl.dtrtri(W, "L"))
total = n ** 3 / 3.0
by = collections.defaultdict(lambda: [0.0, 0.0, 0])
for r in recs:
    key = ("base (trti2)" if r["kind"] == "trti2" else f"level {r['level']}")
    by[key][0] += r["flops"]
    by[key][1] += r["ms"]
    by[key][2] += 1
print(f"dtrtri n={n}: {len(recs)} launches, serial sum {sum(r['ms'] for r in recs):.2f} ms "
      f"(leading-term flops {sum(r['flops'] for r in recs):.4e} vs n^3/3 {total:.4e})")
print(f"{'level':14s} {'flop share':>10s} {'launches':>9s} {'ms':>9s} {'TFLOP/s':>8s} {'% of 37 TF':>10s}")
for key in sorted(by, key=lambda k: (k.startswith('base'), int(k.split()[1]) if k.startswith('level') else 0)):
    fl, ms, cnt = by[key]
    tf = fl / (ms / 1e3) / 1e12 if ms > 0 else 0.0
    print(f"{key:14s} {100 * fl / total:9.2f}% {cnt:9d} {ms:9.3f} {tf:8.2f} {100 * tf / PEAK:9.1f}%")
