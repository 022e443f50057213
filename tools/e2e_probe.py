"""Host-matrix path (relapack_dpotrf on a pinned host matrix) timing, optionally
with the kernel timeline (RELAPACK_TRACE=1): when the compute starts, how much
of it waits for the H2D blocks, and how long the D2H tail is.
  python tools/e2e_probe.py [n] [uplo]"""
import os
import sys

import torch

sys.path.insert(0, ".")
import paper_1602_06763_b200 as rl
from inputs import gen

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
uplo = sys.argv[2] if len(sys.argv) > 2 else "U"
P = gen.spd_torch(n, 1, dist="normal" if uplo == "U" else "uniform", device="cuda")
H0 = P.cpu().pin_memory()
H = torch.empty((n, n), dtype=torch.float64).pin_memory().t()
st = torch.cuda.current_stream()
times = []
for i in range(4):
    H.copy_(H0)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    info = rl.dpotrf(H, uplo)
    e1.record(st)
    torch.cuda.synchronize()
    assert info == 0
    if i > 0:
        times.append(e0.elapsed_time(e1))
tag = " ".join(f"{k}={v}" for k, v in sorted(os.environ.items()) if k.startswith("RELAPACK_"))
print(f"n={n} uplo={uplo} host path {min(times):.3f} ms (mean {sum(times) / len(times):.3f}) [{tag}]")


def curve(recs, label):
    """Fraction of the factorization's flops finished by t = 5, 10, 15 ... ms."""
    recs = [r for r in recs if r["t1_us"] >= 0 and r["kind"] not in ("h2d", "d2h")]
    t0 = min(r["t0_us"] for r in recs)
    tot = sum(r["flops"] for r in recs)
    end = max(r["t1_us"] for r in recs) - t0
    pts = []
    t = 5000.0
    while t < end + 5000:
        pts.append(sum(r["flops"] for r in recs if r["t1_us"] - t0 <= t) / tot)
        t += 5000.0
    print(f"  {label}: kernels span {end / 1e3:.2f} ms; flops done every 5 ms: " + " ".join(f"{100 * x:.0f}" for x in pts))


if os.environ.get("RELAPACK_TRACE") == "1":
    curve(rl.trace_records(), "host path ")
    W = torch.empty_like(P.t()).t()
    d_info = torch.zeros(1, dtype=torch.int32, device="cuda")
    for _ in range(2):
        W.copy_(P)
        torch.cuda.synchronize()
        rl.dpotrf_async(W, d_info, uplo)
        torch.cuda.synchronize()
    curve(rl.trace_records(), "device path")
