"""The paper's central comparison on
B200: the recursive algorithm (no block size to tune; crossover c swept) against
the blocked algorithm with b in {64, 128, 256}, for dpotrf and dtrtri, on the
same kernels and executor.  One GPU; each number = mean of `reps` graph replays
(CUDA events, inputs restored between calls, untimed).

  python tools/sweep_blocked.py [n ...]      (default 4096 16384)
"""
import sys

import torch

sys.path.insert(0, ".")
import paper_1602_06763_b200 as rl
from inputs import gen

PEAK = 37.0
ns = [int(x) for x in sys.argv[1:]] or [4096, 16384]
reps = 5


def timed(fn, P, W):
    st = torch.cuda.current_stream()
    out = []
    for i in range(reps + 2):
        W.copy_(P)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        info = fn(W)
        e1.record(st)
        torch.cuda.synchronize()
        assert info == 0, info
        if i >= 2:
            out.append(e0.elapsed_time(e1))
    return sum(out) / len(out)


print(f"{'op':8s} {'n':>6s} {'variant':24s} {'ms':>9s} {'GFLOP/s':>9s} {'% peak':>7s}")
for n in ns:
    P = gen.spd_torch(n, 1, dist="uniform")
    W = torch.empty_like(P.t()).t()
    fl = n ** 3 / 3.0
    d_info = torch.zeros(1, dtype=torch.int32, device="cuda")

    def rec(W):
        rl.dpotrf_async(W, d_info, "L")
        torch.cuda.synchronize()
        return int(d_info.item())

    rows = []
    for c in (32, 64, 128):
        rl.set_crossover(c)
        rows.append(("potrf", f"recursive c={c}", timed(rec, P, W)))
    rl.set_crossover(128)
    for b in (64, 128, 256):
        rows.append(("potrf", f"blocked b={b}", timed(lambda W, b=b: rl.dpotrf_blocked(W, b, "L"), P, W)))
    # trtri on the Cholesky factor (the blocked plans grow as (n/b)^2 launches:
    # n <= 8192 only)
    T = P.clone()
    assert rl.dpotrf(T, "L") == 0
    rows.append(("trtri", "recursive c=64", timed(lambda W: rl.dtrtri(W, "L"), T, W)))
    for b in ((64, 128, 256) if n <= 8192 else ()):
        rows.append(("trtri", f"blocked b={b}", timed(lambda W, b=b: rl.dtrtri_blocked(W, b, "L"), T, W)))
    for op, var, ms in rows:
        gf = fl / (ms / 1e3) / 1e9
        print(f"{op:8s} {n:6d} {var:24s} {ms:9.3f} {gf:9.1f} {100 * gf / 1e3 / PEAK:7.2f}", flush=True)
    del P, W, T
    torch.cuda.empty_cache()
