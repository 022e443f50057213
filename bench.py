#!/usr/bin/env python
"""bench.py — recursive FP64 Cholesky (xpotrf, arXiv:1602.06763) on B200.

Metric (BASELINE.json): dpotrf FP64 GFLOP/s (n^3/3 flops) and % of FP64 peak.
Default workload (N=1): CFG[2] of BASELINE.json — single dpotrf, uplo=U,
n=16384, A = B B^T + n I with B i.i.d. N(0,1) (seeded Philox, synthetic),
the largest single-matrix config that fits one GPU and the one the >=70 %
update-kernel target is stated on.  Other configs: --config n256|n4096|n16384|n65536|batch.

One "step" = one full factorization (every row of SURVEY §8a) of a fresh copy
of A (restored from a pristine device copy between steps, untimed; A is 2 GiB
> the 126 MB L2, so every step starts cold).  Timing: W untimed warm-up steps,
then K steps, each bracketed by barrier + synchronize and CUDA events on the
launching stream; value = flops / summed device time (max over ranks).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl reference]
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

# NCCL writes its version banner (NCCL_DEBUG=VERSION and above) to stdout, which
# would put a non-JSON line before the one JSON line rank 0 prints: route NCCL's
# debug output to a file unless the caller chose one
os.environ.setdefault("NCCL_DEBUG_FILE", "/tmp/relapack_nccl_debug.%h.%p.log")
# ... and, because a library may still write to file descriptor 1 (NCCL does when
# it cannot open that file), keep the real stdout for the JSON line alone: fd 1
# points at stderr for the rest of the process, emit() writes the line to the
# saved descriptor.
sys.stdout.flush()
_JSON_OUT = os.fdopen(os.dup(1), "w")
os.dup2(2, 1)


def emit(obj):
    _JSON_OUT.write(json.dumps(obj) + "\n")
    _JSON_OUT.flush()


ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: (n, uplo, dist, BASELINE.json config index)
    "n256": (256, "L", "uniform", 0),
    "n4096": (4096, "L", "uniform", 1),
    "n16384": (16384, "U", "normal", 2),
    "n65536": (65536, "L", "uniform", 3),
    "batch": (None, "L", "uniform", 4),
}
# §8(f) rows: the paper's other recursive operations, measured with the
# same harness (GFLOP/s of the leading-term flop count, % of FP64 peak).
# name: (flops(n, nrhs), description)
NEXT = {
    "trtri": (lambda n, r: n ** 3 / 3.0, "recursive dtrtri (N1), uplo L, the Cholesky factor of the CFG recipe"),
    "trtri_blocked": (lambda n, r: n ** 3 / 3.0, "blocked dtrtri (N1/N2 comparison), block --block"),
    "potrf_blocked": (lambda n, r: n ** 3 / 3.0, "blocked right-looking dpotrf (N2), block --block, CFG recipe"),
    "lauum": (lambda n, r: n ** 3 / 3.0, "recursive dlauum (N3), L^T L of the Cholesky factor"),
    "potri": (lambda n, r: 2.0 * n ** 3 / 3.0, "dpotri (N3): dtrtri + dlauum of the Cholesky factor"),
    "potrs": (lambda n, r: 2.0 * n * n * r, "dpotrs (N3): two recursive triangular solves, --nrhs right-hand sides"),
    "getrf": (lambda n, r: 2.0 * n ** 3 / 3.0, "recursive dgetrf with partial pivoting (N4), A ~ U(-1,1)"),
}
FP64_PEAK_TFLOPS_DATASHEET = 37.0  # HGX B200 FP64 / FP64 tensor core datasheet figure


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except Exception:
        return {}


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    def __init__(self, device_index: int):
        self.dev = device_index
        self.samples = []
        self.proc = None
        self.thread = None

    def __enter__(self):
        cmd = ["nvidia-smi", "-i", str(self.dev),
               "--query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
               "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
               "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
               "--format=csv,noheader,nounits", "-lms", "100"]
        try:
            self.proc = subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return self

        def reader():
            for line in self.proc.stdout:
                parts = [p.strip() for p in line.split(",")]
                if len(parts) >= 8:
                    self.samples.append(parts)

        self.thread = threading.Thread(target=reader, daemon=True)
        self.thread.start()
        time.sleep(0.3)
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            time.sleep(0.2)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            if self.thread:
                self.thread.join(timeout=2)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for p in self.samples:
            try:
                sm.append(float(p[0]))
                mx = float(p[1])
            except ValueError:
                continue
            for nm, v in zip(names, p[4:8]):
                if v.lower() == "active":
                    reasons.add(nm)
        sm.sort()
        med = sm[len(sm) // 2] if sm else None
        return {"sm_mhz": med, "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


def gen_matrix(n, uplo, dist, seed, device):
    from inputs import gen

    return gen.spd_torch(n, seed, dist=dist, device=device)  # (n, n) column-major, exactly symmetric


def _cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def cpu_oracle_sample(A_host, n, uplo, full_max=16384):
    """The oracle as it stands on the host cores.  Up to n = full_max the WHOLE
    factorization of the same matrix (~100 s at n = 16384 on 16 cores: the
    representative rate, every column's k-loop at its real length); beyond,
    the first J columns of the left-looking loop (a bounded sample)."""
    import numpy as np

    import oracle

    if n <= full_max:
        X = np.array(A_host, order="F", copy=True)
        t0 = time.perf_counter()
        info = oracle.dpotrf(X, uplo)
        dt = time.perf_counter() - t0
        assert info == 0
        fl = n ** 3 / 3.0
        return {"value": round(fl / dt / 1e9, 3), "unit": "GFLOP/s", "cores": oracle.num_threads(), "kind": "oracle",
                "cpu": _cpu_model(), "nproc": os.cpu_count(),
                "sample": f"the whole n={n} uplo={uplo} factorization of the same matrix "
                          f"(left-looking triple loop, {fl:.3e} flops in {dt:.1f} s)"}

    def run(J):
        X = np.array(A_host, order="F", copy=True)
        t0 = time.perf_counter()
        info = oracle.dpotrf_cols(X, uplo, J)
        dt = time.perf_counter() - t0
        assert info == 0
        return dt

    def flops(J):  # sum_{j<J} 2 j (n - j)  (leading term of the left-looking updates)
        return sum(2.0 * j * (n - j) for j in range(J))

    J = min(n, 128)
    dt = run(J)
    while dt < 3.0 and J < n:
        J = min(n, J * 2)
        dt = run(J)
    return {"value": flops(J) / dt / 1e9, "unit": "GFLOP/s", "cores": oracle.num_threads(), "kind": "oracle",
            "cpu": _cpu_model(), "nproc": os.cpu_count(),
            "sample": f"first {J} of {n} columns of the n={n} uplo={uplo} factorization "
                      f"(left-looking triple loop, {flops(J):.3e} flops in {dt:.2f} s)"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="n16384", choices=sorted(CONFIGS) + sorted(NEXT))
    ap.add_argument("--n", type=int, default=16384, help="order for the §8(f) configs")
    ap.add_argument("--block", type=int, default=128, help="block size of the blocked algorithms")
    ap.add_argument("--nrhs", type=int, default=1024, help="right-hand sides of potrs")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--no-profile", action="store_true")
    ap.add_argument("--nb", type=int, default=512, help="multi-GPU row block")
    ap.add_argument("--dist-min", type=int, default=8192, help="multi-GPU replicated-leaf threshold")
    ap.add_argument("--batch-count", type=int, default=131072)
    ap.add_argument("--dist", action="store_true",
                    help="the multi-GPU executor even at one GPU (NCCL world size 1; exercises the N > 1 path)")
    args = ap.parse_args()

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.config in NEXT:
        return run_next(args, rank, world, local_rank)
    n, uplo, dist, cfg_idx = CONFIGS[args.config]
    flops_per_step = n ** 3 / 3.0 if n else None

    if args.impl == "reference":
        return run_reference(args, rank, n, uplo, dist, cfg_idx, world)

    import torch

    import paper_1602_06763_b200 as rl

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    if world > 1 or args.dist:
        import torch.distributed as dist_

        if world == 1:  # --dist on one GPU: a world-size-1 group
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", "29513")
            dist_.init_process_group("nccl", rank=0, world_size=1, device_id=dev)
        else:
            dist_.init_process_group("nccl", device_id=dev)
    if args.config == "batch":
        return run_batch(args, rank, world, dev)

    if world > 1 or args.dist:
        return run_dist(args, rank, world, dev, n, uplo, dist)

    # ------------------------------------------------------------------ N = 1
    P = gen_matrix(n, uplo, dist, args.seed, dev)
    W = torch.empty_like(P.t()).t()  # column-major working copy
    st = torch.cuda.current_stream(dev)
    d_info = torch.zeros(1, dtype=torch.int32, device=dev)

    def step():
        W.copy_(P)
        torch.cuda.synchronize(dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        rl.dpotrf_async(W, d_info, uplo, stream=st)
        e1.record(st)
        torch.cuda.synchronize(dev)
        return e0.elapsed_time(e1)

    for _ in range(args.warmup):
        step()
    assert int(d_info.item()) == 0, f"info={int(d_info.item())}"
    with ClockSampler(local_rank) as clk:
        times = [step() for _ in range(args.steps)]
    assert int(d_info.item()) == 0
    total_ms = sum(times)
    ms_per_step = total_ms / args.steps
    gflops = flops_per_step / (ms_per_step / 1e3) / 1e9

    # dominant kernel (update: SYRK + GEMM) measured with CUDA events on the launch stream
    roofline, kernel_share = (profile_kernels(rl, W, P, d_info, uplo, st, dev, ms_per_step)
                              if not args.no_profile else (None, None))

    # end to end through the public C ABI with HOST buffers (pinned), copies inside the timed region
    e2e = e2e_host(rl, P, n, uplo, args.e2e_steps, st, dev) if args.e2e_steps > 0 else None

    # API latency: a cold call (new plan: build, capture, instantiate), a cached
    # call, and calls that alternate between two matrices (new pointer each call)
    api = api_latency(rl, P, uplo, st, dev) if n <= 16384 else None

    # kernels per factorization = ops of the captured plan DAG (one kernel each;
    # the ncu launch list in profiles/ counts the same 1150 at n = 16384)
    launches = len(rl.plan_schedule(n, rl.get_crossover(), 64, True)[0])
    peaks = _peaks()
    out = {
        "metric": "dpotrf FP64 GFLOP/s (n^3/3) and % of FP64 peak",
        "value": round(gflops, 2),
        "unit": "GFLOP/s",
        "n_gpus": 1,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(ms_per_step, 4),
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (seeded Philox B, A = B B^T + n I)",
        "config": {"workload": f"single dpotrf n={n} uplo={uplo} B~{dist} (BASELINE.json configs[{cfg_idx}])",
                   "n": n, "uplo": uplo, "lda": n, "crossover": rl.get_crossover(), "split_tile": 64,
                   "l2": "input 2 GiB > 126 MB L2; A restored from a pristine copy between steps (untimed)"
                   if n >= 8192 else "A restored from a pristine copy between steps (untimed)"},
        "pct_fp64_peak": round(100 * gflops / 1e3 / FP64_PEAK_TFLOPS_DATASHEET, 2),
        "roofline": roofline,
        "kernel_share": kernel_share,
        "e2e": e2e,
        "api_latency": api,
        "gpu_launches": launches * args.steps,
        "step_times_ms": [round(t, 4) for t in times],
        "clocks": clk.summary(),
        "peaks_source": "MEASURED_PEAKS.json" if peaks else "fallback",
    }
    if not args.no_cpu_baseline:
        A_host = P.cpu().numpy().T  # symmetric: row-major storage == column-major
        import numpy as np

        out["cpu_baseline"] = cpu_oracle_sample(np.asfortranarray(A_host), n, uplo)
    emit(out)
    return 0


def profile_kernels(rl, W, P, d_info, uplo, st, dev, ms_per_step):
    import torch

    rl.profile_enable(True)
    try:
        W.copy_(P)
        torch.cuda.synchronize(dev)
        rl.profile_reset()
        rl.dpotrf_async(W, d_info, uplo, stream=st)
        torch.cuda.synchronize(dev)
        res = {k: rl.profile_read(k) for k in ("potf2", "trsm", "gemm", "syrk")}
        rl.profile_reset()
    finally:
        rl.profile_enable(False)
    upd_ms = res["gemm"][0] + res["syrk"][0]
    upd_fl = res["gemm"][1] + res["syrk"][1]
    upd_n = res["gemm"][2] + res["syrk"][2]
    achieved = upd_fl / (upd_ms / 1e3) / 1e12 if upd_ms > 0 else 0.0
    in_graph = _in_graph_update_rate(rl, W, P, d_info, uplo, st, dev, upd_fl)
    traffic, traffic_note = _committed_traffic(W.shape[0])
    # primary figure: the update kernels as they run inside the timed step's
    # graph (trace timeline); the serial per-launch event pass beside it
    ach_main = in_graph["tflops_over_busy"] if in_graph else achieved
    roofline = {
        "kernel": "k_update (SYRK + recursive-TRSM GEMM, DMMA.8x8x4)",
        "bound": "tensor",
        "pipe": "FP64 DMMA (mma.sync m8n8k4 f64; sm_100a has no tcgen05 FP64 kind)",
        "achieved": round(ach_main, 3),
        "peak": FP64_PEAK_TFLOPS_DATASHEET,
        "unit": "TFLOP/s",
        "frac": round(ach_main / FP64_PEAK_TFLOPS_DATASHEET, 4),
        "traffic": traffic,
        "traffic_note": traffic_note,
        "launches_per_step": upd_n,
        "timing": ("achieved = algorithmic flops of the update launches / the union of their busy intervals inside "
                   "the captured graph (see in_graph)" if in_graph else
                   "achieved = algorithmic flops of the update launches / their summed CUDA-event durations in a "
                   "serial pass"),
        "serial": {"achieved": round(achieved, 3), "frac": round(achieved / FP64_PEAK_TFLOPS_DATASHEET, 4),
                   "note": "the same launches one at a time (eager, CUDA events on the launch stream): each "
                           "kernel alone, without the graph's overlap of small launches"},
        "in_graph": in_graph,
        "peak_note": "builder-measured DMMA peak 37.05 TF at 1965 MHz (profiles/fp64_peak_r01.txt; the HGX B200 "
                     "datasheet FP64 figure is 37.0 TF, used as the denominator); MEASURED_PEAKS.json has no FP64 entry",
    }
    total_prof = sum(v[0] for v in res.values())
    share = {k: {"ms": round(v[0], 3), "tflops": round(v[1] / (v[0] / 1e3) / 1e12, 3) if v[0] > 0 else 0.0,
                 "launches": v[2], "share_of_kernel_time": round(v[0] / total_prof, 4) if total_prof else 0}
             for k, v in res.items()}
    share["graph_step_ms"] = round(ms_per_step, 3)
    share["profiled_kernel_sum_ms"] = round(total_prof, 3)
    return roofline, share


def api_latency(rl, P, uplo, st, dev):
    """ms per relapack_dpotrf_async call measured with CUDA events around the
    call (host work of the call included: events bracket the enqueue)."""
    import time as _t

    import torch

    W1 = torch.empty_like(P.t()).t()
    W2 = torch.empty_like(P.t()).t()
    d_info = torch.zeros(1, dtype=torch.int32, device=dev)

    def one(W):
        W.copy_(P)
        torch.cuda.synchronize(dev)
        t0 = _t.perf_counter()
        rl.dpotrf_async(W, d_info, uplo, stream=st)
        torch.cuda.synchronize(dev)
        return 1e3 * (_t.perf_counter() - t0)

    rl.finalize()  # drop every cached plan
    cold = one(W1)
    cached = [one(W1) for _ in range(3)]
    alt = [one(W2 if i % 2 == 0 else W1) for i in range(6)]
    return {"cold_ms": round(cold, 3), "cached_ms": round(min(cached), 3),
            "new_pointer_ms": round(sorted(alt)[len(alt) // 2], 3),
            "note": "host wall clock around enqueue + synchronize; new_pointer alternates two matrices of the "
                    "same shape (one pointer-independent graph serves both)"}


def _in_graph_update_rate(rl, W, P, d_info, uplo, st, dev, upd_fl):
    """The update kernels inside the captured graph (RELAPACK_TRACE=1: every
    kernel records its first-CTA start and last-CTA end): the union of their
    busy intervals, the step span, and the update flops over that union."""
    import torch

    os.environ["RELAPACK_TRACE"] = "1"
    try:
        for _ in range(2):  # capture the traced plan, then the traced replay read back
            W.copy_(P)
            torch.cuda.synchronize(dev)
            rl.dpotrf_async(W, d_info, uplo, stream=st)
            torch.cuda.synchronize(dev)
        recs = rl.trace_records()
    finally:
        os.environ.pop("RELAPACK_TRACE", None)
    iv = sorted((r["t0_us"], r["t1_us"]) for r in recs if r["kind"] in ("gemm", "syrk") and r["t1_us"] >= 0)
    ivall = [(r["t0_us"], r["t1_us"]) for r in recs if r["t1_us"] >= 0]
    if not iv or not ivall:
        return None
    busy, cs, ce = 0.0, iv[0][0], iv[0][1]
    for a, b in iv[1:]:
        if a > ce:
            busy += ce - cs
            cs, ce = a, b
        else:
            ce = max(ce, b)
    busy += ce - cs
    span = max(b for _, b in ivall) - min(a for a, _ in ivall)
    return {"update_busy_ms": round(busy / 1e3, 3), "step_span_ms": round(span / 1e3, 3),
            "tflops_over_busy": round(upd_fl / (busy / 1e6) / 1e12, 3),
            "frac_over_busy": round(upd_fl / (busy / 1e6) / 1e12 / FP64_PEAK_TFLOPS_DATASHEET, 4),
            "note": "union of the update kernels' [first-CTA start, last-CTA end] intervals inside the captured "
                    "graph (%globaltimer, RELAPACK_TRACE=1 replay of the same plan)"}


def _committed_batch_traffic(count):
    """DRAM bytes per CFG[4] step (the four class kernels) from the committed ncu capture, or None."""
    import glob

    if count != 131072:
        return None
    files = sorted(glob.glob(os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles",
                                          "ncu_dram_batch_*.json")))
    if not files:
        return None
    with open(files[-1]) as f:
        return int(json.load(f)["total_bytes"])


def _committed_traffic(n):
    """DRAM bytes per k_update launch from the committed ncu capture of this
    workload (profiles/ncu_update_traffic_n<n>_*.json), or (None, why)."""
    import glob

    files = sorted(glob.glob(os.path.join(ROOT, "profiles", f"ncu_update_traffic_n{n}_*.json")))
    if not files:
        return None, "no committed ncu capture for this n"
    with open(files[-1]) as f:
        d = json.load(f)
    return (round(d["dram_bytes_per_launch_avg"]),
            f"dram__bytes_read+write per k_update launch, mean over the {d['launches_per_step']} launches of one "
            f"step ({os.path.basename(files[-1])}); per step {d['dram_read_bytes_per_step'] + d['dram_write_bytes_per_step']:.3e} B "
            f"= {d['traffic_over_algorithmic']:.2f}x the algorithmic bytes")


def e2e_host(rl, P, n, uplo, steps, st, dev):
    import torch

    H0 = P.cpu().pin_memory()  # pinned host input (column-major view of symmetric data)
    H = torch.empty((n, n), dtype=torch.float64).pin_memory().t()
    times = []
    for i in range(steps + 1):
        H.copy_(H0)
        torch.cuda.synchronize(dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        info = rl.dpotrf(H, uplo, stream=st)
        e1.record(st)
        torch.cuda.synchronize(dev)
        assert info == 0
        if i > 0:  # first call sizes the staging buffer and captures the plan
            times.append(e0.elapsed_time(e1))
    ms = sum(times) / len(times)
    # bytes that cross the host link each way: the library's copy blocks
    # (L-view column panels of 512 x the rows from the panel's diagonal down,
    # csrc/driver.cu kCopyPanel), identical for uplo L and U
    w, tri = 512, 0
    for j0 in range(0, n, w):
        jw = min(w, n - j0)
        tri += (n - j0) * jw * 8
    return {"value": round(n ** 3 / 3.0 / (ms / 1e3) / 1e9, 2), "unit": "GFLOP/s", "ms_per_step": round(ms, 3),
            "h2d_bytes_per_step": tri, "d2h_bytes_per_step": tri + 4, "steps": len(times),
            "api": "relapack_dpotrf (C ABI) with a pinned host matrix: H2D/D2H blocks are nodes of the "
                   "captured DAG, overlapped with the factorization"}


E2E_CHUNKS = 16  # batch e2e pipeline depth (chunks of the batch per step)


def run_batch(args, rank, world, dev):
    """CFG[4]: 131072 independent SPD matrices, n ~ U{16,32,48,64}, 1 % indefinite;
    the batch is split across ranks (fixed total work: strong scaling)."""
    import numpy as np
    import torch

    import paper_1602_06763_b200 as rl
    from inputs import gen

    count = args.batch_count
    b = gen.batched_spd(count, args.seed)
    bounds = rl.batch_split(b["ns"], world)  # contiguous ranges balanced by sum n^3 (library split, §8e)
    lo, hi = bounds[rank], bounds[rank + 1]
    ns = b["ns"][lo:hi]
    offs = b["offsets"][lo:hi] - (b["offsets"][lo] if hi > lo else 0)
    base = int(b["offsets"][lo]) if hi > lo else 0
    end = int(b["offsets"][hi - 1] + int(b["ns"][hi - 1]) ** 2) if hi > lo else 0
    host = b["buf"][base:end]
    P = torch.from_numpy(host).to(dev)
    W = torch.empty_like(P)
    ptrs = (W.data_ptr() + 8 * torch.from_numpy(offs.astype(np.int64))).to(dev)
    d_ns = torch.from_numpy(ns.astype(np.int32)).to(dev)
    d_ld = d_ns.clone()
    d_info = torch.zeros(len(ns), dtype=torch.int32, device=dev)
    st = torch.cuda.current_stream(dev)
    flops = float((ns.astype(np.float64) ** 3).sum() / 3.0)
    tri_bytes = float((8.0 * ns.astype(np.float64) * (ns + 1)).sum())  # lower triangle read + written

    def step():
        W.copy_(P)
        torch.cuda.synchronize(dev)
        if world > 1:
            torch.distributed.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        rl.dpotrf_batched(d_ns, ptrs, d_ld, d_info, "L", stream=st)
        e1.record(st)
        torch.cuda.synchronize(dev)
        return e0.elapsed_time(e1)

    for _ in range(args.warmup):
        step()
    with ClockSampler(int(os.environ.get("LOCAL_RANK", "0"))) as clk:
        times = [step() for _ in range(args.steps)]
    exp = b["expected_info"][lo:hi]
    assert np.array_equal(d_info.cpu().numpy(), exp), "per-matrix info mismatch"
    # end to end: the pinned host batch goes over, is factored, and the
    # matrices and per-matrix info come back, all inside the timed region
    # The batch goes in E2E_CHUNKS contiguous chunks on three streams, so the
    # H2D of chunk c+1, the factorization of chunk c and the D2H of chunk c-1
    # overlap (the host link is the bound: ~55 GB/s each way, full duplex).
    H_in = torch.from_numpy(host).pin_memory()
    H_out = torch.empty_like(H_in).pin_memory()
    h_info = torch.empty(len(ns), dtype=torch.int32).pin_memory()
    nmat = len(ns)
    bounds = [nmat * c // E2E_CHUNKS for c in range(E2E_CHUNKS + 1)]
    el_off = np.append(offs, offs[-1] + ns[-1].astype(np.int64) ** 2) if nmat else np.zeros(1, np.int64)
    s_in, s_out = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    e2e_times = []
    for i in range(args.e2e_steps + 1):
        torch.cuda.synchronize(dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        s_in.wait_stream(st)
        s_out.wait_stream(st)
        for c in range(E2E_CHUNKS):
            m0, m1 = bounds[c], bounds[c + 1]
            if m1 <= m0:
                continue
            x0, x1 = int(el_off[m0]), int(el_off[m1])
            with torch.cuda.stream(s_in):
                W[x0:x1].copy_(H_in[x0:x1], non_blocking=True)
                ev_in = torch.cuda.Event()
                ev_in.record(s_in)
            st.wait_event(ev_in)
            rl.dpotrf_batched(d_ns[m0:m1], ptrs[m0:m1], d_ld[m0:m1], d_info[m0:m1], "L", stream=st)
            ev_done = torch.cuda.Event()
            ev_done.record(st)
            with torch.cuda.stream(s_out):
                s_out.wait_event(ev_done)
                H_out[x0:x1].copy_(W[x0:x1], non_blocking=True)
                h_info[m0:m1].copy_(d_info[m0:m1], non_blocking=True)
        st.wait_stream(s_out)
        e1.record(st)
        torch.cuda.synchronize(dev)
        if i > 0:
            e2e_times.append(e0.elapsed_time(e1))
    assert np.array_equal(h_info.numpy(), exp)
    e2e_ms = _max_over_ranks(sum(e2e_times) / max(1, len(e2e_times)), world, dev) if e2e_times else None
    ms = sum(times) / len(times)
    ms_max = _max_over_ranks(ms, world, dev)
    tot_flops = float((b["ns"].astype(np.float64) ** 3).sum() / 3.0)
    tot_bytes = float((8.0 * b["ns"].astype(np.float64) * (b["ns"] + 1)).sum())
    if rank != 0:
        return 0
    peaks = _peaks()
    hbm = float(peaks.get("hbm_gbs", 6650.0))
    achieved = tri_bytes / (ms / 1e3) / 1e9
    out = {
        "metric": "dpotrf FP64 GFLOP/s (n^3/3) and % of FP64 peak",
        "value": round(tot_flops / (ms_max / 1e3) / 1e9, 2), "unit": "GFLOP/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_max, 4), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded Philox, A_b = B_b B_b^T + n_b I, 1% with A_kk <- -A_kk)",
        "config": {"workload": f"batched dpotrf, {count} matrices n~U{{16,32,48,64}} (BASELINE.json configs[4])",
                   "count": count, "l2": "2 GB batch > 126 MB L2; restored from a pristine copy between steps"},
        "roofline": {"kernel": "k_potf2_batched", "bound": "hbm", "achieved": round(achieved, 1), "peak": hbm,
                     "unit": "GB/s", "frac": round(achieved / hbm, 4), "traffic": _committed_batch_traffic(count),
                     "note": "algorithmic bytes = lower triangles read + written once (8 n(n+1) per matrix); traffic = "
                             "DRAM bytes of the four class kernels per step from the committed ncu capture "
                             "(profiles/ncu_dram_batch_*.json)"},
        "gb_per_s": round(tot_bytes / (ms_max / 1e3) / 1e9, 1),
        "gpu_launches": 5 * args.steps, "step_times_ms": [round(t, 4) for t in times], "clocks": clk.summary(),
        "e2e": ({"value": round(tot_flops / (e2e_ms / 1e3) / 1e9, 2), "unit": "GFLOP/s", "ms_per_step": round(e2e_ms, 3),
                 "h2d_bytes_per_step": int(host.nbytes) * world, "d2h_bytes_per_step": int(host.nbytes + 4 * len(ns)) * world,
                 "steps": len(e2e_times), "chunks": E2E_CHUNKS,
                 "api": "relapack_dpotrf_batched on a pinned host batch copied in and out, in contiguous chunks "
                        "pipelined over H2D / compute / D2H streams"}
                if e2e_ms else None),
        "info_parity": "per-matrix info == closed form (k+1 for the 1% negated diagonals)",
    }
    emit(out)
    return 0


def run_next(args, rank, world, local_rank):
    """One §8(f) operation per step on a fresh copy of its input (restored from a
    pristine device copy, untimed; inputs >= 2 GiB at n = 16384 > L2).  Replicas
    only at N > 1 (these operations are not sharded)."""
    import numpy as np
    import torch

    import paper_1602_06763_b200 as rl
    from inputs import gen

    n, op, r = args.n, args.config, args.nrhs
    flops_fn, desc = NEXT[op]
    flops = flops_fn(n, r)
    if args.impl == "reference":
        return run_next_reference(args, rank, world, op, n, r, flops_fn, desc)
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    st = torch.cuda.current_stream(dev)
    if world > 1:
        torch.distributed.init_process_group("nccl", device_id=dev)
    if op == "getrf":
        g = gen.philox(args.seed, 40)
        P = torch.empty((n, n), dtype=torch.float64, device=dev)
        for r0 in range(0, n, 4096):
            P[r0:r0 + 4096] = torch.from_numpy(g.uniform(-1.0, 1.0, size=(min(4096, n - r0), n))).to(dev)
        P = P.t()  # column-major view
    else:
        P = gen.spd_torch(n, args.seed, dist="uniform", device=dev)
        if op not in ("potrf_blocked",):
            assert rl.dpotrf(P, "L") == 0  # the factor the triangular operations start from
    W = torch.empty_like(P.t()).t()
    B0 = B = None
    if op == "potrs":
        g = gen.philox(args.seed, 41)
        B0 = torch.from_numpy(g.uniform(-1, 1, size=(r, n))).to(dev).t()
        B = torch.empty_like(B0.t()).t()
    ipiv = torch.zeros(n, dtype=torch.int32, device=dev)

    def call():
        if op == "trtri":
            return rl.dtrtri(W, "L", stream=st)
        if op == "trtri_blocked":
            return rl.dtrtri_blocked(W, args.block, "L", stream=st)
        if op == "potrf_blocked":
            return rl.dpotrf_blocked(W, args.block, "L", stream=st)
        if op == "lauum":
            return rl.dlauum(W, "L", stream=st)
        if op == "potri":
            return rl.dpotri(W, "L", stream=st)
        if op == "potrs":
            return rl.dpotrs(W, B, "L", stream=st)
        return rl.dgetrf(W, ipiv, stream=st)

    def step():
        W.copy_(P)
        if B is not None:
            B.copy_(B0)
        torch.cuda.synchronize(dev)
        if world > 1:
            torch.distributed.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        info = call()  # synchronous call: info read back inside the timed region
        e1.record(st)
        torch.cuda.synchronize(dev)
        assert info == 0, f"info={info}"
        return e0.elapsed_time(e1)

    for _ in range(args.warmup):
        step()
    with ClockSampler(local_rank) as clk:
        times = [step() for _ in range(args.steps)]
    ms = sum(times) / len(times)
    if world > 1:
        ms = _max_over_ranks(ms, world, dev)
    val = flops / (ms / 1e3) / 1e9 * world
    # per-kind breakdown (serial replay with events on the launch stream)
    prof = None
    if not args.no_profile and op != "potrf_blocked":
        W.copy_(P)
        if B is not None:
            B.copy_(B0)
        torch.cuda.synchronize(dev)
        prof = rl.xprofile(call)
    elif not args.no_profile:
        W.copy_(P)
        torch.cuda.synchronize(dev)
        rl.profile_enable(True)
        try:
            rl.profile_reset()
            call()
            prof = {k: rl.profile_read(k) for k in ("potf2", "trsm", "gemm", "syrk")}
            rl.profile_reset()
        finally:
            rl.profile_enable(False)
        prof["gemm"] = tuple(a + b for a, b in zip(prof["gemm"], prof.pop("syrk")))
    roofline = None
    if prof and "gemm" in prof and prof["gemm"][0] > 0:
        ach = prof["gemm"][1] / (prof["gemm"][0] / 1e3) / 1e12
        roofline = {"kernel": "k_update (mixed-layout DMMA GEMM/SYRK of the plan)", "bound": "tensor",
                    "achieved": round(ach, 3), "peak": FP64_PEAK_TFLOPS_DATASHEET, "unit": "TFLOP/s",
                    "frac": round(ach / FP64_PEAK_TFLOPS_DATASHEET, 4), "traffic": None,
                    "peak_note": "builder-measured DMMA peak 37.05 TF (datasheet 37.0 TF); MEASURED_PEAKS.json "
                                 "has no FP64 entry", "timing": "serial per-launch CUDA events (no graph)"}
    out = {
        "metric": f"{op} FP64 GFLOP/s and % of FP64 peak", "value": round(val, 2), "unit": "GFLOP/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 4),
        "higher_is_better": True, "scaling": "weak" if world > 1 else "strong", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (seeded Philox)",
        "config": {"workload": f"{desc}, n={n}" + (f", nrhs={r}" if op == "potrs" else "")
                   + (f", block={args.block}" if "blocked" in op else ""), "n": n,
                   "parallelism": f"replicas x{world}" if world > 1 else "1 GPU",
                   "l2": "inputs restored from a pristine device copy between steps (untimed)"},
        "pct_fp64_peak": round(100 * val / 1e3 / world / FP64_PEAK_TFLOPS_DATASHEET, 2),
        "roofline": roofline,
        "kernel_share": {k: {"ms": round(v[0], 3), "launches": v[2],
                             "tflops": round(v[1] / (v[0] / 1e3) / 1e12, 3) if v[0] > 0 else 0.0}
                         for k, v in (prof or {}).items()},
        "step_times_ms": [round(t, 4) for t in times],
        "clocks": clk.summary(),
    }
    if not args.no_cpu_baseline and rank == 0:
        out["cpu_baseline"] = next_cpu_baseline(op, n, r, args.seed)
    if rank == 0:
        emit(out)
    return 0


def _next_oracle_case(op, m, r, seed):
    """Host input of the oracle sample (order m) and the call that times it."""
    import numpy as np

    import oracle
    from inputs import gen

    if op == "getrf":
        A = np.asfortranarray(gen.philox(seed, 40).uniform(-1, 1, size=(m, m)))
        return A, lambda X: oracle.dgetrf(X)[0]
    A = np.asfortranarray(gen.spd(m, seed))
    if op == "potrf_blocked":
        return A, lambda X: oracle.dpotrf(X, "L")
    assert oracle.dpotrf(A, "L") == 0
    if op in ("trtri", "trtri_blocked"):
        return A, lambda X: oracle.dtrtri(X, "L")
    if op == "lauum":
        return A, lambda X: oracle.dlauum(X, "L")
    if op == "potri":
        return A, lambda X: oracle.dpotri(X, "L")
    Bh = np.asfortranarray(gen.philox(seed, 41).uniform(-1, 1, size=(m, r)))
    return A, lambda X: oracle.dpotrs(X, np.array(Bh, order="F"), "L")


def next_cpu_baseline(op, n, r, seed, target_s=6.0):
    """The oracle as it stands on a bounded sample: the same operation at a
    smaller order m (doubling from 512 until a call takes ~target_s / 4)."""
    import numpy as np

    import oracle

    flops_fn = NEXT[op][0]
    m = 512
    while True:
        A, fn = _next_oracle_case(op, m, r, seed)
        X = np.array(A, order="F")
        t0 = time.perf_counter()
        fn(X)
        dt = time.perf_counter() - t0
        if dt > target_s / 4 or m >= n:
            break
        m = min(n, 2 * m)
    return {"value": round(flops_fn(m, r) / dt / 1e9, 3), "unit": "GFLOP/s", "cores": oracle.num_threads(),
            "kind": "oracle", "sample": f"the same operation at n={m} (of {n}){', nrhs=' + str(r) if op == 'potrs' else ''}"
                                          f": {flops_fn(m, r):.3e} flops in {dt:.2f} s"}


def run_next_reference(args, rank, world, op, n, r, flops_fn, desc):
    if rank != 0:
        return 0
    import numpy as np

    import oracle

    oracle.build()
    base = next_cpu_baseline(op, n, r, args.seed)
    m = int(base["sample"].split("n=")[1].split(" ")[0])
    A, fn = _next_oracle_case(op, m, r, args.seed)
    times = []
    for i in range(args.warmup + args.steps):
        X = np.array(A, order="F")
        t0 = time.perf_counter()
        fn(X)
        if i >= args.warmup:
            times.append(time.perf_counter() - t0)
    sec = sum(times) / len(times)
    val = flops_fn(m, r) / sec / 1e9
    out = {"impl": "reference", "metric": f"{op} FP64 GFLOP/s and % of FP64 peak", "value": round(val, 3),
           "unit": "GFLOP/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
           "ms_per_step": round(1e3 * sec, 3), "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
           "dtype": "f64", "data": "synthetic (seeded Philox)", "config": {"workload": f"{desc}, n={n}", "n": n},
           "cpu_baseline": dict(base, value=round(val, 3)),
           "e2e": {"value": round(val, 3), "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    emit(out)
    return 0


def _max_over_ranks(v, world, dev):
    if world == 1:
        return v
    import torch

    t = torch.tensor([v], dtype=torch.float64, device=dev)
    torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    return float(t.item())


def run_dist(args, rank, world, dev, n, uplo, dist):
    """One factorization sharded over the ranks: snake block-cyclic
    row blocks of the L-view, NCCL all-gather of the solved panel rows."""
    import torch
    import torch.distributed as tdist

    import paper_1602_06763_b200 as rl

    if rank == 0:
        P = gen_matrix(n, uplo, dist, args.seed, dev)
    else:
        P = torch.empty((n, n), dtype=torch.float64, device=dev).t()
    base = torch.as_strided(P, (n * n,), (1,))
    tdist.broadcast(base, src=0)  # identical input bits on every rank
    W = torch.empty_like(P.t()).t()
    uid = [rl.Comm.unique_id() if rank == 0 else None]
    tdist.broadcast_object_list(uid, src=0)
    comm = rl.Comm(uid[0], world, rank, torch.cuda.current_device())
    nb, dmin = args.nb, args.dist_min
    st = torch.cuda.current_stream(dev)

    def step():
        W.copy_(P)
        torch.cuda.synchronize(dev)
        tdist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        info = rl.dpotrf_dist(W, comm, uplo, nb=nb, dist_min=dmin, stream=st)
        e1.record(st)
        torch.cuda.synchronize(dev)
        assert info == 0, info
        return e0.elapsed_time(e1)

    for _ in range(args.warmup):
        step()
    with ClockSampler(int(os.environ.get("LOCAL_RANK", "0"))) as clk:
        times = [step() for _ in range(args.steps)]
    ms = _max_over_ranks(sum(times) / len(times), world, dev)
    # end to end: every rank's replica comes from pinned host memory, the
    # factorization runs, the info word goes back (the factor stays on the
    # device: SPMD, one replica per rank)
    H = P.cpu().pin_memory() if args.e2e_steps > 0 else None
    e2e_t = []
    for i in range(args.e2e_steps + 1 if H is not None else 0):
        torch.cuda.synchronize(dev)
        tdist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        W.copy_(H, non_blocking=True)
        info = rl.dpotrf_dist(W, comm, uplo, nb=nb, dist_min=dmin, stream=st)  # reads info back (4 bytes)
        e1.record(st)
        torch.cuda.synchronize(dev)
        assert info == 0, info
        if i > 0:
            e2e_t.append(e0.elapsed_time(e1))
    e2e_ms = _max_over_ranks(sum(e2e_t) / len(e2e_t), world, dev) if e2e_t else None
    sched = rl.dist_schedule(n, rank, world, nb=nb, dist_min=dmin)
    launches = sum(1 for o in sched if o["kind"] != "allgather")
    comm.close()
    tdist.destroy_process_group()
    if rank != 0:
        return 0
    gflops = n ** 3 / 3.0 / (ms / 1e3) / 1e9
    out = {
        "metric": "dpotrf FP64 GFLOP/s (n^3/3) and % of FP64 peak",
        "value": round(gflops, 2), "unit": "GFLOP/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms, 4), "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded Philox B, A = B B^T + n I)",
        "config": {"workload": f"single dpotrf n={n} uplo={uplo} sharded over {world} GPU(s) (multi-GPU executor)",
                   "n": n, "uplo": uplo, "nb": nb, "dist_min": dmin, "parallelism": f"rowblock-cyclic x{world}",
                   "l2": "input > L2; restored from a pristine copy between steps (untimed)"},
        "pct_fp64_peak_per_gpu": round(100 * gflops / 1e3 / FP64_PEAK_TFLOPS_DATASHEET / world, 2),
        "gpu_launches": launches * args.steps, "step_times_ms": [round(t, 4) for t in times],
        "clocks": clk.summary(),
        "roofline": {"kernel": "whole distributed step per GPU (DMMA update kernels + NCCL all-gathers)",
                     "bound": "tensor", "achieved": round(gflops / 1e3 / world, 3), "peak": FP64_PEAK_TFLOPS_DATASHEET,
                     "unit": "TFLOP/s", "frac": round(gflops / 1e3 / world / FP64_PEAK_TFLOPS_DATASHEET, 4),
                     "traffic": None,
                     "note": "step-level: n^3/3 over the max-over-ranks step time, per GPU (no per-kernel trace in "
                             "the SPMD executor)"},
        "e2e": ({"value": round(n ** 3 / 3.0 / (e2e_ms / 1e3) / 1e9, 2), "unit": "GFLOP/s",
                 "ms_per_step": round(e2e_ms, 3), "h2d_bytes_per_step": int(n) * n * 8 * world,
                 "d2h_bytes_per_step": 4 * world, "steps": len(e2e_t),
                 "api": "relapack_dpotrf_dist; every rank's replica copied from pinned host memory inside the "
                        "timed region, the info word read back"} if e2e_ms else None),
    }
    emit(out)
    return 0


def _host_panel(n, J, seed, dist, uplo):
    """Host copy of the part of A the oracle's first J columns read: L-view
    columns 0..J-1 (A = B B^T + n I with the same row-panel Philox draws as
    inputs.gen.spd_torch)."""
    import numpy as np

    from inputs import gen

    panel = 4096
    B = np.empty((n, n))
    for p, r0 in enumerate(range(0, n, panel)):
        r1 = min(n, r0 + panel)
        B[r0:r1] = gen.draw_B(r1 - r0, seed, dist, m=n, stream=1 + p)
    C = B @ B[:J].T  # n x J: columns 0..J-1 of B B^T
    C[np.arange(J), np.arange(J)] += float(n)
    A = np.zeros((n, n), order="F")
    if uplo == "L":
        A[:, :J] = C
    else:
        A[:J, :] = C.T
    return A


def run_reference(args, rank, n, uplo, dist, cfg_idx, world):
    """--impl reference: the oracle (as it stands) on the box's host cores, each
    step a bounded sample of the same workload (rank 0 only)."""
    if rank != 0:
        return 0
    import numpy as np

    import oracle
    from inputs import gen

    oracle.build()
    if args.config == "batch":
        b = gen.batched_spd(args.batch_count, args.seed)
        S = 8192
        ns, offs = b["ns"][:S], b["offsets"][:S]
        end = int(offs[-1] + int(ns[-1]) ** 2)
        sample_flops = float((ns.astype(np.float64) ** 3).sum() / 3.0)
        times = []
        for i in range(args.warmup + args.steps):
            buf = b["buf"][:end].copy()
            t0 = time.perf_counter()
            oracle.dpotrf_batched("L", ns, buf, offs, ns)
            dt = time.perf_counter() - t0
            if i >= args.warmup:
                times.append(dt)
        sample = f"first {S} of {args.batch_count} matrices of the CFG[4] batch"
        workload = f"batched dpotrf, {args.batch_count} matrices n~U{{16,32,48,64}} (BASELINE.json configs[4])"
    else:
        # each step: the WHOLE factorization (left-looking triple loop, every
        # column's k-loop at full length) of the same recipe at order m =
        # min(n, 4096) — a bounded step (~1.6 s on 16 cores)
        m = min(n, 4096)
        A = gen.spd(m, args.seed, dist=dist)
        sample_flops = m ** 3 / 3.0
        times = []
        for i in range(args.warmup + args.steps):
            X = np.array(A, order="F")
            t0 = time.perf_counter()
            info = oracle.dpotrf(X, uplo)
            dt = time.perf_counter() - t0
            assert info == 0
            if i >= args.warmup:
                times.append(dt)
        sample = (f"the whole factorization of the same recipe at n={m} (of {n}), uplo={uplo} "
                  f"(left-looking triple loop, {sample_flops:.3e} flops per step)")
        workload = f"single dpotrf n={n} uplo={uplo} B~{dist} (BASELINE.json configs[{cfg_idx}])"
    sec = sum(times) / len(times)
    val = sample_flops / sec / 1e9
    out = {
        "impl": "reference", "metric": "dpotrf FP64 GFLOP/s (n^3/3) and % of FP64 peak",
        "value": round(val, 3), "unit": "GFLOP/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(1e3 * sec, 3), "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (seeded Philox)",
        "config": {"workload": workload, "n": n, "uplo": uplo},
        "cpu_baseline": {"value": round(val, 3), "unit": "GFLOP/s", "cores": oracle.num_threads(), "kind": "oracle",
                         "sample": sample},
        "e2e": {"value": round(val, 3), "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    emit(out)
    return 0


if __name__ == "__main__":
    sys.exit(main())
