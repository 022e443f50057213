# ncu launch list of the bench command itself (profiling recipe): every kernel of
# `bench.py --steps 1 --warmup 3` (no profile pass / e2e / cpu baseline), then the
# last factorization's launches summarised by kernel
CMD="python bench.py --steps 1 --warmup 3 --no-profile --e2e-steps 0 --no-cpu-baseline"
$CMD > gpurun_out/bench_plain.log 2>&1 && tail -c 200 gpurun_out/bench_plain.log
ncu --metrics gpu__time_duration.sum --clock-control none -c 8000 --csv --log-file gpurun_out/launches_bench.csv $CMD > gpurun_out/bench_ncu.log 2>&1
python - <<'PY'
import csv, collections
rows = [r for r in csv.reader(open("gpurun_out/launches_bench.csv")) if len(r) > 10]
h = rows[0]
ki, vi, ui, idi = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit"), h.index("ID")
sc = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
ks = [(r[ki].split("(")[0].replace("void ", "").split("::")[-1], float(r[vi].replace(",", "")) * sc.get(r[ui], 1.0)) for r in rows[1:]]
plan = [k for k in ks if k[0].startswith(("k_update", "k_trsm", "k_potf2"))]
print(f"{len(ks)} launches in the bench command, {len(plan)} plan kernels ({len(plan) // 1150} factorizations of 1150)")
last = plan[-1150:]
agg = collections.defaultdict(list)
for k, v in last:
    agg[k].append(v)
tot = sum(v for _, v in last)
print(f"last factorization (the timed step): {len(last)} launches, {tot / 1e3:.3f} ms summed (serialised, cold cache)")
for k, vs in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    print(f"  {k:28s} n={len(vs):5d} sum={sum(vs) / 1e3:9.3f} ms ({100 * sum(vs) / tot:5.1f}%) mean={sum(vs) / len(vs):9.2f} us")
PY
