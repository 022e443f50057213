"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list by kernel."""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
gi = h.index("Grid Size")
agg = collections.defaultdict(list)
scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
for r in rows[1:]:
    v = float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
    name = r[ki].split("(")[0].replace("void ", "")[-48:]
    agg[name].append(v)
tot = sum(sum(v) for v in agg.values())
for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    print(f"{k:48s} n={len(v):5d} sum={sum(v)/1e3:9.3f} ms ({100*sum(v)/tot:5.1f}%) mean={sum(v)/len(v):8.2f} us min={min(v):7.2f} max={max(v):8.2f}")
