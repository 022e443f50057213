"""DRAM traffic of the update kernels of one factorization against their
algorithmic bytes, from an ncu metrics CSV of tools/ncu_step.py (two
factorizations; the last one's k_update launches are used).
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
      -k regex:k_update --csv --log-file t.csv python tools/ncu_step.py 16384 U
  python tools/update_traffic.py t.csv 16384 out.json"""
import csv
import json
import sys

sys.path.insert(0, ".")
import paper_1602_06763_b200 as rl

path, n, out = sys.argv[1], int(sys.argv[2]), sys.argv[3]
rows = [r for r in csv.reader(open(path)) if len(r) > 10]
h = rows[0]
ii, mi, vi, ui = h.index("ID"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
launch = {}
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-6, "nsecond": 1e-6, "us": 1e-3,
         "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}
for r in rows[1:]:
    launch.setdefault(int(r[ii]), {})[r[mi]] = float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
ops, _ = rl.plan_schedule(n, rl.get_crossover(), 64, True)
upd = [o for o in ops if o["kind"] in ("gemm", "syrk")]
ids = sorted(launch)[-len(upd):]
rd = sum(launch[i].get("dram__bytes_read.sum", 0) for i in ids)
wr = sum(launch[i].get("dram__bytes_write.sum", 0) for i in ids)
ms = sum(launch[i].get("gpu__time_duration.sum", 0) for i in ids)
alg = 0.0
for o in upd:
    m, nn, k = o["m"], o["n"], o["k"]
    if o["kind"] == "syrk":
        alg += 8.0 * (nn * k + nn * (nn + 1))  # A once, lower triangle of C read + written
    else:
        alg += 8.0 * (m * k + nn * k + 2 * m * nn)
res = {"config": f"n{n} (one factorization, graph replay), kernel k_update (GEMM+SYRK)",
       "command": "ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none "
                  f"-k regex:k_update python tools/ncu_step.py {n} U; python tools/update_traffic.py",
       "launches_per_step": len(upd), "dram_read_bytes_per_step": rd, "dram_write_bytes_per_step": wr,
       "dram_bytes_per_launch_avg": (rd + wr) / len(upd), "algorithmic_bytes_per_step": alg,
       "traffic_over_algorithmic": (rd + wr) / alg, "ncu_serial_kernel_ms_per_step": ms,
       "note": "algorithmic bytes = A + B read once, C read and written once, per update launch (SYRK: lower triangle)"}
json.dump(res, open(out, "w"), indent=1)
print(json.dumps(res, indent=1))
