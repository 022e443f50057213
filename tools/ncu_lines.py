"""Aggregate ncu --page source --print-source cuda,sass CSV stall samples by CUDA source line.
  ncu -i rep --page source --csv --print-source cuda,sass > x.csv; python tools/ncu_lines.py x.csv [top]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
agg, srcl, cur, hdr, si = collections.Counter(), {}, "?", None, None
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        si = r.index("Warp Stall Sampling (All Samples)")
        continue
    if hdr is None or len(r) <= si or not r[0].isdigit():
        continue
    try:
        v = float(r[si] or 0)
    except ValueError:
        continue
    agg[(cur, int(r[0]))] += v
    if r[1].strip():
        srcl[(cur, int(r[0]))] = r[1].strip()[:90]
tot = sum(agg.values()) or 1
print("total samples", tot)
for k, v in agg.most_common(top):
    print(f"{100 * v / tot:5.1f}% {k[0]}:{k[1]} {srcl.get(k, '')}")
