"""A/B of two library builds on one box: python tools/ab_bench.py LIB_A LIB_B CONFIG REPS
(loads each .so in its own process through the package's library_path)."""
import json
import subprocess
import sys

a, b, cfg, reps = sys.argv[1], sys.argv[2], sys.argv[3], int(sys.argv[4])
code = ("import sys, runpy; sys.path.insert(0, '.'); import paper_1602_06763_b200 as rl; rl.library_path = {lib!r}; "
        "sys.argv = ['bench.py', '--config', {cfg!r}, '--steps', '20', '--warmup', '3', '--no-profile', "
        "'--e2e-steps', '0', '--no-cpu-baseline']; runpy.run_path('bench.py', run_name='__main__')")
for r in range(reps):
    for lib in (a, b):
        out = subprocess.run([sys.executable, "-c", code.format(lib=lib, cfg=cfg)], capture_output=True, text=True).stdout
        line = [x for x in out.splitlines() if x.startswith("{")][-1]
        print(lib.split("/")[-1], cfg, json.loads(line)["ms_per_step"], flush=True)
