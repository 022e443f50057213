"""A/B of two source trees on one box (each runs its own bench.py in its own
process, alternating): python tools/ab_trees.py TREE_A TREE_B CONFIG REPS [extra bench args]"""
import json
import subprocess
import sys

a, b, cfg, reps = sys.argv[1], sys.argv[2], sys.argv[3], int(sys.argv[4])
extra = sys.argv[5:]
for r in range(reps):
    for tree in (a, b):
        cmd = [sys.executable, "bench.py", "--config", cfg, "--steps", "20", "--warmup", "3", "--no-profile",
               "--e2e-steps", "0", "--no-cpu-baseline", *extra]
        out = subprocess.run(cmd, capture_output=True, text=True, cwd=tree).stdout
        lines = [x for x in out.splitlines() if x.startswith("{")]
        print(tree, cfg, json.loads(lines[-1])["ms_per_step"] if lines else "FAILED", flush=True)
