#!/bin/bash
# Lookahead / DAG-capture sweep: ms per factorization for several knob settings.
mkdir -p gpurun_out
for cfg in n4096 n16384; do
  for env in "RELAPACK_DAG=0 RELAPACK_LOOKAHEAD=0" "RELAPACK_DAG=1 RELAPACK_LOOKAHEAD=0" \
             "RELAPACK_DAG=1 RELAPACK_LOOKAHEAD=1" "RELAPACK_DAG=1 RELAPACK_LOOKAHEAD=1 RELAPACK_BULK_CTAS=132" \
             "RELAPACK_DAG=1 RELAPACK_LOOKAHEAD=1 RELAPACK_BULK_CTAS=116"; do
    r=$(env $env timeout 300 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline --no-profile --e2e-steps 1 2>&1 | tail -1)
    echo "$cfg | $env | $(echo "$r" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["value"])' 2>&1)"
  done
done
