# scheduling knobs re-swept under the three priority levels (same box)
run() { python bench.py --config $2 --steps 20 --warmup 3 --no-profile --e2e-steps 0 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$1 $2', d['ms_per_step'])"; }
for c in n16384 n4096; do
  run default $c
  RELAPACK_DEFER_B21=0 run b21_nodefer $c
  RELAPACK_BULK_CTAS=124 run bulk124 $c
  RELAPACK_BULK_CTAS=140 run bulk140 $c
  RELAPACK_BULK_MIN_GF=8 run bmin8 $c
  RELAPACK_BULK_MIN_GF=32 run bmin32 $c
  RELAPACK_PDL=1 run pdl1 $c
  RELAPACK_LOOKAHEAD_DEPTH=2 run la2 $c
  run default $c
done
