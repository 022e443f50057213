# TRSM row-panel split sweep (RELAPACK_TRSM_ROWS) at n=4096 / 16384
B="python bench.py --no-cpu-baseline --e2e-steps 0 --no-profile"
for r in 0 512 1024 2048 4096; do
  for c in n4096 n16384; do
    RELAPACK_TRSM_ROWS=$r $B --config $c | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('rows=$r $c', d['ms_per_step'], d['value'])"
  done
done
