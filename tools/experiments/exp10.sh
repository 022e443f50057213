B="python bench.py --no-cpu-baseline --e2e-steps 0 --no-profile"
for r in 0 4096 2048; do for cfg in n16384; do
  RELAPACK_TRSM_ROWS=$r $B --config $cfg | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('trsm_rows=$r $cfg', d['ms_per_step'], d['value'])"
done; done
for b in 132 140 124 0; do
  RELAPACK_BULK_CTAS=$b $B --config n16384 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bulk=$b n16384', d['ms_per_step'], d['value'])"
done
