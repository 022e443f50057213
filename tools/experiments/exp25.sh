B="python bench.py --no-cpu-baseline --e2e-steps 0 --no-profile"
for db in 1 0; do for bulk in 132 116; do for cfg in n16384 n4096; do
  RELAPACK_DEFER_B21=$db RELAPACK_BULK_CTAS=$bulk $B --config $cfg | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('defer_b21=$db bulk=$bulk $cfg', d['ms_per_step'], d['value'])"
done; done; done
