B="python bench.py --no-cpu-baseline --e2e-steps 0 --no-profile"
for lo in 1 0; do for bulk in 132 148; do for cfg in n4096 n16384; do
  RELAPACK_DEFER_LOW=$lo RELAPACK_BULK_CTAS=$bulk $B --config $cfg | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('defer_low=$lo bulk=$bulk $cfg', d['ms_per_step'], d['value'])"
done; done; done
