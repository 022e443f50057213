B="python bench.py --no-cpu-baseline --e2e-steps 0 --no-profile"
for m8 in 4096 2048 1024 8192; do for cfg in n16384 n4096; do
  RELAPACK_TRSM_NW8_FROM=$m8 $B --config $cfg | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('nw8_from=$m8 $cfg', d['ms_per_step'], d['value'])"
done; done
