B="python bench.py --no-cpu-baseline --e2e-steps 0 --no-profile"
for m in 0 1; do for cfg in n4096 n16384; do
  RELAPACK_SPLITK_MID=$m $B --config $cfg | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('splitk_mid=$m $cfg', d['ms_per_step'], d['value'])"
done; done
