B="python bench.py --no-cpu-baseline --e2e-steps 0 --no-profile"
for d in 1 2 3 4; do for cfg in n4096 n16384; do
  RELAPACK_LOOKAHEAD_DEPTH=$d $B --config $cfg | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('depth=$d $cfg', d['ms_per_step'], d['value'])"
done; done
RELAPACK_LOOKAHEAD_DEPTH=2 timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "recursive or crossover" 2>&1 | tail -1
