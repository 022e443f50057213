B="python bench.py --no-cpu-baseline --e2e-steps 0 --no-profile"
for kt in 8 4 2; do for cfg in n4096 n16384; do
  RELAPACK_SPLITK_KT=$kt $B --config $cfg | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('splitk_kt=$kt $cfg', d['ms_per_step'], d['value'])"
done; done
RELAPACK_SPLITK_KT=2 timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "recursive or crossover or node128" 2>&1 | tail -1
