B="python bench.py --no-cpu-baseline --e2e-steps 0 --no-profile"
for ch in 1 2 4; do for db in 1 0; do for cfg in n16384 n4096; do
  RELAPACK_B21_CHUNKS=$ch RELAPACK_DEFER_B21=$db $B --config $cfg | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('b21_chunks=$ch defer_b21=$db $cfg', d['ms_per_step'], d['value'])"
done; done; done
RELAPACK_B21_CHUNKS=4 timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "recursive or crossover" 2>&1 | tail -1
