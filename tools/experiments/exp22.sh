./tools/microbench/update_small | grep "(auto)"
B="python bench.py --no-cpu-baseline --e2e-steps 0 --no-profile"
for s128 in 1 0; do for cfg in n4096 n16384 n256; do
  RELAPACK_SPLIT128=$s128 $B --config $cfg | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('split128=$s128 $cfg', d['ms_per_step'], d['value'])"
done; done
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -1
