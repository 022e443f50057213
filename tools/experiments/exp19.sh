./tools/microbench/update_small | grep "(auto)"
B="python bench.py --no-cpu-baseline --e2e-steps 0 --no-profile"
for th in 0 32 64; do for cfg in n4096 n256 n16384; do
  RELAPACK_TILE32_BELOW=$th $B --config $cfg | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('tile32_below=$th $cfg', d['ms_per_step'], d['value'])"
done; done
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
RELAPACK_TILE32_BELOW=100000 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -1
