# tail split of the big 128-tile grids (RELAPACK_TAIL_SPLIT): kernel tests, then A/B on one box
python -m pytest tests/test_gpu_kernels.py -x -q 2>&1 | tail -2
for rep in 1 2; do
for t in 0 1; do
  for cfg in n16384 n65536 trtri lauum; do
    RELAPACK_TAIL_SPLIT=$t python bench.py --config $cfg --steps 8 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('tail=$t', '$cfg', d['ms_per_step'], d.get('roofline',{}).get('frac'))"
  done
done
done
