set -x
python -m pytest tests/test_gpu_parity.py -x -q -k "node256 or node128 or recursive or lda or P1 or P7 or crossover" 2>&1 | tail -5
for rep in 1 2; do
for c in 128 256; do
  for cfg in n256 n4096 n16384; do
    RELAPACK_CROSSOVER=$c python bench.py --config $cfg --steps 10 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('c=$c', '$cfg', d['ms_per_step'], d.get('roofline',{}).get('frac'))"
  done
done
done
