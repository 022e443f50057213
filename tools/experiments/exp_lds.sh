# update kernel fragment reads as LDS (shared address space kept) — parity + bench lines
python -m pytest tests/test_gpu_kernels.py tests/test_gpu_fullsize.py -x -q 2>&1 | tail -3
for cfg in n16384 n4096 n65536 trtri lauum potrs getrf; do
  python bench.py --config $cfg 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('$cfg', d['ms_per_step'], d['value'], d.get('roofline',{}).get('frac'), d.get('clocks',{}).get('sm_mhz'))"
done
