# r2m: faster k_tri_rows (unrolled dot products over masked T), getrf interchanges folded into the panel kernel
timeout 900 python -m pytest tests/test_gpu_next.py -q -x > gpurun_out/r2m_tests.log 2>&1
for c in trtri lauum potri potrs getrf; do
  timeout 900 python bench.py --config $c --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/r2m_next_$c.json 2> gpurun_out/r2m_next_$c.err
done
timeout 900 python bench.py --config trtri_blocked --n 4096 --block 128 --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/r2m_next_trtri_blocked.json 2>&1
