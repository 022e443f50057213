# r2n: staged loads in the x kernels, decoupled interchange warps in the getrf panel; dist local-first SYRK
timeout 900 python -m pytest tests/test_gpu_next.py tests/test_gpu_dist.py -q -x > gpurun_out/r2n_tests.log 2>&1
for c in trtri lauum potri potrs getrf; do
  timeout 900 python bench.py --config $c --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/r2n_next_$c.json 2> gpurun_out/r2n_next_$c.err
done
timeout 900 python bench.py --config trtri_blocked --n 4096 --block 128 --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/r2n_next_trtri_blocked.json 2>&1
timeout 600 python tools/trtri_breakdown.py 16384 > gpurun_out/r2n_trtri_breakdown.txt 2>&1
timeout 600 python tools/dist_world1.py 16384 8192 512 > gpurun_out/r2n_dist_world1.txt 2>&1
