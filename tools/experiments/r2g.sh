# r2g: exact-fallback cost (microbench), rebased plan graphs: tests + bench n4096 / n16384
./abtest/base_kernels_cur > gpurun_out/r2g_bk_cur.txt 2>&1
./abtest/base_kernels_nofb > gpurun_out/r2g_bk_nofb.txt 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_kernels.py tests/test_gpu_next.py tests/test_gpu_dist.py tests/test_gpu_variants.py -q -x > gpurun_out/r2g_tests.log 2>&1
python bench.py --config n4096 --no-cpu-baseline > gpurun_out/r2g_b4k.json 2>gpurun_out/r2g_b4k.err
python bench.py --no-cpu-baseline > gpurun_out/r2g_b16k.json 2>gpurun_out/r2g_b16k.err
python tools/ab_trees.py . abtest/r1tree n4096 3 > gpurun_out/r2g_ab.log 2>&1
