# r2f: after-the-fact subnormal detection: base-kernel microbench vs round 1, n=4096 A/B, parity tests
./abtest/base_kernels_cur > gpurun_out/r2f_bk_cur.txt 2>&1
python tools/ab_trees.py . abtest/r1tree n4096 3 > gpurun_out/r2f_ab.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_kernels.py -q -x > gpurun_out/r2f_tests.log 2>&1
