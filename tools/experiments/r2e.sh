# r2e: base-kernel microbench (round-1 sources vs current), n=4096 A/B, the regrow test
./abtest/base_kernels_r1 > gpurun_out/r2e_bk_r1.txt 2>&1
./abtest/base_kernels_cur > gpurun_out/r2e_bk_cur.txt 2>&1
python tools/ab_trees.py . abtest/r1tree n4096 3 > gpurun_out/r2e_ab.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "regrow or subnormal or node128" > gpurun_out/r2e_tests.log 2>&1
