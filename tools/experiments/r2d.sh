python tools/ab_trees.py . abtest/r1tree n4096 3 > gpurun_out/r2d_ab.log 2>&1
python tools/ab_trees.py abtest/treeB abtest/r1tree n4096 3 >> gpurun_out/r2d_ab.log 2>&1
RELAPACK_TRACE=1 python tools/trace_timeline.py 4096 L > gpurun_out/r2d_trace_cur.txt 2>&1
(cd abtest/r1tree && RELAPACK_TRACE=1 python ../../tools/trace_timeline.py 4096 L > ../../gpurun_out/r2d_trace_r1.txt 2>&1)
timeout 1500 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_next.py tests/test_gpu_parity.py tests/test_gpu_dist.py tests/test_gpu_variants.py -q --durations=20 > gpurun_out/r2d_tests.log 2>&1
