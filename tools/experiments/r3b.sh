# r3b: panel factorization with a redundant per-lane 8x8 diagonal block (RELAPACK_PANEL_BD) vs the shuffle chain
cd tools/microbench
for bd in 0 1; do nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -I ../../include -DRELAPACK_PANEL_BD=$bd -o /tmp/bk$bd base_kernels.cu && /tmp/bk$bd | grep potf2 | sed "s/^/bd=$bd /" >> ../../gpurun_out/r3b_base.txt; done
cd ../..
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_kernels.py -q -m gpu -x -k "potf2 or base or node or recurs" > gpurun_out/r3b_tests.txt 2>&1
python tools/ab_bench.py abtest/old/librelapack_b200.so paper_1602_06763_b200/librelapack_b200.so n4096 3 > gpurun_out/r3b_ab4k.txt 2>&1
python tools/ab_bench.py abtest/old/librelapack_b200.so paper_1602_06763_b200/librelapack_b200.so n256 2 > gpurun_out/r3b_ab256.txt 2>&1
