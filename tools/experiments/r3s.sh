# r3s: node-128 with one inlined potf2_smem copy for both diagonal blocks (RELAPACK_NODE_ONE_POTF2)
cd tools/microbench
for v in 0 1; do nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -I ../../include -DRELAPACK_NODE_ONE_POTF2=$v -o /tmp/bk$v base_kernels.cu && /tmp/bk$v | grep "potf2 n=128\|node128 phases\|potf2 n=96" | sed "s/^/one=$v /" >> ../../gpurun_out/r3s_base.txt; done
cd ../..
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_kernels.py -q -m gpu -x > gpurun_out/r3s_tests.txt 2>&1
python tools/ab_bench.py abtest/old/librelapack_b200.so paper_1602_06763_b200/librelapack_b200.so n4096 3 > gpurun_out/r3s_ab4k.txt 2>&1
python tools/ab_bench.py abtest/old/librelapack_b200.so paper_1602_06763_b200/librelapack_b200.so n256 2 > gpurun_out/r3s_ab256.txt 2>&1
