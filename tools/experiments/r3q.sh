# r3q: register-resident cluster panel (k_getf2_clr): probe, tests, getrf bench vs cooperative kernel
cd tools/microbench
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -I ../../include -o /tmp/gp getf2_probe.cu
for mw in "16384 16" "8192 32" "1024 32" "32768 8"; do /tmp/gp $mw >> ../../gpurun_out/r3q_probe.txt; done
cd ../..
timeout 900 python -m pytest tests/test_gpu_next.py -q -m gpu -x -k "getrf" > gpurun_out/r3q_tests.txt 2>&1
for cl in 0 16; do RELAPACK_GETF2_CLUSTER=$cl python bench.py --config getrf --steps 3 --warmup 1 --no-cpu-baseline 2>gpurun_out/r3q_err_$cl.txt | tail -1 > gpurun_out/r3q_getrf_$cl.json; done
