# r3m: getrf panels on one thread-block cluster (DSMEM + cluster barrier) + permutation kernel vs the cooperative grid kernel
timeout 900 python -m pytest tests/test_gpu_next.py -q -m gpu -x -k "getrf" > gpurun_out/r3m_tests.txt 2>&1
for cl in 0 16 8; do RELAPACK_GETF2_CLUSTER=$cl python bench.py --config getrf --steps 3 --warmup 1 --no-cpu-baseline 2>gpurun_out/r3m_err_$cl.txt | tail -1 > gpurun_out/r3m_getrf_$cl.json; done
