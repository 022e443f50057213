# r3n: getrf after the unrolled rank-1 update; ncu launch list of one getrf step (cluster panels)
timeout 900 python -m pytest tests/test_gpu_next.py -q -m gpu -x -k "getrf" > gpurun_out/r3n_tests.txt 2>&1
for cl in 0 16; do RELAPACK_GETF2_CLUSTER=$cl python bench.py --config getrf --steps 3 --warmup 1 --no-cpu-baseline 2>gpurun_out/r3n_err_$cl.txt | tail -1 > gpurun_out/r3n_getrf_$cl.json; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r3n_launches.csv python bench.py --config getrf --steps 1 --warmup 0 --no-cpu-baseline --no-profile > gpurun_out/r3n_ncu.log 2>&1
