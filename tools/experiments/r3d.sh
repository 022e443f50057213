# r3d: two-warp team kernel for the 48/64 batched classes vs the warp kernel
cd tools/microbench
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -I ../../include -o /tmp/bprobe batched_probe.cu
for tm in 0 1; do RELAPACK_BATCH_TEAM=$tm /tmp/bprobe | sed "s/^/team=$tm /" >> ../../gpurun_out/r3d_probe.txt; done
cd ../..
timeout 900 python -m pytest tests -q -m gpu -x -k "batch" > gpurun_out/r3d_tests.txt 2>&1
for tm in 0 1 0 1; do RELAPACK_BATCH_TEAM=$tm python bench.py --config batch --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('team=$tm', d['ms_per_step'])" >> gpurun_out/r3d_bench.txt; done
