# r3i: batched after the spill fix + single load/store paths: tests, probe, bench
cd tools/microbench
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -I ../../include -o /tmp/bprobe batched_probe.cu && /tmp/bprobe > ../../gpurun_out/r3i_probe.txt
cd ../..
timeout 900 python -m pytest tests -q -m gpu -x -k "batch" > gpurun_out/r3i_tests.txt 2>&1
python bench.py --config batch --no-cpu-baseline > gpurun_out/r3i_bench.json 2>gpurun_out/r3i_bench.err
