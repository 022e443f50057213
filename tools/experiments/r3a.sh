# batched K2 diagnosis: register-factorization cycles vs warps/SM; ncu source/stall capture of the 64-class
set -x
cd tools/microbench
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -o /tmp/regchol regchol_probe.cu && /tmp/regchol > ../../gpurun_out/r3a_regchol.txt 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -I ../../include -o /tmp/bprobe batched_probe.cu && /tmp/bprobe > ../../gpurun_out/r3a_bprobe.txt 2>&1
cd ../..
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_batched_cls -c 4 -o gpurun_out/r3a_batch python bench.py --config batch --steps 1 --warmup 0 > gpurun_out/r3a_ncu.log 2>&1
python bench.py --config batch --steps 10 --warmup 3 > gpurun_out/r3a_bench_batch.json 2>/dev/null
python bench.py --config n4096 --steps 10 --warmup 3 > gpurun_out/r3a_bench_n4096.json 2>/dev/null
python bench.py --config n256 --steps 10 --warmup 3 > gpurun_out/r3a_bench_n256.json 2>/dev/null
