# r3l: register factorization with panel P-1's trailing DMMAs spread over panel P's column steps (RELAPACK_REG_DEFER)
cd tools/microbench
for d in 0 1; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -I ../../include -DRELAPACK_REG_DEFER=$d -o /tmp/regchol$d regchol_probe.cu && /tmp/regchol$d | sed "s/^/defer=$d /" >> ../../gpurun_out/r3l_regchol.txt
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -I ../../include -DRELAPACK_REG_DEFER=$d -o /tmp/bprobe$d batched_probe.cu && /tmp/bprobe$d | sed "s/^/defer=$d /" >> ../../gpurun_out/r3l_probe.txt
done
cd ../..
timeout 900 python -m pytest tests -q -m gpu -x -k "batch or base or potf2" > gpurun_out/r3l_tests.txt 2>&1
python bench.py --config batch --no-cpu-baseline > gpurun_out/r3l_bench.json 2>/dev/null
