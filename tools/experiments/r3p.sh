# r3p: getrf cluster panel: CTA size 256 / 512 / 1024, direct pivot-column load
cd tools/microbench
for t in 256 512 1024; do nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -I ../../include -DRELAPACK_GETF2_CL_THREADS=$t -o /tmp/gp$t getf2_probe.cu
for mw in "16384 16" "8192 32" "1024 32"; do /tmp/gp$t $mw | sed "s/^/threads=$t /" >> ../../gpurun_out/r3p_probe.txt; done; done
