# r3o: getrf cluster panel phase probes (tools/microbench/getf2_probe.cu)
cd tools/microbench
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -I ../../include -o /tmp/gp getf2_probe.cu
for mw in "16384 16" "8192 32" "1024 32"; do /tmp/gp $mw >> ../../gpurun_out/r3o_probe2.txt; done
