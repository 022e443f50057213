# r4c: debug: epoch exchange with an additional grid barrier
cd tools/microbench
rm -f /tmp/gpd; nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -I ../../include -DRELAPACK_GETF2_POLL_DEBUG_BARRIER -o /tmp/gpd getf2_probe.cu
for mw in "33 32 32" "1024 32 32"; do timeout 60 /tmp/gpd $mw | grep -v "^cluster\|^m=" >> ../../gpurun_out/r4c_probe.txt; done
