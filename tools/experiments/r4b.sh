# r4b: getf2 epoch-stamped exchange vs grid barrier on one panel (pivots and values must agree)
cd tools/microbench
rm -f /tmp/gp; nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -I ../../include -o /tmp/gp getf2_probe.cu
for mw in "33 32 32" "64 32 32" "1024 32 32" "16384 32 128" "16384 32 111" "4096 32 32" "8192 16 64"; do timeout 60 /tmp/gp $mw | grep -v "^cluster\|^m=" >> ../../gpurun_out/r4b_probe.txt; done
