# r3x: per-column phases of the cooperative getrf panel kernel (k_getf2) at several CTA row counts
cd tools/microbench
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -I ../../include -o /tmp/gp getf2_probe.cu
for rc in 32 64 128; do for mw in "16384 32" "4096 32"; do RELAPACK_GETF2_CLUSTER=16 /tmp/gp $mw $rc | grep coop >> ../../gpurun_out/r3x_probe.txt; done; done
