# r3z: TRSM base (k_trsm_reg) phases and times, m = 128 .. 16384
cd tools/microbench
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -I ../../include -o /tmp/bk base_kernels.cu && /tmp/bk | grep "trsm" > ../../gpurun_out/r3z_base.txt
