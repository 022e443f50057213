# r3g: batched warp kernel with per-panel stores (early register release)
cd tools/microbench
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -I ../../include -o /tmp/bprobe batched_probe.cu
for tm in 0 1; do RELAPACK_BATCH_TEAM=$tm /tmp/bprobe | sed "s/^/team=$tm /" >> ../../gpurun_out/r3g_probe.txt; done
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -I ../../include -o /tmp/regchol regchol_probe.cu && /tmp/regchol > ../../gpurun_out/r3g_regchol.txt 2>&1
