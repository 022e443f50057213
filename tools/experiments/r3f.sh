# r3f: team kernel phase probes (48/64 classes); fused panel A/B (r3e)
cd tools/microbench
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -I ../../include -DRELAPACK_TEAM_PROBE -o /tmp/bprobe batched_probe.cu && RELAPACK_BATCH_TEAM=1 /tmp/bprobe > ../../gpurun_out/r3f_probe.txt 2>&1
cd ../..
bash tools/experiments/r3e.sh
