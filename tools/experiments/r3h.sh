# r3h: batched classes after the spill fix (opaque lane offsets); occupancy variants; team vs warp
cd tools/microbench
i=0
for d in "" "-DRELAPACK_BATCH_MINB32=4" "-DRELAPACK_BATCH_MINB48=4" "-DRELAPACK_BATCH_MINB64=3"; do
  i=$((i+1)); nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -I ../../include $d -o /tmp/bprobe$i batched_probe.cu
  for tm in 0 1; do RELAPACK_BATCH_TEAM=$tm /tmp/bprobe$i | sed "s/^/[$d] team=$tm /" >> ../../gpurun_out/r3h_probe.txt; done
done
