# r3j: batched descriptor loads one matrix ahead (RELAPACK_BATCH_DESC_AHEAD); 16-class occupancy (MINB16)
cd tools/microbench
i=0
for d in "-DRELAPACK_BATCH_DESC_AHEAD=0" "" "-DRELAPACK_BATCH_MINB16=6" "-DRELAPACK_BATCH_MINB16=4"; do
  i=$((i+1)); nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -I ../../include $d -o /tmp/bprobe$i batched_probe.cu
  /tmp/bprobe$i | sed "s/^/[$d] /" >> ../../gpurun_out/r3j_probe.txt
  /tmp/bprobe$i | sed "s/^/[$d] /" >> ../../gpurun_out/r3j_probe.txt
done
