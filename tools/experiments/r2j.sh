# r2j: §8(f) rows measured with the bench harness (n = 16384; potrs nrhs 1024), blocked-vs-recursive sweep,
# ncu DRAM bytes of the batched kernels, the 128-node base case and the n = 256 factorization
set -x
for c in trtri lauum potri potrs getrf potrf_blocked trtri_blocked; do
  extra=""
  [ "$c" = "trtri_blocked" ] && extra="--n 4096 --block 128"
  [ "$c" = "potrf_blocked" ] && extra="--block 256"
  timeout 900 python bench.py --config $c $extra --steps 3 --warmup 2 > gpurun_out/r2j_next_$c.json 2> gpurun_out/r2j_next_$c.err
done
timeout 900 python tools/sweep_blocked.py 4096 16384 > gpurun_out/r2j_sweep_blocked.txt 2>&1
NCU="ncu --clock-control none --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__warps_active.avg.pct_of_peak_sustained_active,dram__throughput.avg.pct_of_peak_sustained_elapsed --csv"
timeout 600 $NCU -k regex:k_batched_cls python bench.py --config batch --steps 1 --warmup 0 --no-profile --e2e-steps 0 --no-cpu-baseline > gpurun_out/r2j_ncu_batch.csv 2>&1
timeout 600 $NCU -k regex:k_potf2 -c 40 python bench.py --config n4096 --steps 1 --warmup 0 --no-profile --e2e-steps 0 --no-cpu-baseline > gpurun_out/r2j_ncu_potf2.csv 2>&1
timeout 600 $NCU python bench.py --config n256 --steps 1 --warmup 0 --no-profile --e2e-steps 0 --no-cpu-baseline > gpurun_out/r2j_ncu_n256.csv 2>&1
