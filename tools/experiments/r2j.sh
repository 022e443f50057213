# r2j: §8(f) rows measured with the bench harness (n = 16384; potrs nrhs 1024), blocked-vs-recursive sweep,
# ncu DRAM bytes of the batched kernels, the 128-node base case and the n = 256 factorization
set -x
for c in trtri lauum potri potrs getrf potrf_blocked trtri_blocked; do
  extra=""
  [ "$c" = "trtri_blocked" ] && extra="--n 4096 --block 128"
  [ "$c" = "potrf_blocked" ] && extra="--block 256"
  timeout 900 python bench.py --config $c $extra --steps 3 --warmup 2 > gpurun_out/r2j_next_$c.json 2> gpurun_out/r2j_next_$c.err
done
for r in 32 128 256 512; do echo "GETF2_ROWS=$r $(RELAPACK_GETF2_ROWS=$r timeout 600 python bench.py --config getrf --steps 3 --warmup 1 --no-profile --no-cpu-baseline | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d["ms_per_step"], d["value"])')" >> gpurun_out/r2j_getf2_rows.txt; done
timeout 900 python tools/sweep_blocked.py 4096 16384 > gpurun_out/r2j_sweep_blocked.txt 2>&1
NCU="ncu --clock-control none --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__warps_active.avg.pct_of_peak_sustained_active,dram__throughput.avg.pct_of_peak_sustained_elapsed --csv"
timeout 600 $NCU -k regex:k_batched_cls python bench.py --config batch --steps 1 --warmup 0 --no-profile --e2e-steps 0 --no-cpu-baseline > gpurun_out/r2j_ncu_batch.csv 2>&1
timeout 600 $NCU -k regex:k_potf2 -c 40 python bench.py --config n4096 --steps 1 --warmup 0 --no-profile --e2e-steps 0 --no-cpu-baseline > gpurun_out/r2j_ncu_potf2.csv 2>&1
timeout 600 $NCU python bench.py --config n256 --steps 1 --warmup 0 --no-profile --e2e-steps 0 --no-cpu-baseline > gpurun_out/r2j_ncu_n256.csv 2>&1
b() { python bench.py --config $1 --steps 20 --warmup 3 --no-profile --e2e-steps 0 --no-cpu-baseline | python -c 'import json,sys; print(json.loads(sys.stdin.read().strip().splitlines()[-1])["ms_per_step"])'; }
for cfg in n4096 n16384 n4096 n16384; do echo "cur $cfg $(b $cfg)"; echo "r1 $cfg $(cd abtest/r1tree && b $cfg)"; done > gpurun_out/r2j_ab.log 2>&1
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_next.py -q -x > gpurun_out/r2j_tests.log 2>&1
