# r2o: blocked (8-column) triangular rows kernel; getf2 rows sweep; dist world 1 with larger row blocks
timeout 900 python -m pytest tests/test_gpu_next.py -q -x > gpurun_out/r2o_tests.log 2>&1
for c in trtri lauum potri potrs getrf; do
  timeout 900 python bench.py --config $c --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/r2o_next_$c.json 2> gpurun_out/r2o_next_$c.err
done
timeout 600 python tools/trtri_breakdown.py 16384 > gpurun_out/r2o_trtri_breakdown.txt 2>&1
for r in 64 256; do echo "GETF2_ROWS=$r $(RELAPACK_GETF2_ROWS=$r timeout 600 python bench.py --config getrf --steps 3 --warmup 1 --no-profile --no-cpu-baseline | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d["ms_per_step"], d["value"])')" >> gpurun_out/r2o_getf2_rows.txt; done
for nb in 1024 2048; do timeout 600 python tools/dist_world1.py 16384 8192 $nb >> gpurun_out/r2o_dist_world1.txt 2>&1; done
