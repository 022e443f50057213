# r7a: potrs right-hand-side panels (RELAPACK_POTRS_COLS) and trtri / lauum row panels (RELAPACK_TRI_ROWS):
# independent chains for the DAG to overlap.  Same box, 2 reps.
mkdir -p gpurun_out
O=gpurun_out/exp_panels_r02i.txt; : > $O
RELAPACK_POTRS_COLS=256 RELAPACK_TRI_ROWS=1024 python -m pytest tests/test_gpu_next.py -x -q 2>&1 | tail -2 >> $O
for rep in 1 2; do
  for c in 0 128 256 512; do
    RELAPACK_POTRS_COLS=$c python bench.py --config potrs --steps 5 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('potrs cols=$c', d['ms_per_step'])" >> $O
  done
  for r in 0 512 1024 2048; do
    for cfg in trtri lauum; do
      RELAPACK_TRI_ROWS=$r python bench.py --config $cfg --steps 5 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('$cfg rows=$r', d['ms_per_step'])" >> $O
    done
  done
done
cat $O
