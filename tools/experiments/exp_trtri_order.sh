# r7c: trtri with the level's solve first (RELAPACK_TRTRI_ORDER=1: both recursive calls independent in the DAG),
# alone and with row panels on the TRSM / TRMM operands.  Same box, 2 reps.
mkdir -p gpurun_out
O=gpurun_out/exp_trtri_order_r02i.txt; : > $O
python -m pytest tests/test_gpu_next.py -x -q -k "solve_first" 2>&1 | tail -2 >> $O
for rep in 1 2; do
  for v in "0 0" "1 0" "1 1024" "1 2048" "1 4096"; do
    set -- $v
    for cfg in trtri potri; do
      RELAPACK_TRTRI_ORDER=$1 RELAPACK_TRI_ROWS=$2 python bench.py --config $cfg --steps 5 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('$cfg order=$1 rows=$2', d['ms_per_step'])" >> $O
    done
  done
done
cat $O
