# r7c: trtri with the level's solve first (RELAPACK_TRTRI_ORDER=1: both recursive calls independent in the DAG),
# alone and with row panels on the TRSM / TRMM operands.  Same box.
mkdir -p gpurun_out
O=gpurun_out/exp_trtri_order_r02i.txt; : > $O
python -m pytest tests/test_gpu_next.py -x -q -k "solve_first" 2>&1 | tail -2 >> $O
run() {  # cfg order rows
  RELAPACK_TRTRI_ORDER=$2 RELAPACK_TRI_ROWS=$3 python bench.py --config $1 --steps 5 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('$1 order=$2 rows=$3', d['ms_per_step'])" >> $O
}
run trtri 0 0; run trtri 1 0; run trtri 1 2048; run trtri 1 1024; run trtri 1 4096
run potri 0 0; run potri 1 0
run trtri 0 0; run trtri 1 0
cat $O
