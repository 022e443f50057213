# r7b: the panel-split variant tests, getrf / lauum with TRSM row panels, the update-traffic capture and
# the round's final bench set (TAG r02i) from one box.
mkdir -p gpurun_out
O=gpurun_out/exp_panels2_r02i.txt; : > $O
python -m pytest tests/test_gpu_next.py -x -q -k "panel_split or potrs" 2>&1 | tail -2 >> $O
for r in 0 2048 4096; do
  for cfg in getrf lauum; do
    RELAPACK_TRI_ROWS=$r python bench.py --config $cfg --steps 5 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('$cfg rows=$r', d['ms_per_step'])" >> $O
  done
done
for x in 64 128; do
  RELAPACK_XBASE=$x python bench.py --config potrs --steps 5 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('potrs xbase=$x', d['ms_per_step'])" >> $O
done
cat $O
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:k_update --csv --log-file gpurun_out/t_r02i.csv python tools/ncu_step.py 16384 U > gpurun_out/ncu_traffic_r02i.log 2>&1
python tools/update_traffic.py gpurun_out/t_r02i.csv 16384 gpurun_out/ncu_update_traffic_n16384_r02i.json > /dev/null 2>gpurun_out/traffic_r02i.err
rm -f gpurun_out/t_r02i.csv
bash tools/experiments/bench_all.sh r02i
rm -f gpurun_out/launches_n16384_r02i.csv
