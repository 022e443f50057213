# r3u: session refresh (round 2, second session): full GPU suite, smoke, bench lines, reference arm,
# ncu launch list of the default step, traces, ncu DRAM of the batched classes, the §8(f) bench lines
TAG=r02b bash tools/experiments/refresh.sh
O=gpurun_out
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:k_batched_cls -c 4 --csv --log-file $O/r02b_ncu_batch.csv python bench.py --config batch --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0 --no-profile > /dev/null 2>&1
for op in trtri lauum potri potrs getrf; do python bench.py --config $op --steps 3 --warmup 1 2>/dev/null | tail -1 >> $O/r02b_bench_next.jsonl; done
