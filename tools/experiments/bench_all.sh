# every bench line of the round (one box), the reference arm, the dist executor at world size 1,
# and the ncu launch list of the default bench command
TAG=${1:-r02f}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu_${TAG}.txt
for cfg in n16384 n4096 n256 n65536 batch; do
  python bench.py --config $cfg > gpurun_out/bench_${cfg}_${TAG}.json 2>gpurun_out/bench_${cfg}_${TAG}.err
done
for cfg in trtri trtri_blocked potrf_blocked lauum potri potrs getrf; do
  python bench.py --config $cfg >> gpurun_out/bench_next_${TAG}.jsonl 2>>gpurun_out/bench_next_${TAG}.err
done
python bench.py --impl reference > gpurun_out/bench_reference_${TAG}.json 2>gpurun_out/bench_reference_${TAG}.err
python bench.py --dist > gpurun_out/bench_dist_world1_n16384_${TAG}.json 2>gpurun_out/bench_dist_${TAG}.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_n16384_${TAG}.csv \
    python bench.py --steps 2 --warmup 1 > gpurun_out/ncu_bench_${TAG}.log 2>&1
python tools/launches.py gpurun_out/launches_n16384_${TAG}.csv > gpurun_out/ncu_launches_n16384_${TAG}.txt
