# round end: the §8(f) GPU tests with the trtri solve-first default, the trtri / potri / trtri_blocked lines, the stdout check
mkdir -p gpurun_out
python -m pytest tests/test_gpu_next.py -x -q > gpurun_out/pytest_gpu_next_r02j.txt 2>&1; tail -2 gpurun_out/pytest_gpu_next_r02j.txt
for cfg in trtri potri trtri_blocked; do python bench.py --config $cfg >> gpurun_out/bench_next_r02j.jsonl 2>/dev/null; done
python bench.py --dist --steps 3 --warmup 3 > gpurun_out/bench_dist_stdout_r02j.txt 2>/dev/null; wc -l gpurun_out/bench_dist_stdout_r02j.txt
python bench.py --config n4096 > gpurun_out/bench_n4096_r02j.json 2>/dev/null; wc -l gpurun_out/bench_n4096_r02j.json
python -c "
import json
for l in open('gpurun_out/bench_next_r02j.jsonl'):
    j=json.loads(l); print(j['config']['workload'][:40], j['ms_per_step'], j.get('pct_fp64_peak'))"
