# r4d: epoch-stamped getrf exchange with strong 128-bit accesses: panel probe, getrf tests, bench
bash tools/experiments/r4b.sh
timeout 300 python -m pytest tests/test_gpu_next.py -q -m gpu -x -k "getrf" > gpurun_out/r4d_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/r4d_tests.txt
for v in 0 1; do RELAPACK_GETF2_POLL=$v timeout 300 python bench.py --config getrf --steps 3 --warmup 1 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('poll=$v', d['ms_per_step'], d.get('pct_fp64_peak'), d['kernel_share'])" >> gpurun_out/r4d_bench.txt; done
