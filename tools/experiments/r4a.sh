# r4a: getrf panels with the epoch-stamped exchange (RELAPACK_GETF2_POLL) vs the grid barrier
timeout 300 python -m pytest tests/test_gpu_next.py -q -m gpu -x -k "getrf and not variants" > gpurun_out/r4a_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/r4a_tests.txt
if grep -q "rc=0" gpurun_out/r4a_tests.txt; then
timeout 600 python -m pytest tests/test_gpu_next.py -q -m gpu -x > gpurun_out/r4a_tests_all.txt 2>&1
for v in 0 1; do RELAPACK_GETF2_POLL=$v timeout 300 python bench.py --config getrf --steps 3 --warmup 1 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('poll=$v', d['ms_per_step'], d.get('pct_fp64_peak'), d['kernel_share'])" >> gpurun_out/r4a_bench.txt; done
fi
