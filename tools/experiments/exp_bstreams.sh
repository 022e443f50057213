# batched size classes on forked streams (RELAPACK_BATCH_STREAMS)
python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x -k batch 2>&1 | tail -1
for r in 1 2 3; do for b in 0 1; do RELAPACK_BATCH_STREAMS=$b python bench.py --config batch 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('streams$b', d['ms_per_step'], d['e2e']['ms_per_step'])"; done; done
