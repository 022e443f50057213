# programmatic dependent launch on the plan DAG's kernel edges (RELAPACK_PDL=mode)
RELAPACK_PDL=2 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -1
run() { python bench.py --config $2 --steps 20 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$1 $2', d['ms_per_step'], min(d['step_times_ms']), max(d['step_times_ms']))"; }
for r in 1 2 3; do for m in 0 1 2 3; do RELAPACK_PDL=$m run pdl$m n4096; done; done
for m in 0 2 3; do RELAPACK_PDL=$m run pdl$m n16384; done
