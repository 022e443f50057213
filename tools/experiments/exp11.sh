# e2e (pinned host matrix, copies inside the DAG) with compute kernels replaced by empty ones
for m in 0 15; do
  RELAPACK_DEBUG_SKIP=$m python bench.py --config n16384 --no-cpu-baseline --no-profile --steps 3 --e2e-steps 3 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('skip=$m', d['ms_per_step'], d['e2e']['ms_per_step'])"
done
