# e2e with host copies as SM kernels vs memcpy nodes
for ck in 1 0; do for cfg in n16384 n4096; do
  RELAPACK_COPY_KERNEL=$ck python bench.py --config $cfg --no-cpu-baseline --no-profile --steps 3 --e2e-steps 3 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('copy_kernel=$ck $cfg', d['ms_per_step'], d['e2e']['ms_per_step'], d['e2e']['value'])"
done; done
RELAPACK_COPY_KERNEL=1 RELAPACK_DEBUG_SKIP=15 python bench.py --config n16384 --no-cpu-baseline --no-profile --steps 3 --e2e-steps 3 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('copies alone (kernels)', d['e2e']['ms_per_step'])"
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k host_matrix 2>&1 | tail -1
