# e2e: host copies on two copy streams (events) vs memcpy nodes inside the graph
for sc in 1; do for cfg in n16384 n4096 n65536; do
  st=5; [ $cfg = n65536 ] && st=3
  RELAPACK_SPLIT_COPIES=$sc python bench.py --config $cfg --no-cpu-baseline --no-profile --steps $st --e2e-steps 2 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('split_copies=$sc $cfg', d['ms_per_step'], d['e2e']['ms_per_step'], d['e2e']['value'])"
done; done
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "host_matrix" 2>&1 | tail -1
RELAPACK_SPLIT_COPIES=0 timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "host_matrix" 2>&1 | tail -1
