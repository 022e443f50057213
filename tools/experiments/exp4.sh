B="python bench.py --no-cpu-baseline --e2e-steps 0 --no-profile"
for nw in 8 4; do
  RELAPACK_TRSM_NW=$nw ./tools/microbench/base_kernels | grep trsm_fused | sed "s/^/nw=$nw /"
  for c in n4096 n16384; do
    RELAPACK_TRSM_NW=$nw $B --config $c | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('nw=$nw $c', d['ms_per_step'], d['value'])"
  done
done
