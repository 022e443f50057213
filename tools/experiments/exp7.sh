B="python bench.py --no-cpu-baseline --e2e-steps 0 --no-profile"
./tools/microbench/base_kernels | grep "trsm_fused"
for tb in 256 128; do for cfg in n4096 n16384; do
  RELAPACK_TRSM_BASE=$tb $B --config $cfg | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('tb=$tb $cfg', d['ms_per_step'], d['value'])"
done; done
