B="python bench.py --no-cpu-baseline --e2e-steps 0 --no-profile"
./tools/microbench/base_kernels | grep "potf2 n=" 
for nd in 0 1; do for c in 64 128; do for cfg in n4096 n16384; do
  RELAPACK_NODE128=$nd RELAPACK_CROSSOVER=$c $B --config $cfg | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('node128=$nd c=$c $cfg', d['ms_per_step'], d['value'])"
done; done; done
