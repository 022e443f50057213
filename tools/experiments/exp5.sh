B="python bench.py --no-cpu-baseline --e2e-steps 0 --no-profile"
for pv in smem reg; do
  RELAPACK_POTF2=$pv ./tools/microbench/base_kernels | grep "potf2 n=" | sed "s/^/$pv /"
done
for pv in smem reg; do for c in 64 48 32; do for cfg in n4096 n16384; do
  RELAPACK_POTF2=$pv RELAPACK_CROSSOVER=$c $B --config $cfg | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$pv c=$c $cfg', d['ms_per_step'], d['value'])"
done; done; done
