for th in 32 300; do RELAPACK_TILE32_BELOW=$th ./tools/microbench/update_small | grep "(auto)" | sed "s/^/th=$th /"; done
B="python bench.py --no-cpu-baseline --e2e-steps 0 --no-profile"
for th in 32 150 300; do for cfg in n4096 n16384; do
  RELAPACK_TILE32_BELOW=$th $B --config $cfg | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('tile32_below=$th $cfg', d['ms_per_step'], d['value'])"
done; done
