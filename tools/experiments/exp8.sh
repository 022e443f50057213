B="python bench.py --no-cpu-baseline --e2e-steps 0 --no-profile"
for nw in 8 4; do for tb in 128 64; do for cfg in n4096 n16384; do
  RELAPACK_TRSM_NW=$nw RELAPACK_TRSM_BASE=$tb $B --config $cfg | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('nw=$nw tb=$tb $cfg', d['ms_per_step'], d['value'])"
done; done; done
