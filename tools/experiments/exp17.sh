B="python bench.py --no-cpu-baseline --e2e-steps 0 --no-profile"
for cap in 0 144 140 136 128; do for cfg in n16384 n4096; do
  RELAPACK_UPD_CTAS=$cap $B --config $cfg | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('upd_cap=$cap $cfg', d['ms_per_step'], d['value'])"
done; done
RELAPACK_UPD_CTAS=140 RELAPACK_TRACE=1 python tools/trace_timeline.py 16384 U > gpurun_out/trace16k_cap140.txt 2>&1
