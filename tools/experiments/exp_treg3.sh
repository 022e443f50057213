# register TRSM CTA size after the masked-load change (same box)
run() { python bench.py --config $2 --steps 20 --warmup 3 --no-profile --e2e-steps 0 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$1 $2', d['ms_per_step'])"; }
for r in 1 2; do
  for f in 1024 2048 4096 100000; do RELAPACK_TRSM_REG8_FROM=$f run reg8from$f n4096; done
  RELAPACK_TRSM_REG=2 run rg2 n4096
done
for f in 1024 2048 4096; do RELAPACK_TRSM_REG8_FROM=$f run reg8from$f n16384; done
