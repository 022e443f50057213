# TRSM base width with the register-slab kernel
for b in 64 128; do for c in n16384 n4096; do for rep in 1 2; do RELAPACK_TRSM_BASE=$b python bench.py --config $c --steps 10 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('trsm_base $b $c', d['ms_per_step'])"; done; done; done
