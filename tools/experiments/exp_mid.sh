# mid-size update tiling at n=16384 (register-slab TRSM era)
run() { python bench.py --config n16384 --steps 10 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$1', d['ms_per_step'])"; }
run default; run default
RELAPACK_SPLIT128=1 run split128; RELAPACK_SPLIT128=1 run split128
RELAPACK_SPLITK_MID=1 run splitk_mid
RELAPACK_TILE32_BELOW=0 run tile32_off
RELAPACK_TILE32_BELOW=64 run tile32_below64
