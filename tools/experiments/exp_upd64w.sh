# 64-tile update config: 4 warps of 32x32 vs 8 warps of 32x16 (compile-time RELAPACK_UPD64_WARPS)
python -m pytest tests/test_gpu_parity.py -q -x -k "recursion or crossover" 2>&1 | tail -1
run() { python bench.py --config $1 --steps 10 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$1', d['ms_per_step'])"; }
for r in 1 2; do run n16384; run n4096; done
python tools/profile_plan.py 16384 U 2>/dev/null | head -24
