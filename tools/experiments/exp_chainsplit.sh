# split-K granularity for the chain's non-deferred SYRKs (RELAPACK_SPLITK_CHAIN_KT), same box
run() { python bench.py --config $2 --steps 20 --warmup 3 --no-profile --e2e-steps 0 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$1 $2', d['ms_per_step'])"; }
for r in 1 2; do for k in 0 2 4; do RELAPACK_SPLITK_CHAIN_KT=$k run chainkt$k n4096; done; done
for k in 0 2 4; do RELAPACK_SPLITK_CHAIN_KT=$k run chainkt$k n16384; done
RELAPACK_SPLITK_CHAIN_KT=2 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -1
