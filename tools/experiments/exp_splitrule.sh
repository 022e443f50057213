# split-K count: ceil(296 / tiles) (rule 0) vs one wave of the resident CTA slots (rule 1)
run() { python bench.py --config $2 --steps 10 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$1 $2', d['ms_per_step'])"; }
for r in 0 1; do for c in n16384 n4096; do RELAPACK_SPLITK_RULE=$r run rule$r $c; RELAPACK_SPLITK_RULE=$r run rule$r $c; done; done
RELAPACK_SPLITK_RULE=1 python -m pytest tests/test_gpu_parity.py -q -x -k "recursion or crossover" 2>&1 | tail -1
