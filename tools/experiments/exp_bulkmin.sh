# deferred-update CTA cap only above a size threshold (RELAPACK_BULK_MIN_GF)
run() { python bench.py --config $2 --steps 10 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$1 $2', d['ms_per_step'])"; }
for r in 1 2; do for g in 0 4 16 64 100000; do RELAPACK_BULK_MIN_GF=$g run min$g n4096; RELAPACK_BULK_MIN_GF=$g run min$g n16384; done; done
