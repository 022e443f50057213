# deferred-update CTA cap re-sweep (RELAPACK_BULK_CTAS) after the TRSM / PDL changes
run() { python bench.py --config $2 --steps 10 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$1 $2', d['ms_per_step'])"; }
for b in 108 120 132 140 148 0; do RELAPACK_BULK_CTAS=$b run bulk$b n16384; RELAPACK_BULK_CTAS=$b run bulk$b n4096; done
