# small (< RELAPACK_PRIO_SMALL_GF) TRSM GEMMs one level above the big ones (RELAPACK_PRIO_MODE=8), same box
run() { python bench.py --config $2 --steps 20 --warmup 3 --no-profile --e2e-steps 0 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$1 $2', d['ms_per_step'])"; }
for r in 1 2; do for m in 1 8; do RELAPACK_PRIO_MODE=$m run prio$m n16384; RELAPACK_PRIO_MODE=$m run prio$m n4096; done; done
for g in 1 16; do RELAPACK_PRIO_MODE=8 RELAPACK_PRIO_SMALL_GF=$g run prio8_small$g n16384; RELAPACK_PRIO_MODE=8 RELAPACK_PRIO_SMALL_GF=$g run prio8_small$g n4096; done
