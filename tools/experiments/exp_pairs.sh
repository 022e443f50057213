# 128-node copies as 16-byte pairs for uplo L (RELAPACK_COPY_PAIRS), same box A/B
python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -1
run() { python bench.py --config $2 --steps 20 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$1 $2', d['ms_per_step'])"; }
for r in 1 2 3; do for p in 0 1; do RELAPACK_COPY_PAIRS=$p run pairs$p n4096; done; done
for p in 0 1; do RELAPACK_COPY_PAIRS=$p run pairs$p n65536; done
