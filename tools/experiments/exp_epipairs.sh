# update-kernel epilogue with 16-byte global accesses (RELAPACK_EPI_PAIRS), same-box A/B
python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -1
RELAPACK_EPI_PAIRS=0 python -m pytest tests/test_gpu_parity.py -q -x -k "recursion" 2>&1 | tail -1
run() { python bench.py --config $2 --steps 20 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$1 $2', d['ms_per_step'])"; }
for r in 1 2; do for p in 0 1; do RELAPACK_EPI_PAIRS=$p run epi$p n4096; RELAPACK_EPI_PAIRS=$p run epi$p n16384; done; done
