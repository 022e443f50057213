# 128-node copies for uplo U as 8x8 patches with 16-byte global accesses
cd tools/microbench; ./base_kernels 2>&1 | grep -E "potf2 n=128 layout"; cd ../..
python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -1
run() { python bench.py --config $2 --steps 10 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$1 $2', d['ms_per_step'])"; }
for r in 1 2; do for p in 0 1; do RELAPACK_COPY_PAIRS=$p run pairs$p n16384; done; done
RELAPACK_TRACE=1 python tools/trace_timeline.py 16384 U 2>&1 | head -3
