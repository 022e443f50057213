# TRSM register kernel: L blocks staged by bulk copies (lines of 512 B; column-major for uplo L)
cd tools/microbench; ./base_kernels 2>&1 | grep -E "trsm_reg|trsm_fused m=(2048|8192) t=(64|128)"; cd ../..
python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -1
run() { python bench.py --config $2 --steps 10 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$1 $2', d['ms_per_step'])"; }
for r in 1 2; do for b in 0 1; do RELAPACK_TRSM_BULKL=$b run bulkl$b n4096; RELAPACK_TRSM_BULKL=$b run bulkl$b n16384; done; done
