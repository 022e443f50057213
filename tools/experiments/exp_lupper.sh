# TRSM register kernel: diagonal L blocks staged without their upper halves (masked loads)
cd tools/microbench; ./base_kernels 2>&1 | grep -E "trsm_reg|trsm_fused m=(2048|8192) t=(64|128)"; cd ../..
python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -1
run() { python bench.py --config $1 --steps 10 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$1', d['ms_per_step'])"; }
for r in 1 2; do run n4096; run n16384; done
