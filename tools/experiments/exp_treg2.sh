# register-slab TRSM with a 1-chunk instance for t <= 64
cd tools/microbench && ./base_kernels 2>&1 | grep trsm_fused; cd ../..
python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -2
for c in n16384 n4096; do for rep in 1 2; do python bench.py --config $c --steps 10 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$c', d['ms_per_step'])"; done; done
