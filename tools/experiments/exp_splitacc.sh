# TRSM register kernel: split accumulators for the next sub-block's tile
cd tools/microbench
for b in base_kernels_nosplit base_kernels; do echo "== $b"; ./$b 2>&1 | grep -E "trsm_fused m=(64|2048|8192|16384) t=(64|128)|trsm_reg"; done
cd ../..
python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -2
for c in n16384 n4096; do for rep in 1 2; do python bench.py --config $c --steps 10 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$c', d['ms_per_step'])"; done; done
