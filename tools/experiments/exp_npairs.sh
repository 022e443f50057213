# TRSM register kernel, uplo L: slab loads/stores as 16-byte pairs via a lane^4 exchange (RELAPACK_TRSM_NPAIRS)
cd tools/microbench; for b in base_kernels_old base_kernels base_kernels_old base_kernels; do echo == $b; ./$b 2>&1 | grep -E "trsm_reg|trsm_fused m=(64|2048|8192|16384) t=(64|128) layout N"; done; rm -f base_kernels_old; cd ../..
python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -1
run() { python bench.py --config $1 --steps 20 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$1', d['ms_per_step'])"; }
for r in 1 2 3; do run n4096; done
