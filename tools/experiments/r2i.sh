# r2i: FTZ pivot semantics (round-1 base kernels), same-box A/B vs the round-1 tree at n=4096 / 16384 / batch, REBASE on/off
./abtest/base_kernels_cur > gpurun_out/r2i_bk_cur.txt 2>&1
python tools/ab_trees.py . abtest/r1tree n4096 3 > gpurun_out/r2i_ab.log 2>&1
python tools/ab_trees.py . abtest/r1tree n16384 2 >> gpurun_out/r2i_ab.log 2>&1
python tools/ab_trees.py . abtest/r1tree batch 2 >> gpurun_out/r2i_ab.log 2>&1
for v in 0 1 0 1; do echo "REBASE=$v n4096 $(RELAPACK_REBASE=$v python bench.py --config n4096 --steps 20 --warmup 3 --no-profile --e2e-steps 0 --no-cpu-baseline | python -c 'import json,sys; print(json.loads(sys.stdin.read().strip().splitlines()[-1])["ms_per_step"])')" >> gpurun_out/r2i_ab.log; done
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "subnormal or scaled or batched or reuse" > gpurun_out/r2i_tests.log 2>&1
