# r2h: rebased graphs vs per-pointer graphs (RELAPACK_REBASE) at n=16384 / 4096, same box; base-kernel microbench; round-1 tree
./abtest/base_kernels_cur > gpurun_out/r2h_bk_cur.txt 2>&1
for r in 1 2 3; do
  for v in 1 0; do
    echo "REBASE=$v $(RELAPACK_REBASE=$v python bench.py --steps 10 --warmup 3 --no-profile --e2e-steps 0 --no-cpu-baseline | python -c 'import json,sys; print(json.loads(sys.stdin.read().strip().splitlines()[-1])["ms_per_step"])')" >> gpurun_out/r2h_ab16k.log
  done
done
python tools/ab_trees.py . abtest/r1tree n16384 2 > gpurun_out/r2h_ab_r1_16k.log 2>&1
python tools/ab_trees.py . abtest/r1tree n4096 3 > gpurun_out/r2h_ab_r1_4k.log 2>&1
python tools/ab_trees.py . abtest/r1tree batch 2 > gpurun_out/r2h_ab_r1_batch.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "subnormal or scaled or batched or host" > gpurun_out/r2h_tests.log 2>&1
