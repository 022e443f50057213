# r4e: node-128 base case alone on its SM (RELAPACK_NODE_EXCLUSIVE: 220 KB shared memory requested) + getrf poll variant test
timeout 900 python -m pytest tests/test_gpu_next.py -q -m gpu -x -k "variants" > gpurun_out/r4e_tests.txt 2>&1
for rep in 1 2; do for v in 0 1; do for c in n4096 n256 n16384; do RELAPACK_NODE_EXCLUSIVE=$v python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-profile --e2e-steps 0 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('excl=$v $c', d['ms_per_step'])" >> gpurun_out/r4e_bench.txt; done; done; done
