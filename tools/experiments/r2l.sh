# r2l: update kernel with a compile-time global-descriptor variant (fence before griddepcontrol.wait) vs REBASE=0 vs round 1
b() { python bench.py --config $1 --steps 20 --warmup 3 --no-profile --e2e-steps 0 --no-cpu-baseline | python -c 'import json,sys; print(json.loads(sys.stdin.read().strip().splitlines()[-1])["ms_per_step"])'; }
for r in 1 2; do
  for cfg in n4096 n16384; do
    echo "cur $cfg $(b $cfg)"; echo "cur-REBASE0 $cfg $(RELAPACK_REBASE=0 b $cfg)"; echo "r1 $cfg $(cd abtest/r1tree && b $cfg)"
  done
done > gpurun_out/r2l.log 2>&1
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py -q -x > gpurun_out/r2l_tests.log 2>&1
