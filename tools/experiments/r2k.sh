# r2k: cost of the pointer-independent graphs: acquire fence (unsafe no-fence build), REBASE=0, round-1 tree
b() { python bench.py --config $1 --steps 20 --warmup 3 --no-profile --e2e-steps 0 --no-cpu-baseline | python -c 'import json,sys; print(json.loads(sys.stdin.read().strip().splitlines()[-1])["ms_per_step"])'; }
for r in 1 2; do
  for cfg in n4096 n16384; do
    echo "cur $cfg $(b $cfg)"; echo "cur-REBASE0 $cfg $(RELAPACK_REBASE=0 b $cfg)"
    echo "noacq $cfg $(cd abtest/noacq && b $cfg)"; echo "r1 $cfg $(cd abtest/r1tree && b $cfg)"
  done
done > gpurun_out/r2k.log 2>&1
