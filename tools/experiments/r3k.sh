# r3k: ncu source-level capture of the four batched class kernels (one CFG[4] step)
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_batched_cls -c 4 -o gpurun_out/r3k_batch python bench.py --config batch --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0 --no-profile > gpurun_out/r3k_ncu.log 2>&1
python bench.py --config batch --no-cpu-baseline > gpurun_out/r3k_bench.json 2>/dev/null
