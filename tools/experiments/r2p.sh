# r2p: round-2 validation: full GPU suite, bench lines of every config, the ncu launch list of the bench command
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r2p_smoke.log 2>&1
timeout 2400 python -m pytest tests -q -m gpu --durations=20 > gpurun_out/r2p_tests.log 2>&1
python bench.py > gpurun_out/r2p_b16k.json 2> gpurun_out/r2p_b16k.err
python bench.py --config n4096 --no-cpu-baseline > gpurun_out/r2p_b4k.json 2> gpurun_out/r2p_b4k.err
python bench.py --config n256 --no-cpu-baseline > gpurun_out/r2p_b256.json 2> gpurun_out/r2p_b256.err
python bench.py --config batch --no-cpu-baseline > gpurun_out/r2p_batch.json 2> gpurun_out/r2p_batch.err
python bench.py --config n65536 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/r2p_b65k.json 2> gpurun_out/r2p_b65k.err
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2p_ref.json 2> gpurun_out/r2p_ref.err
python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-profile --e2e-steps 0 > gpurun_out/r2p_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 2500 --csv --log-file gpurun_out/r2p_launches.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-profile --e2e-steps 0 > gpurun_out/r2p_ncu.log 2>&1
