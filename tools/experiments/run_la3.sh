B="timeout 300 python bench.py --config getrf --no-cpu-baseline --no-profile --steps 3 --warmup 3"
echo chain-alone; RELAPACK_GETRF_LA=1 RELAPACK_GETRF_SKIP_DEFER=1 $B 2>&1 | tail -1 | cut -c100-200
echo chain-alone-w512; RELAPACK_GETRF_LA=1 RELAPACK_GETRF_WINDOW=512 RELAPACK_GETRF_SKIP_DEFER=1 $B 2>&1 | tail -1 | cut -c100-200
echo reserve64; RELAPACK_GETRF_LA=1 RELAPACK_GETRF_RESERVE=64 $B 2>&1 | tail -1 | cut -c100-200
echo reserve100; RELAPACK_GETRF_LA=1 RELAPACK_GETRF_RESERVE=100 $B 2>&1 | tail -1 | cut -c100-200
