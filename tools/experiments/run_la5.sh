B="timeout 300 python bench.py --config getrf --no-cpu-baseline --no-profile --steps 3 --warmup 3"
echo base; RELAPACK_GETRF_LA=0 $B 2>&1 | tail -1 | cut -c100-200
echo la; RELAPACK_GETRF_LA=1 $B 2>&1 | tail -1 | cut -c100-200
echo p0first; RELAPACK_GETRF_LA=1 RELAPACK_GETRF_P0FIRST=1 $B 2>&1 | tail -1 | cut -c100-200
echo p0first-w512; RELAPACK_GETRF_LA=1 RELAPACK_GETRF_P0FIRST=1 RELAPACK_GETRF_WINDOW=512 $B 2>&1 | tail -1 | cut -c100-200
echo p0first-nocap; RELAPACK_GETRF_LA=1 RELAPACK_GETRF_P0FIRST=1 RELAPACK_GETRF_RESERVE=-1 $B 2>&1 | tail -1 | cut -c100-200
