B="timeout 300 python bench.py --config getrf --no-cpu-baseline --no-profile --steps 3 --warmup 3"
echo nocap-serial; RELAPACK_GETRF_LA=1 RELAPACK_GETRF_RESERVE=-1 $B 2>&1 | tail -1 | cut -c100-200
echo nocap-parallel; RELAPACK_GETRF_LA=1 RELAPACK_GETRF_RESERVE=-1 RELAPACK_GETRF_SERIAL=0 $B 2>&1 | tail -1 | cut -c100-200
echo nocap-serial-w512; RELAPACK_GETRF_LA=1 RELAPACK_GETRF_RESERVE=-1 RELAPACK_GETRF_WINDOW=512 $B 2>&1 | tail -1 | cut -c100-200
echo reserve8; RELAPACK_GETRF_LA=1 RELAPACK_GETRF_RESERVE=8 RELAPACK_GETF2_CLUSTER=8 $B 2>&1 | tail -1 | cut -c100-200
