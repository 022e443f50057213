# host-matrix path: TRSM GEMMs in column chunks (RELAPACK_HOST_GEMM_COLS)
python tools/e2e_probe.py 16384 U
for c in 512 1024 2048; do RELAPACK_HOST_GEMM_COLS=$c python tools/e2e_probe.py 16384 U; done
RELAPACK_HOST_GEMM_COLS=1024 RELAPACK_TRACE=1 python tools/e2e_probe.py 16384 U
python tools/e2e_probe.py 4096 L
RELAPACK_HOST_GEMM_COLS=1024 python tools/e2e_probe.py 4096 L
