# host-matrix path: TRSM GEMM column chunks x copy panel x B21 chunks
for c in 256 512; do RELAPACK_HOST_GEMM_COLS=$c python tools/e2e_probe.py 16384 U; done
RELAPACK_HOST_GEMM_COLS=512 RELAPACK_COPY_PANEL=256 python tools/e2e_probe.py 16384 U
RELAPACK_HOST_GEMM_COLS=256 RELAPACK_COPY_PANEL=256 python tools/e2e_probe.py 16384 U
for b in 4 8; do RELAPACK_HOST_GEMM_COLS=512 RELAPACK_HOST_B21_CHUNKS=$b python tools/e2e_probe.py 16384 U; done
RELAPACK_HOST_GEMM_COLS=512 RELAPACK_COPY_ROWS=4096 python tools/e2e_probe.py 16384 U
RELAPACK_HOST_GEMM_COLS=512 RELAPACK_TRACE=1 python tools/e2e_probe.py 16384 U
RELAPACK_HOST_GEMM_COLS=512 python tools/e2e_probe.py 65536 L
python tools/e2e_probe.py 65536 L
