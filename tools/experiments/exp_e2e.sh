# host-matrix path at n=16384: copy block granularity and the kernel timeline
python tools/e2e_probe.py 16384 U
RELAPACK_TRACE=1 python tools/e2e_probe.py 16384 U
for p in 256 1024; do RELAPACK_COPY_PANEL=$p python tools/e2e_probe.py 16384 U; done
for r in 1024 4096; do RELAPACK_COPY_ROWS=$r python tools/e2e_probe.py 16384 U; done
RELAPACK_DEFER_LOW=0 python tools/e2e_probe.py 16384 U
