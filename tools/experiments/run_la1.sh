set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests/test_gpu_next.py -q -x -k "getrf" 2>&1 | tail -15
for la in 0 1; do
  RELAPACK_GETRF_LA=$la timeout 300 python bench.py --config getrf --no-cpu-baseline --no-profile --steps 3 --warmup 3 2>&1 | tail -1 | cut -c1-400
done
for w in 128 512; do
  RELAPACK_GETRF_LA=1 RELAPACK_GETRF_WINDOW=$w timeout 300 python bench.py --config getrf --no-cpu-baseline --no-profile --steps 3 --warmup 3 2>&1 | tail -1 | cut -c1-300
done
RELAPACK_GETRF_LA=1 RELAPACK_GETRF_SERIAL=0 timeout 300 python bench.py --config getrf --no-cpu-baseline --no-profile --steps 3 --warmup 3 2>&1 | tail -1 | cut -c1-300
RELAPACK_GETRF_LA=1 RELAPACK_GETRF_RESERVE=32 timeout 300 python bench.py --config getrf --no-cpu-baseline --no-profile --steps 3 --warmup 3 2>&1 | tail -1 | cut -c1-300
