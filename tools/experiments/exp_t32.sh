# 32-tiles for short-K updates with few 32-tiles (RELAPACK_TILE32_MAX_TILES / _MAX_K)
run() { python bench.py --config $2 --steps 20 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$1 $2', d['ms_per_step'])"; }
for r in 1 2; do
  RELAPACK_TILE32_MAX_TILES=0 run t32off n4096
  RELAPACK_TILE32_MAX_TILES=296 run t32_296 n4096
  RELAPACK_TILE32_MAX_TILES=592 run t32_592 n4096
  RELAPACK_TILE32_MAX_TILES=592 RELAPACK_TILE32_MAX_K=512 run t32_592k512 n4096
done
RELAPACK_TILE32_MAX_TILES=0 run t32off n16384
RELAPACK_TILE32_MAX_TILES=296 run t32_296 n16384
RELAPACK_TILE32_MAX_TILES=592 run t32_592 n16384
RELAPACK_TILE32_MAX_TILES=592 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -1
