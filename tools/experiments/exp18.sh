# e2e vs host copy block shape
for pr in "512 2048" "1024 4096" "2048 8192" "256 1024" "512 16384"; do set -- $pr
  RELAPACK_COPY_PANEL=$1 RELAPACK_COPY_ROWS=$2 python bench.py --config n16384 --no-cpu-baseline --no-profile --steps 3 --e2e-steps 3 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('panel=$1 rows=$2', d['e2e']['ms_per_step'])"
done
