# graph node priority classes (RELAPACK_PRIO_MODE), same box
python -c "import torch; print(torch.cuda.Stream.priority_range())"
run() { python bench.py --config $2 --steps 20 --warmup 3 --no-profile --e2e-steps 0 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$1 $2', d['ms_per_step'])"; }
for r in 1 2; do for m in 0 1 3; do RELAPACK_PRIO_MODE=$m run prio$m n16384; RELAPACK_PRIO_MODE=$m run prio$m n4096; done; done
