set -x
B="python bench.py --no-cpu-baseline --e2e-steps 0 --no-profile"
for c in 64 96 128; do
  RELAPACK_CROSSOVER=$c $B --config n4096 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c=$c n4096', d['ms_per_step'], d['value'])"
  RELAPACK_CROSSOVER=$c $B --config n16384 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c=$c n16384', d['ms_per_step'], d['value'])"
done
python tools/profile_plan.py 16384 U > gpurun_out/pp16k.txt 2>&1
$B --config n65536 --steps 3 > gpurun_out/b65k.json 2> gpurun_out/b65k.err
