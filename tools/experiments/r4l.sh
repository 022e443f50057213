# r4l: compute-sanitizer memcheck / racecheck / synccheck on a small workload of every kernel family
export RELAPACK_GRAPH=0
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitizer_workload.py > gpurun_out/r4l_$tool.txt 2>&1; echo "exit=$?" >> gpurun_out/r4l_$tool.txt
done
