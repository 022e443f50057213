# r3t: current critical path of n = 4096 / 256 (serial durations on the DAG, traced timeline)
python tools/critical_path.py 4096 L > gpurun_out/r3t_cp4096.txt 2>&1
RELAPACK_TRACE=1 python tools/trace_timeline.py 4096 L > gpurun_out/r3t_tl4096.txt 2>&1
python tools/critical_path.py 256 L > gpurun_out/r3t_cp256.txt 2>&1
RELAPACK_TRACE=1 python tools/trace_timeline.py 256 L > gpurun_out/r3t_tl256.txt 2>&1
