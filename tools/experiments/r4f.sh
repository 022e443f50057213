# r4f: multi-GPU executor with the all-gather in place (packed chunk = the rank's slot of the receive buffer)
timeout 900 python -m pytest tests/test_gpu_dist.py -q -m gpu -x > gpurun_out/r4f_tests.txt 2>&1
for nb in 512 1024; do python tools/dist_world1.py 16384 8192 $nb >> gpurun_out/r4f_dist.txt 2>&1; done
