# Round-end style refresh: GPU tests, smoke, every bench config, the reference
# arm and the ncu launch list of the default step.  Outputs in gpurun_out/$TAG_*.
TAG=${TAG:-r01n}
O=gpurun_out
python -m pytest tests -m gpu -q > $O/${TAG}_pytest_gpu.txt 2>&1; tail -1 $O/${TAG}_pytest_gpu.txt
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/${TAG}_smoke.txt 2>&1; tail -1 $O/${TAG}_smoke.txt
python bench.py > $O/${TAG}_bench_n16384.json 2> $O/${TAG}_bench_n16384.err; tail -c 300 $O/${TAG}_bench_n16384.json
for c in n4096 n256 batch n65536; do python bench.py --config $c > $O/${TAG}_bench_$c.json 2> $O/${TAG}_bench_$c.err; tail -c 200 $O/${TAG}_bench_$c.json; done
python bench.py --impl reference > $O/${TAG}_bench_reference.json 2> $O/${TAG}_bench_reference.err; tail -c 200 $O/${TAG}_bench_reference.json
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/${TAG}_launches16k.csv python tools/ncu_step.py 16384 U > /dev/null 2>&1
python tools/launches.py $O/${TAG}_launches16k.csv > $O/${TAG}_launches16k.txt; head -8 $O/${TAG}_launches16k.txt
RELAPACK_TRACE=1 python tools/trace_timeline.py 4096 L > $O/${TAG}_trace4k.txt 2>&1; head -8 $O/${TAG}_trace4k.txt
RELAPACK_TRACE=1 python tools/trace_timeline.py 16384 U > $O/${TAG}_trace16k.txt 2>&1; head -3 $O/${TAG}_trace16k.txt
RELAPACK_TRACE=1 python tools/e2e_probe.py 16384 U > $O/${TAG}_e2e16k.txt 2>&1; cat $O/${TAG}_e2e16k.txt | grep -v Warn
