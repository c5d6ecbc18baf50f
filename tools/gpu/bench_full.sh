WBX_VERBOSE=1 timeout 300 python tools/c3_probe.py > gpurun_out/bf_c3_probe.log 2>&1
timeout 1200 python bench.py --steps 10 --warmup 3 > gpurun_out/bf_bench.json 2> gpurun_out/bf_bench.err
echo bench=$?
