WBX_VERBOSE=1 timeout 300 python tools/c3_probe.py > gpurun_out/c3_probe2.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/gputest13.log 2>&1
echo pytest=$?
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench13.json 2> gpurun_out/bench13.err
echo bench=$?
