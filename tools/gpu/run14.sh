WBX_VERBOSE=1 timeout 300 python tools/c3_probe.py > gpurun_out/c3_probe3.log 2>&1
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench14.json 2> gpurun_out/bench14.err
echo bench=$?
timeout 1500 python -m pytest tests/test_varying.py tests/test_gpu_parity.py tests/test_tracking.py tests/test_full_size.py -m gpu -q -x > gpurun_out/gputest14.log 2>&1
echo pytest=$?
