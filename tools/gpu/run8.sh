set -x
timeout 600 python tools/barrier_sweep.py 1,2,4,8,16 20 > gpurun_out/barrier_sweep.jsonl 2> gpurun_out/barrier_sweep.err
echo sweep=$?
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_tracking.py -m gpu -q -x > gpurun_out/gputest8.log 2>&1
echo pytest=$?
