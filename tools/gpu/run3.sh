set -x
timeout 1200 python -m pytest tests/test_tracking.py tests/test_full_size.py tests/test_spmv_compact.py tests/test_reference_suites.py -m gpu -q -x > gpurun_out/gputest3.log 2>&1
echo pytest_rc=$?
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench3.json 2> gpurun_out/bench3.err
echo bench_rc=$?
