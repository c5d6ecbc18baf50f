set -x
timeout 1500 python -m pytest tests/test_tracking.py tests/test_psf.py tests/test_reference_suites.py tests/test_full_size.py tests/test_gpu_parity.py -m gpu -q > gpurun_out/gputest4.log 2>&1
echo pytest_rc=$?
