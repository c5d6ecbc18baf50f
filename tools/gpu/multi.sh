timeout 900 python -m pytest tests/test_spectral_fista.py tests/test_batch.py tests/test_gpu_parity.py tests/test_full_size.py -m gpu -x -q > gpurun_out/mu_tests.log 2>&1; echo rc=$? >> gpurun_out/mu_tests.log
timeout 300 python tools/c5_probe.py >> gpurun_out/mu_probe.log 2>&1
