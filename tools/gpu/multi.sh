timeout 900 python -m pytest tests/test_spectral_fista.py -m gpu -x -q -k "512" > gpurun_out/mu_tests.log 2>&1; echo rc=$? >> gpurun_out/mu_tests.log
