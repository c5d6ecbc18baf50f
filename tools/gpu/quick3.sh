timeout 300 python -m pytest tests/test_spectral_fista.py tests/test_tracking.py tests/test_circ_tau.py -x -q > gpurun_out/q3_tests.log 2>&1
timeout 300 python tools/pgd_probe.py > gpurun_out/pgd_probe.log 2>&1
