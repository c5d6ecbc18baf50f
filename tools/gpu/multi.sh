timeout 900 python -m pytest tests/test_spectral_fista.py tests/test_tracking.py tests/test_circ_tau.py -m gpu -x -q > gpurun_out/mu_tests.log 2>&1; echo rc=$? >> gpurun_out/mu_tests.log
timeout 300 python tools/c5_probe.py >> gpurun_out/mu_probe.log 2>&1
timeout 300 python bench.py --no-extra --no-cpu-baseline --steps 20 > gpurun_out/mu_bench.json 2>/dev/null
