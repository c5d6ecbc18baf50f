timeout 900 python -m pytest tests/test_spectral_fista.py tests/test_tracking.py -m gpu -x -q > gpurun_out/ab2_tests.log 2>&1; echo rc=$? >> gpurun_out/ab2_tests.log
bash tools/gpu/ab.sh
