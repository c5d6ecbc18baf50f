# spectral engine with the data-flag exchange: parity tests, C2 bench, barrier-mode comparison, C5
timeout 600 python -m pytest tests/test_spectral_fista.py tests/test_tracking.py -m gpu -x -q > gpurun_out/fl_tests.log 2>&1; echo rc=$? >> gpurun_out/fl_tests.log
timeout 300 python bench.py --no-extra --no-cpu-baseline --steps 20 > gpurun_out/fl_bench.json 2>gpurun_out/fl_bench.err
WBX_CIRC_SYNC=barrier timeout 300 python bench.py --no-extra --no-cpu-baseline --steps 20 > gpurun_out/fl_bench_barrier.json 2>/dev/null
