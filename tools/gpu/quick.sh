timeout 200 python -m pytest tests/test_spectral_fista.py tests/test_gpu_parity.py -x -q -k "spectral or graph or deblur" > gpurun_out/q_tests.log 2>&1
timeout 300 python bench.py --no-extra --no-cpu-baseline > gpurun_out/q_bench.json 2> gpurun_out/q_bench.err
