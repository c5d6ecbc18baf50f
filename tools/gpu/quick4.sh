timeout 300 python -m pytest tests/test_spectral_fista.py tests/test_circ_tau.py -x -q > gpurun_out/q4_tests.log 2>&1
timeout 60 python tools/circ_probe.py 100 > gpurun_out/sp_probe.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/q4_launches.csv python tools/circ_probe.py 100 > gpurun_out/q4_ncu.log 2>&1
