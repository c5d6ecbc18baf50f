timeout 120 python -m pytest tests/test_spectral_fista.py tests/test_circ_tau.py -x -q -s > gpurun_out/sp_tests.log 2>&1
timeout 60 python tools/circ_probe.py 100 > gpurun_out/sp_probe.log 2>&1
WBX_LIB=paper_1512_08401_b200/lib/libwbx_cprof.so WBX_GRAPH=0 timeout 60 python tools/circ_probe.py 100 > gpurun_out/sp_prof.log 2>&1
