WBX_GRAPH=0 WBX_CIRC_DIAG=prof timeout 120 python tools/circ_probe.py 100 > gpurun_out/s12_prof.log 2>&1
