timeout 300 python tools/pgd_probe.py > gpurun_out/pgd_probe.log 2>&1
