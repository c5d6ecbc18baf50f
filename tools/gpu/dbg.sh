timeout 60 python tools/spectral_debug.py > gpurun_out/dbg.log 2>&1; timeout 60 python tools/spectral_debug.py 128 2 >> gpurun_out/dbg.log 2>&1
