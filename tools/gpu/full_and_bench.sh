timeout 1300 python -m pytest tests -m gpu -x -q > gpurun_out/fb_gputests.log 2>&1; echo rc=$? >> gpurun_out/fb_gputests.log
timeout 400 python bench.py > gpurun_out/fb_bench.json 2> gpurun_out/fb_bench.err
