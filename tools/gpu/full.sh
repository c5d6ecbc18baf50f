timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/full_gputest.log 2>&1
echo pytest=$?
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/full_bench.json 2> gpurun_out/full_bench.err
echo bench=$?
