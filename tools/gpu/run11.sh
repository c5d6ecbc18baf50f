timeout 1200 python -m pytest tests/test_sharded.py tests/test_full_size.py -m gpu -q -x > gpurun_out/gputest11.log 2>&1
echo pytest=$?
timeout 600 python bench.py --workload c4 --size 4096 --steps 3 --warmup 1 > gpurun_out/c4_4096c.json 2> gpurun_out/c4_4096c.err
echo c4=$?
