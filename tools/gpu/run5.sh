set -x
timeout 1200 python -m pytest tests/test_sharded.py tests/test_opfile.py tests/test_full_size.py -m gpu -q -x > gpurun_out/gputest5.log 2>&1
echo pytest_rc=$?
timeout 600 python bench.py --workload c4 --size 4096 --steps 3 --warmup 1 > gpurun_out/c4_4096.json 2> gpurun_out/c4_4096.err
echo c4_rc=$?
timeout 600 python bench.py --workload c4 --size 2048 --steps 3 --warmup 1 > gpurun_out/c4_2048.json 2> gpurun_out/c4_2048.err
timeout 600 python bench.py --workload c4 --size 1024 --steps 3 --warmup 1 > gpurun_out/c4_1024.json 2> gpurun_out/c4_1024.err
echo done
