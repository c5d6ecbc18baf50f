set -x
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/gputest6.log 2>&1
echo pytest_rc=$?
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench6.json 2> gpurun_out/bench6.err
echo bench_rc=$?
WBX_GRAPH=0 timeout 900 python bench.py --steps 20 --warmup 5 --no-extra --no-cpu-baseline > gpurun_out/bench6_nograph.json 2> gpurun_out/bench6_nograph.err
timeout 600 python bench.py --workload c4 --size 4096 --steps 3 --warmup 1 > gpurun_out/c4_4096b.json 2> gpurun_out/c4_4096b.err
echo done
