set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 600 python tools/spmv_sweep.py 4096 10 quarter,row,row4 0,2,8,16,32,64 > gpurun_out/sweep1.jsonl 2> gpurun_out/sweep1.err
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gputest1.log 2>&1
echo pytest_rc=$?
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench1.json 2> gpurun_out/bench1.err
echo bench_rc=$?
