set -x
timeout 600 python tools/spmv_sweep.py 4096 10 row2,row,row8 0 > gpurun_out/sweep2.jsonl 2> gpurun_out/sweep2.err
timeout 1500 python -m pytest tests/test_full_size.py tests/test_spmv_compact.py tests/test_gpu_parity.py -m gpu -x -q -k "full_size or spmv or preconditioner" > gpurun_out/gputest2.log 2>&1
echo pytest_rc=$?
WBX_VERBOSE=1 timeout 300 python tools/spai_time.py > gpurun_out/spai2.log 2>&1
# ncu: DRAM bytes of the default row kernel (forward + adjoint), one --set full capture each
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sell_row_kernel -c 2 -o gpurun_out/spmv_row_full python tools/spmv_sweep.py 4096 1 row 0 > gpurun_out/ncu2.log 2>&1
echo ncu_rc=$?
timeout 900 python bench.py --steps 10 --warmup 3 --no-extra > gpurun_out/bench2.json 2> gpurun_out/bench2.err
echo bench_rc=$?
