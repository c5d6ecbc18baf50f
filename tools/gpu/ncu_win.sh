timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-extra > gpurun_out/nw_bench.json 2> gpurun_out/nw_bench.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fista_win_kernel -c 1 -o gpurun_out/nw -f python tools/profile_case.py deblur > gpurun_out/nw_ncu.log 2>&1
echo ncu=$?
