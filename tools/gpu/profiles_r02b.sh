set -x
timeout 600 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-extra > gpurun_out/pb_bench_plain.json 2>&1
echo plain=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/pb_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-extra > gpurun_out/pb_launches.log 2>&1
echo launches=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"circ_|fwd_rows_kernel|fwd_cols_kernel|inv_rows_kernel|inv_cols_kernel" -c 14 -o gpurun_out/spectral_full -f python tools/profile_case.py deblur > gpurun_out/pb_full.log 2>&1
echo full=$?
