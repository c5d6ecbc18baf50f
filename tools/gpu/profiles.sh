set -x
timeout 900 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-extra > gpurun_out/pf_bench_plain.json 2>&1
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/pf_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-extra > gpurun_out/pf_launches.log 2>&1
echo launches=$?
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"fista_win_track_kernel|fwd_rows_kernel|fwd_cols_kernel|inv_rows_kernel|inv_cols_kernel|fista_win_kernel|tau_lanczos_win_kernel" -c 12 -o gpurun_out/solver_full -f python tools/profile_case.py > gpurun_out/pf_solver.log 2>&1
echo full=$?
