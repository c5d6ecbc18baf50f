set -x
mkdir -p gpurun_out/r7
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r7/launches.csv python bench.py --steps 2 --warmup 1 --no-extra --no-cpu-baseline > gpurun_out/r7/ncu_launch.log 2>&1
echo ncu1=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"fista_win_track_kernel|fwd_rows_kernel|fwd_cols_kernel|inv_rows_kernel|inv_cols_kernel|fista_win_kernel|tau_lanczos_win_kernel" -c 12 -o gpurun_out/r7/solver_full python tools/profile_case.py > gpurun_out/r7/ncu_full.log 2>&1
echo ncu2=$?
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python tools/sanitize_case.py > gpurun_out/r7/memcheck.log 2>&1
echo memcheck=$?
timeout 900 compute-sanitizer --tool racecheck --print-limit 20 python tools/sanitize_case.py > gpurun_out/r7/racecheck.log 2>&1
echo racecheck=$?
timeout 900 compute-sanitizer --tool synccheck --print-limit 20 python tools/sanitize_case.py > gpurun_out/r7/synccheck.log 2>&1
echo synccheck=$?
