# round-2 final: GPU suite, smoke, bench (both arms), launch list, ncu --set full (C2 deblur, C5 batch)
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/e_gputests.log 2>&1; echo rc=$? >> gpurun_out/e_gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/e_smoke.log 2>&1; echo rc=$? >> gpurun_out/e_smoke.log
timeout 400 python bench.py > gpurun_out/e_bench.json 2> gpurun_out/e_bench.err
timeout 400 python bench.py --impl reference > gpurun_out/e_bench_ref.json 2> gpurun_out/e_bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/e_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-extra > gpurun_out/e_launches.log 2>&1
echo launches=$? >> gpurun_out/e_launches.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"circ_fista|circ_decoupled|fwd_rows|inv_rows" -c 6 -o gpurun_out/e_c5_full -f python tools/profile_case.py c5 > gpurun_out/e_c5_full.log 2>&1
echo c5full=$? >> gpurun_out/e_c5_full.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"circ_fista" -c 2 -o gpurun_out/e_c2_full -f python tools/profile_case.py deblur > gpurun_out/e_c2_full.log 2>&1
echo c2full=$? >> gpurun_out/e_c2_full.log
