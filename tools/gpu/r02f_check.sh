# last check of the committed code: GPU suite, smoke, bench (both arms)
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/f_gputests.log 2>&1; echo rc=$? >> gpurun_out/f_gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f_smoke.log 2>&1; echo rc=$? >> gpurun_out/f_smoke.log
timeout 400 python bench.py > gpurun_out/f_bench.json 2> gpurun_out/f_bench.err
timeout 400 python bench.py --impl reference > gpurun_out/f_bench_ref.json 2> gpurun_out/f_bench_ref.err
