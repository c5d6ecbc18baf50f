# round-2 re-entry: full GPU suite, smoke, bench (both arms) on the latest commit
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/d_gputests.log 2>&1; echo rc=$? >> gpurun_out/d_gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/d_smoke.log 2>&1; echo rc=$? >> gpurun_out/d_smoke.log
timeout 400 python bench.py > gpurun_out/d_bench.json 2> gpurun_out/d_bench.err
timeout 400 python bench.py --impl reference > gpurun_out/d_bench_ref.json 2> gpurun_out/d_bench_ref.err
echo done
