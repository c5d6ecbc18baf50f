timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "variants or deblurrer or fista_fp32" > gpurun_out/snake_test.log 2>&1
echo pytest=$?
for v in 1 0; do
WBX_WIN_SNAKE=$v timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-extra > gpurun_out/snake_bench_$v.json 2> gpurun_out/snake_bench_$v.err
WBX_WIN_SNAKE=$v WBX_LIB=paper_1512_08401_b200/lib/libwbx_prof.so timeout 300 python tools/win_profile.py > gpurun_out/snake_prof_$v.json 2>&1
done
