WBX_CIRC_STAGED=1 timeout 900 python -m pytest tests/test_spectral_fista.py -m gpu -x -q > gpurun_out/st_tests.log 2>&1; echo rc=$? >> gpurun_out/st_tests.log
for r in 1 2 3; do
  for m in 0 1; do
    WBX_CIRC_STAGED=$m timeout 300 python bench.py --no-extra --no-cpu-baseline --steps 30 > gpurun_out/st_$m.$r.json 2>/dev/null
  done
done
