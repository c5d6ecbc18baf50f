timeout 900 python -m pytest tests/test_spectral_fista.py tests/test_batch.py -m gpu -x -q > gpurun_out/ab2_tests.log 2>&1; echo rc=$? >> gpurun_out/ab2_tests.log
for r in 1 2; do
  for lib in libwbx_prev.so libwbx.so; do
    WBX_LIB=$PWD/paper_1512_08401_b200/lib/$lib timeout 300 python tools/c5_probe.py > gpurun_out/ab_$lib.$r.json 2>/dev/null
  done
done
