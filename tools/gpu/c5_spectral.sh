# spectral C5 batches: parity tests, then images/s by slots per launch vs the fp32 batch kernel
timeout 600 python -m pytest tests/test_spectral_fista.py tests/test_batch.py -m gpu -x -q > gpurun_out/c5_tests.log 2>&1; echo rc=$? >> gpurun_out/c5_tests.log
for e in "X=1" "WBX_CIRC_SLOTS=1" ${C5_EXTRA}; do
  echo "== $e" >> gpurun_out/c5_probe.log
  env $e timeout 300 python tools/c5_probe.py >> gpurun_out/c5_probe.log 2>&1
done
timeout 300 python bench.py --no-extra --no-cpu-baseline --steps 10 > gpurun_out/c5_c2bench.json 2>/dev/null
