# quick GPU check: parity tests + phase traces + probe (used during development)
# usage: bash tools/gpu_quick.sh [ENV=VAL ...]   (extra configurations probed after the default)
set -e
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1 || { tail -30 gpurun_out/pytest_gpu.log; exit 1; }
tail -1 gpurun_out/pytest_gpu.log
trace() {
  export WBX_TRACE_FILE=/tmp/tf.bin; rm -f $WBX_TRACE_FILE
  python tools/trace_phases.py run fista 32 > /dev/null && echo "fista $(python tools/trace_phases.py show $WBX_TRACE_FILE blocks)"
  export WBX_TRACE_FILE=/tmp/tt.bin; rm -f $WBX_TRACE_FILE
  python tools/trace_phases.py run tau 32 > /dev/null && echo "tau $(python tools/trace_phases.py show $WBX_TRACE_FILE blocks)"
  unset WBX_TRACE_FILE
  python tools/probe_solver.py
}
echo "== default"; trace
for kv in "$@"; do
  echo "== $kv"
  if [ "${kv%%=*}" = "TEST" ]; then env ${kv#TEST=} timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -1; continue; fi
  env $kv bash -c "$(declare -f trace); trace"
done
