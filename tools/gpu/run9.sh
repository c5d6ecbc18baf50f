set -x
export WBX_TRACE_FILE=/tmp/trace_fista.bin
rm -f $WBX_TRACE_FILE
timeout 300 python tools/trace_phases.py run fista > gpurun_out/trace_run.log 2>&1
timeout 300 python tools/trace_phases.py show /tmp/trace_fista.bin blocks > gpurun_out/trace_fista.json 2>&1
export WBX_TRACE_FILE=/tmp/trace_tau.bin
rm -f $WBX_TRACE_FILE
timeout 300 python tools/trace_phases.py run tau >> gpurun_out/trace_run.log 2>&1
timeout 300 python tools/trace_phases.py show /tmp/trace_tau.bin blocks > gpurun_out/trace_tau.json 2>&1
echo done
