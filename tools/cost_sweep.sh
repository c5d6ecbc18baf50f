for c in 16,1 4,1 1,1 2,1 8,1; do
  export WBX_WIN_COST=$c
  export WBX_TRACE_FILE=/tmp/tf$c.bin; python tools/trace_phases.py run fista 32 >/dev/null; echo "$c fista $(python tools/trace_phases.py show $WBX_TRACE_FILE blocks | tr '\n' ' ' | cut -c1-420)"
  unset WBX_TRACE_FILE; python tools/probe_solver.py | cut -c1-200
done
