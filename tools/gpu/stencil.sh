export WBX_STENCIL=1
timeout 600 python -m pytest tests/test_stencil_engine.py -q -x > gpurun_out/stencil_test.log 2>&1
echo pytest=$?
for f in 0 1; do
WBX_ST_FILL=$f WBX_LIB=paper_1512_08401_b200/lib/libwbx_prof.so timeout 300 python tools/st_profile.py > gpurun_out/stencil_prof$f.json 2>&1
WBX_ST_FILL=$f timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-extra > gpurun_out/stencil_bench$f.json 2> gpurun_out/stencil_bench$f.err
done
export WBX_TRACE_FILE=/tmp/trace_st.bin
rm -f $WBX_TRACE_FILE
timeout 300 python tools/trace_phases.py run fista > gpurun_out/stencil_trace_run.log 2>&1
timeout 300 python tools/trace_phases.py show /tmp/trace_st.bin blocks > gpurun_out/stencil_trace.json 2>&1
