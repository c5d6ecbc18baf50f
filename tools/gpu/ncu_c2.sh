timeout 900 ncu --set full --clock-control none --import-source on -k regex:"circ_fista" -c 1 -o gpurun_out/f_c2_full -f python tools/profile_case.py deblur > gpurun_out/f_c2_full.log 2>&1
echo c2full=$? >> gpurun_out/f_c2_full.log
