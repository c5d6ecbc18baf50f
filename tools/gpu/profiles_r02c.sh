timeout 900 ncu --set full --clock-control none --import-source on -k regex:"circ_fista|inv_rows_kernel|inv_cols_kernel" -c 9 -o gpurun_out/spectral_fista_full -f python tools/profile_case.py deblur > gpurun_out/pc_full.log 2>&1
echo full=$?
