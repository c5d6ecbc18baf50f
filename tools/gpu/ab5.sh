for r in 1 2; do
  for lib in libwbx.so libwbx_b32.so libwbx_b128.so; do
    WBX_LIB=$PWD/paper_1512_08401_b200/lib/$lib timeout 300 python bench.py --no-extra --no-cpu-baseline --steps 30 > gpurun_out/ab_$lib.$r.json 2>/dev/null
  done
done
