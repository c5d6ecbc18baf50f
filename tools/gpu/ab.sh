# A/B of two library builds in one box: WBX_LIB=lib/libwbx_prev.so (previous commit) vs the current one
for r in 1 2 3; do
  for lib in libwbx_prev.so libwbx.so; do
    WBX_LIB=$PWD/paper_1512_08401_b200/lib/$lib timeout 300 python bench.py --no-extra --no-cpu-baseline --steps 30 > gpurun_out/ab_$lib.$r.json 2>/dev/null
  done
done
