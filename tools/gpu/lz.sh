# Lanczos step-estimate check schedule on C3: where the 1e-8 agreement is first reached
for fe in "48 4" "24 8" "32 8" "32 4" "40 8" "36 4"; do set -- $fe
  echo "== first $1 every $2" >> gpurun_out/lz.log
  WBX_LZ_FIRST=$1 WBX_LZ_EVERY=$2 timeout 300 python tools/c3_probe.py 2>&1 | tail -1 >> gpurun_out/lz.log
done
