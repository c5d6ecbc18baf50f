export WBX_TRACE_FILE=/tmp/trace_w.bin
rm -f $WBX_TRACE_FILE
timeout 300 python tools/trace_phases.py run fista > gpurun_out/tw_run.log 2>&1
timeout 300 python tools/trace_phases.py show /tmp/trace_w.bin blocks > gpurun_out/tw_fista.json 2>&1
python - > gpurun_out/tw_percta.txt 2>&1 <<'PY'
import numpy as np
raw = np.fromfile('/tmp/trace_w.bin', dtype=np.uint64)
G, cap = int(raw[0]), int(raw[1])
rec = 2 + cap * G * 2
last = raw[(len(raw) // rec - 1) * rec:][2:].reshape(cap, G, 2).astype(np.int64)
used = [i for i in range(cap) if last[i, :, 1].max() > 0]
arr = last[used]
work = (arr[1:, :, 0] - arr[:-1, :, 1]) / 1e3
A = work[0::2].mean(0); T = work[1::2].mean(0)
np.set_printoptions(precision=2, linewidth=200)
print("A by cta:", A)
print("T by cta:", T)
PY
