"""L2/HBM streaming bandwidth: TMA bulk copies per warp vs 16-B loads (wbx_diag.h)."""
import ctypes as C
import json
from pathlib import Path

lib = C.CDLL(str(Path(__file__).resolve().parents[1] / "paper_1512_08401_b200" / "lib" / "libwbx.so"))
lib.wbx_diag_stream_gbs.argtypes = [C.c_int, C.c_int, C.c_uint64, C.c_int, C.c_int, C.c_int, C.c_int,
                                    C.POINTER(C.c_double)]
out = {}
for size_mb in (48, 1024):
    for mode, chunk, infl, bps in [(1, 0, 0, 2), (1, 0, 0, 4), (0, 4096, 2, 2), (0, 4096, 3, 2), (0, 4096, 4, 1),
                                   (0, 8192, 3, 1), (0, 16384, 2, 1), (0, 2048, 6, 2)]:
        g = C.c_double()
        reps = 20 if size_mb < 100 else 2
        rc = lib.wbx_diag_stream_gbs(0, mode, size_mb << 20, reps, chunk, infl, bps, C.byref(g))
        out[f"{size_mb}MB mode{mode} chunk{chunk} inflight{infl} bps{bps}"] = round(g.value, 1) if rc == 0 else f"rc={rc}"
print(json.dumps(out, indent=1))
