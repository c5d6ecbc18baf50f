import ctypes as C, json, sys
from pathlib import Path
lib = C.CDLL(str(Path(__file__).resolve().parents[1] / "paper_1512_08401_b200" / "lib" / "libwbx.so"))
lib.wbx_diag_barrier_us.argtypes = [C.c_int, C.c_int, C.c_int, C.POINTER(C.c_double)]
out = {}
for bps in (1, 2, 4, 8):
    us = C.c_double()
    rc = lib.wbx_diag_barrier_us(0, 2000, bps, C.byref(us))
    out[f"{bps}_blocks_per_sm"] = round(us.value, 3) if rc == 0 else f"rc={rc}"
print(json.dumps({"grid_barrier_us": out}))
