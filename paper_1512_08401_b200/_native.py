"""ctypes binding of libwbx.so (the C ABI declared in include/wbx.h).

The library is built in-tree by `paper_1512_08401_b200/Makefile` (see
`__graft_entry__.build()`). There is no fallback: if the shared object is missing,
importing this module raises, and every product entry point fails loudly.
"""
from __future__ import annotations

import atexit
import ctypes as C
import os
from pathlib import Path

# WBX_LIB selects a diagnostics build (e.g. lib/libwbx_prof.so from `make prof`)
LIB_PATH = Path(os.environ.get("WBX_LIB") or Path(__file__).resolve().parent / "lib" / "libwbx.so")

WBX_OK = 0
WBX_FP32 = 32
WBX_FP64 = 64
WBX_PSF_GAUSSIAN, WBX_PSF_SKEWED, WBX_PSF_MOTION, WBX_PSF_AIRY, WBX_PSF_DEFOCUS = range(5)


class wbx_band(C.Structure):
    _fields_ = [("level", C.c_uint32), ("orientation", C.c_uint32),
                ("shape", C.c_uint64 * 2), ("offset", C.c_uint64)]


class wbx_solver_cfg(C.Structure):
    _fields_ = [("max_iters", C.c_uint64), ("rel_energy_tol", C.c_double),
                ("step_safety", C.c_double), ("ref_energy", C.c_double),
                ("zero_momentum", C.c_int32), ("track_support", C.c_int32),
                ("track_energy", C.c_int32), ("precision", C.c_int32), ("tau", C.c_double)]


class wbx_report(C.Structure):
    _fields_ = [("iters_used", C.c_uint64), ("initial_energy", C.c_double),
                ("wall_time_s", C.c_double), ("tau", C.c_double), ("tau_iters", C.c_uint32),
                ("ops_per_pixel_per_iter", C.c_double),
                ("energies", C.POINTER(C.c_double)),
                ("support_sizes", C.POINTER(C.c_uint64))]


class wbx_op_info(C.Structure):
    _fields_ = [("n", C.c_uint64), ("nnz", C.c_uint64), ("nonempty_rows", C.c_uint64),
                ("nonempty_cols", C.c_uint64), ("sell_rows_padded", C.c_uint64),
                ("sell_cols_padded", C.c_uint64), ("device_bytes", C.c_uint64),
                ("bytes_per_iter_fp32", C.c_uint64)]


_P = C.c_void_p
_D = C.POINTER(C.c_double)
_U64 = C.POINTER(C.c_uint64)
_U32 = C.POINTER(C.c_uint32)

# name -> (restype, argtypes); every symbol include/wbx.h declares
SIGNATURES = {
    "wbx_last_error": (C.c_char_p, []),
    "wbx_abi_version": (C.c_int, []),
    "wbx_ctx_create": (C.c_int, [C.c_int, C.POINTER(_P)]),
    "wbx_ctx_destroy": (C.c_int, [_P]),
    "wbx_ctx_stream": (C.c_void_p, [_P]),
    "wbx_ctx_synchronize": (C.c_int, [_P]),
    "wbx_ctx_launch_count": (C.c_uint64, [_P]),
    "wbx_make_filters": (C.c_int, [C.c_uint32, C.c_uint32, _D, _D, _U32]),
    "wbx_parse_filter": (C.c_int, [C.c_char_p, _U32, _U32]),
    "wbx_make_layout": (C.c_int, [C.c_uint32, _U64, C.c_uint32, C.POINTER(wbx_band), _U32]),
    "wbx_basis_create": (C.c_int, [_P, C.c_uint32, C.c_uint32, C.c_uint32, _U64, C.c_uint32,
                                   C.POINTER(_P)]),
    "wbx_basis_destroy": (C.c_int, [_P]),
    "wbx_analyze": (C.c_int, [_P, _P, _D, _D]),
    "wbx_synthesize": (C.c_int, [_P, _P, _D, _D]),
    "wbx_analyze_dev": (C.c_int, [_P, _P, _P, _P]),
    "wbx_synthesize_dev": (C.c_int, [_P, _P, _P, _P]),
    "wbx_single_wavelet": (C.c_int, [_P, _P, C.c_uint32, C.c_uint32, _D]),
    "wbx_op_create": (C.c_int, [_P, C.c_uint64, _U64, _U32, _D, C.POINTER(_P)]),
    "wbx_op_destroy": (C.c_int, [_P]),
    "wbx_op_get_info": (C.c_int, [_P, C.POINTER(wbx_op_info)]),
    "wbx_spmv": (C.c_int, [_P, _P, C.c_int, _D, _D]),
    "wbx_spmv_dev": (C.c_int, [_P, _P, C.c_int, C.c_int, _P, _P]),
    "wbx_spmv_compact_dev": (C.c_int, [_P, _P, C.c_int, C.c_int, _P, _P]),
    "wbx_op_set_generators": (C.c_int, [_P, C.c_uint32, _U64, C.c_uint32, C.c_uint64, _U32, _U32, _U64, _D]),
    "wbx_op_set_layout": (C.c_int, [_P, C.c_uint32, _U64, C.c_uint32]),
    "wbx_write_operator": (C.c_int, [C.c_char_p, C.c_uint32, _U64, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint64,
                                     _U64, _U32, _D]),
    "wbx_read_operator": (C.c_int, [C.c_char_p, _U32, _U64, _U32, _U32, _U32, _U64, _U64, C.POINTER(_U64),
                                    C.POINTER(_U32), C.POINTER(_D)]),
    "wbx_op_save": (C.c_int, [_P, C.c_char_p, _D, C.c_double]),
    "wbx_op_get_csr": (C.c_int, [_P, _U64, _U32, _D]),
    "wbx_op_load": (C.c_int, [_P, C.c_char_p, C.POINTER(_P), _D, C.POINTER(C.c_int), C.POINTER(C.c_double)]),
    "wbx_approx_gradient": (C.c_int, [_P, _P, _D, _D, _D]),
    "wbx_stencil_create": (C.c_int, [_P, C.c_uint32, _U64, C.c_uint32, C.c_uint64, _U32, _U32, _U64, _D,
                                     C.POINTER(C.c_void_p)]),
    "wbx_stencil_destroy": (C.c_int, [_P]),
    "wbx_stencil_spmv_dev": (C.c_int, [_P, C.c_int, C.c_int, _P, _P]),
    "wbx_exact_op_create": (C.c_int, [_P, _P, _D, C.POINTER(C.c_void_p)]),
    "wbx_exact_op_destroy": (C.c_int, [_P]),
    "wbx_exact_apply": (C.c_int, [_P, C.c_int, _D, _D]),
    "wbx_exact_apply_dev": (C.c_int, [_P, C.c_int, _P, _P]),
    "wbx_estimate_step_exact": (C.c_int, [_P, _D, C.c_double, _D, C.POINTER(C.c_uint32)]),
    "wbx_pgd_exact": (C.c_int, [_P, _D, _D, C.c_double, _D, C.POINTER(wbx_solver_cfg), C.c_int, _D,
                                C.POINTER(wbx_report)]),
    "wbx_theta_conv_topk": (C.c_int, [_P, _P, _D, _D, C.c_uint64, C.c_uint64, _U32, _U32, _U64, _D, _U64]),
    "wbx_psf_gaussian": (C.c_int, [C.c_uint32, _U64, C.c_double, _D]),
    "wbx_generate_psf": (C.c_int, [_P, C.c_uint32, _D, C.c_uint32, _U64, _D]),
    "wbx_convolve": (C.c_int, [_P, C.c_uint32, _U64, _D, _D, C.c_int, _D]),
    "wbx_add_noise": (C.c_int, [_P, C.c_uint64, _D, C.c_double, C.c_uint64, _D]),
    "wbx_degrade": (C.c_int, [_P, C.c_uint32, _U64, _D, _D, C.c_double, C.c_uint64, _D]),
    "wbx_theta_expand": (C.c_int, [C.c_uint32, _U64, C.c_uint32, C.c_uint64, _U32, _U32, _U64, _D,
                                   _U64, _U64, _U32, _D]),
    "wbx_theta_varying": (C.c_int, [C.c_uint32, _U64, C.c_uint32, C.c_uint32, _D, _U64, _U32, _U32, _U64, _D,
                                    C.c_double, C.c_double, _U64, C.POINTER(_U64), C.POINTER(_U32),
                                    C.POINTER(_D)]),
    "wbx_free": (None, [C.c_void_p]),
    "wbx_gram_diagonals": (C.c_int, [_P, _P, C.c_uint64, _D, _D]),
    "wbx_spai": (C.c_int, [_P, _P, _D]),
    "wbx_jacobi": (C.c_int, [_P, _P, C.c_double, _D]),
    "wbx_scale_weights": (C.c_int, [C.c_uint32, _U64, C.c_uint32, _D]),
    "wbx_prox_l1w": (C.c_int, [_P, C.c_uint64, _D, C.c_double, _D, C.c_double, _D, _D]),
    "wbx_energy": (C.c_int, [_P, _P, _D, _D, _D, C.c_double, _D]),
    "wbx_estimate_step": (C.c_int, [_P, _P, _D, C.c_double, _D, _U32]),
    "wbx_solver_cfg_default": (None, [C.POINTER(wbx_solver_cfg)]),
    "wbx_pgd": (C.c_int, [_P, _P, _D, _D, C.c_double, _D, C.POINTER(wbx_solver_cfg), C.c_int, _D,
                          C.POINTER(wbx_report)]),
    "wbx_solver_create": (C.c_int, [_P, _P, _P, _D, _D, C.c_double, C.POINTER(wbx_solver_cfg),
                                    C.POINTER(_P)]),
    "wbx_solver_create_batch": (C.c_int, [_P, _P, _P, _D, _D, C.c_double, C.POINTER(wbx_solver_cfg), C.c_int,
                                          C.POINTER(_P)]),
    "wbx_solver_batch": (C.c_int, [_P]),
    "wbx_solver_destroy": (C.c_int, [_P]),
    "wbx_deblur_dev": (C.c_int, [_P, _P, _P, C.c_int]),
    "wbx_deblur": (C.c_int, [_P, _D, _D, C.c_int, C.POINTER(wbx_report)]),
    "wbx_solver_last_stats": (C.c_int, [_P, _U64, C.POINTER(C.c_float)]),
    "wbx_solver_phase_ms": (C.c_int, [_P, C.POINTER(C.c_float), C.POINTER(C.c_float)]),
    "wbx_solver_tau_stats": (C.c_int, [_P, C.POINTER(C.c_double), C.POINTER(C.c_uint32), C.POINTER(C.c_uint32)]),
    "wbx_solver_kernels": (C.c_int, [_P, C.c_char_p, C.c_uint64]),
    "wbx_comm_get_unique_id": (C.c_int, [C.c_char_p]),
    "wbx_comm_create": (C.c_int, [_P, C.c_uint32, C.c_uint32, C.c_char_p, C.POINTER(_P)]),
    "wbx_comm_destroy": (C.c_int, [_P]),
    "wbx_sharded_create": (C.c_int, [_P, C.c_uint64, _U64, _U32, _D, _P, _D, _D, C.c_double,
                                     C.POINTER(wbx_solver_cfg), C.c_uint32, _U32, C.c_uint32, _P, C.POINTER(_P)]),
    "wbx_sharded_destroy": (C.c_int, [_P]),
    "wbx_sharded_estimate_step": (C.c_int, [_P, C.c_double, _D, _U32, _U32]),
    "wbx_sharded_deblur_dev": (C.c_int, [_P, _P, _P, C.c_int]),
    "wbx_sharded_stats": (C.c_int, [_P, _D, _U32, _U32, C.POINTER(C.c_float), C.POINTER(C.c_float), _U64]),
    "wbx_shard_create": (C.c_int, [_P, C.c_uint64, _U64, _U32, _D, C.c_uint32, C.c_uint32, C.POINTER(_P)]),
    "wbx_shard_destroy": (C.c_int, [_P]),
    "wbx_shard_plan": (C.c_int, [C.c_uint64, _U64, _U32, C.c_uint32, _U64, _U64]),
    "wbx_shard_get_info": (C.c_int, [_P, _U64]),
    "wbx_shard_bind": (C.c_int, [_P, _P, _P, _P, _P]),
    "wbx_shard_setup": (C.c_int, [_P, _D, _D, C.c_double, C.c_int, C.c_int]),
    "wbx_shard_init": (C.c_int, [_P, C.c_double, _P, _P]),
    "wbx_shard_phase_a": (C.c_int, [_P]),
    "wbx_shard_phase_t": (C.c_int, [_P, C.c_int]),
    "wbx_shard_finalize": (C.c_int, [_P, _P]),
    "wbx_shard_bind_power": (C.c_int, [_P, _P]),
    "wbx_shard_power_begin": (C.c_int, [_P]),
    "wbx_shard_power_update": (C.c_int, [_P, C.c_int]),
    "wbx_shard_power_step_a": (C.c_int, [_P]),
    "wbx_shard_power_step_t": (C.c_int, [_P]),
    "wbx_shard_power_result": (C.c_int, [_P, C.c_double, _D, C.POINTER(C.c_uint32)]),
    "wbx_shard_lz_begin": (C.c_int, [_P]),
    "wbx_shard_lz_update": (C.c_int, [_P, C.c_int, C.c_int, C.c_int, C.c_int]),
    "wbx_shard_lz_step_a": (C.c_int, [_P]),
    "wbx_shard_lz_step_t": (C.c_int, [_P]),
    "wbx_shard_lz_done": (C.c_int, [_P, C.POINTER(C.c_int)]),
    "wbx_shard_lz_result": (C.c_int, [_P, C.c_double, C.POINTER(C.c_double), C.POINTER(C.c_uint32), C.POINTER(C.c_uint32)]),
}


# include/wbx_diag.h (diagnostics, not part of the drop-in boundary)
DIAG_SIGNATURES = {
    "wbx_diag_barrier_us": (C.c_int, [C.c_int, C.c_int, C.c_int, _D]),
    "wbx_diag_stream_gbs": (C.c_int, [C.c_int, C.c_int, C.c_uint64, C.c_int, C.c_int, C.c_int, C.c_int, _D]),
    "wbx_diag_slice_profile": (C.c_int, [_D]),
    "wbx_diag_spmv_compact_mode": (C.c_int, [_P, _P, C.c_int, C.c_int, _P, _P]),
    "wbx_diag_set_spmv_pf": (C.c_int, [C.c_longlong]),
    "wbx_diag_stencil_apply_host": (C.c_int, [C.c_uint32, _U64, C.c_uint32, C.c_uint64, _U32, _U32, _U64, _D,
                                              C.c_int, C.c_uint32, _D, _D]),
    "wbx_diag_win_features": (C.c_int, [_P, C.c_int, _D, C.POINTER(C.c_int)]),
    "wbx_diag_circ_info": (C.c_int, [_P, C.c_uint32, _U64, C.c_uint32, _U32, C.c_char_p, C.c_uint64]),
}


def _load() -> C.CDLL:
    if not LIB_PATH.exists():
        raise ImportError(
            f"libwbx.so not found at {LIB_PATH}; build it with `python -c 'import __graft_entry__ as g; "
            f"g.build()'` (make -C paper_1512_08401_b200). There is no CPU fallback.")
    lib = C.CDLL(str(LIB_PATH), mode=os.RTLD_NOW | C.RTLD_GLOBAL)
    for name, (res, args) in list(SIGNATURES.items()) + list(DIAG_SIGNATURES.items()):
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


lib = _load()

# Interpreter exit: native objects are NOT released from __del__ any more (finalisation order is
# arbitrary at exit, so an object could otherwise be released after the context it lives on;
# the process exit frees the device anyway).
_SHUTDOWN = [False]
atexit.register(lambda: _SHUTDOWN.__setitem__(0, True))


def alive() -> bool:
    return not _SHUTDOWN[0]


def last_error() -> str:
    msg = lib.wbx_last_error()
    return msg.decode() if msg else ""
