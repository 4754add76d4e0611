"""ctypes binding of the C ABI in include/mpcr_b200.h.

Loads ``paper_2406_02701_b200/libmpcr_b200.so`` (built in-tree by
``__graft_entry__.build()``).  There is no fallback: if the library is missing
or the device is not a B200, every call raises.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libmpcr_b200.so")
HEADER = os.path.join(os.path.dirname(HERE), "include", "mpcr_b200.h")

# mp_status (include/mpcr_b200.h), mirroring errors.hpp:8-76
OK = 0
STATUS_NAMES = {
    0: "OK", 1: "ShapeMismatch", 2: "IndexOutOfRange", 3: "NotAMatrix", 4: "EmptyArray",
    5: "NotPositiveDefinite", 6: "SingularMatrix", 7: "NoConvergence", 8: "UnknownOperation",
    9: "BackendUnavailable", 10: "PrecisionMismatch", 11: "InvalidParam", 12: "IoError",
    100: "CudaError", 101: "NcclError", 102: "OutOfMemory", 103: "InternalError",
}

_i64 = C.c_int64
_vp = C.c_void_p
_ip = C.POINTER(C.c_int64)

# name -> (restype, argtypes); every export of the header
SIGNATURES = {
    "mp_last_error": (C.c_char_p, []),
    "mp_version": (C.c_char_p, []),
    "mp_device_check": (C.c_int, [C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    "mp_ctx_create": (C.c_int, [C.c_int, C.POINTER(_vp)]),
    "mp_ctx_destroy": (C.c_int, [_vp]),
    "mp_ctx_set_stream": (C.c_int, [_vp, _vp]),
    "mp_ctx_get_stream": (C.c_int, [_vp, C.POINTER(_vp)]),
    "mp_ctx_synchronize": (C.c_int, [_vp]),
    "mp_prof_enable": (C.c_int, [_vp, C.c_int]),
    "mp_prof_reset": (C.c_int, [_vp]),
    "mp_prof_trace": (C.c_int, [_vp, C.c_int]),
    "mp_prof_trace_dump": (C.c_int, [_vp, C.c_char_p]),
    "mp_rng_uniform": (C.c_int, [C.c_uint64, C.c_int64, C.c_int64, _vp]),
    "mp_rng_normal": (C.c_int, [C.c_uint64, C.c_int64, _vp]),
    "mp_op_is_unary": (C.c_int, [C.c_char_p, C.POINTER(C.c_int)]),
    "mp_resolve": (C.c_int, [C.c_char_p, C.c_int, C.c_int, _vp]),
    "mp_execute": (C.c_int, [_vp, _vp, C.c_char_p, _vp, _vp, C.POINTER(_vp)]),
    "mp_prof_digit_products": (C.c_int, [_vp, _vp, _vp]),
    "mp_prof_query": (C.c_int, [_vp, C.c_int, C.POINTER(C.c_double), _ip, C.POINTER(C.c_double)]),
    "mp_launch_count": (C.c_int, [_vp, _ip]),
    "mp_host_alloc": (C.c_int, [C.c_size_t, C.POINTER(_vp)]),
    "mp_host_free": (C.c_int, [_vp]),
    "mp_array_create": (C.c_int, [_vp, C.c_int, _i64, _i64, C.c_int, C.POINTER(_vp)]),
    "mp_array_wrap": (C.c_int, [_vp, C.c_int, _i64, _i64, _i64, _vp, C.POINTER(_vp)]),
    "mp_array_destroy": (C.c_int, [_vp]),
    "mp_array_info": (C.c_int, [_vp, C.POINTER(C.c_int), _ip, _ip, _ip, C.POINTER(C.c_int), C.POINTER(_vp)]),
    "mp_array_to_matrix": (C.c_int, [_vp, _i64, _i64]),
    "mp_array_upload": (C.c_int, [_vp, _vp, C.c_size_t]),
    "mp_array_download": (C.c_int, [_vp, _vp, C.c_size_t]),
    "mp_array_from_doubles": (C.c_int, [_vp, _vp, _i64]),
    "mp_array_to_doubles": (C.c_int, [_vp, _vp, _i64]),
    "mp_array_get": (C.c_int, [_vp, _i64, _i64, C.POINTER(C.c_double)]),
    "mp_array_set": (C.c_int, [_vp, _i64, _i64, C.c_double]),
    "mp_convert": (C.c_int, [_vp, _vp, _vp]),
    "mp_convert_raw": (C.c_int, [_vp, C.c_int, _vp, C.c_int, _vp, _i64]),
    "mp_ew_binary": (C.c_int, [_vp, C.c_int, _vp, _vp, _vp]),
    "mp_ew_scalar": (C.c_int, [_vp, C.c_int, _vp, C.c_double, _vp]),
    "mp_ew_unary": (C.c_int, [_vp, C.c_int, _vp, _vp]),
    "mp_reduce": (C.c_int, [_vp, C.c_int, _vp, C.POINTER(C.c_double)]),
    "mp_transpose": (C.c_int, [_vp, _vp, _vp]),
    "mp_diag": (C.c_int, [_vp, _vp, _vp]),
    "mp_gemm": (C.c_int, [_vp, _vp, _vp, _vp, C.c_int, C.c_int, C.c_double, C.c_double]),
    "mp_gemm_raw": (C.c_int, [_vp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, _i64, _i64, _i64,
                              C.c_double, _vp, _i64, _vp, _i64, C.c_double, _vp, _i64]),
    "mp_matmul": (C.c_int, [_vp, _vp, _vp, _vp]),
    "mp_crossprod": (C.c_int, [_vp, _vp, _vp, _vp]),
    "mp_chol": (C.c_int, [_vp, _vp, _vp, _ip]),
    "mp_trsm": (C.c_int, [_vp, _vp, _vp, C.c_int, C.c_int, C.c_int, C.c_double]),
    "mp_forwardsolve": (C.c_int, [_vp, _vp, _vp, _vp]),
    "mp_backsolve": (C.c_int, [_vp, _vp, _vp, _vp]),
    "mp_solve": (C.c_int, [_vp, _vp, _vp, _vp]),
    "mp_chol2inv": (C.c_int, [_vp, _vp, _vp]),
    "mp_tile_create": (C.c_int, [_vp, _i64, _i64, _i64, _i64, C.POINTER(C.c_int), C.POINTER(_vp)]),
    "mp_tile_destroy": (C.c_int, [_vp]),
    "mp_tile_info": (C.c_int, [_vp, _ip, _ip, _ip, _ip, _ip, _ip]),
    "mp_tile_set_values": (C.c_int, [_vp, _vp]),
    "mp_tile_get_values": (C.c_int, [_vp, _vp]),
    "mp_tile_get_rows": (C.c_int, [_vp, _vp, C.c_int64, _vp]),
    "mp_tile_set_values_device": (C.c_int, [_vp, _vp, _i64]),
    "mp_tile_get_tile": (C.c_int, [_vp, _i64, _i64, C.POINTER(_vp)]),
    "mp_tile_precision": (C.c_int, [_vp, _i64, _i64, C.POINTER(C.c_int)]),
    "mp_tile_gemm": (C.c_int, [_vp, _vp, _vp, _vp, C.c_int, C.c_int, C.c_double, C.c_double]),
    "mp_tile_chol": (C.c_int, [_vp, _vp, C.c_int, C.POINTER(_vp), _ip]),
    "mp_tile_trsm": (C.c_int, [_vp, _vp, _vp, C.c_int, C.c_int, C.c_int, C.c_double]),
    "mp_tile_logdet": (C.c_int, [_vp, _vp, C.POINTER(C.c_double)]),
    "mp_tile_fill_matern": (C.c_int, [_vp, _vp, _i64, C.c_double, C.c_double, C.c_double]),
    "mp_tile_fill_matern_points": (C.c_int, [_vp, _vp, _vp, _vp, _i64, C.c_double, C.c_double,
                                             C.c_double, C.c_double]),
    "mp_tile_convert": (C.c_int, [_vp, _vp, _vp]),
    "mp_tile_copy": (C.c_int, [_vp, _vp, _vp]),
    "mp_tile_gaussian_nll": (C.c_int, [_vp, _vp, _vp, C.c_double, C.c_double,
                                       C.POINTER(C.c_double), C.POINTER(C.c_double),
                                       C.POINTER(C.c_double), C.POINTER(C.c_double)]),
    "mp_tile_matern_mle": (C.c_int, [_vp, _vp, _vp, _vp, _vp, _i64, C.c_double, C.c_double, C.c_double,
                                     C.c_int, C.c_double, C.c_double, C.c_double,
                                     C.POINTER(C.c_double), C.POINTER(C.c_double), C.POINTER(C.c_double),
                                     C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    # multi-GPU (2D block-cyclic MPCRTile)
    "mp_nccl_unique_id": (C.c_int, [C.c_char_p]),
    "mp_dist_create": (C.c_int, [_vp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_char_p, C.POINTER(_vp)]),
    "mp_dist_create_sim": (C.c_int, [C.POINTER(_vp), C.c_int, C.c_int, C.c_int, C.POINTER(_vp)]),
    "mp_dist_destroy": (C.c_int, [_vp]),
    "mp_dist_owner": (C.c_int, [_i64, _i64, C.c_int, C.c_int]),
    "mp_dist_schedule": (C.c_int, [C.c_int, C.c_int, C.c_int, _i64, C.POINTER(C.c_int),
                                   C.POINTER(C.c_int32), _i64, _ip]),
    "mp_tile_create_dist": (C.c_int, [_vp, _vp, _i64, _i64, C.POINTER(C.c_int), C.POINTER(_vp)]),
    "mp_tile_owns": (C.c_int, [_vp, _i64, _i64]),
}


class MPError(RuntimeError):
    """Raised for a non-OK mp_status; ``kind`` is the reference exception name."""

    def __init__(self, status: int, message: str, info: int = -1):
        self.status = status
        self.kind = STATUS_NAMES.get(status, f"status{status}")
        self.info = info
        super().__init__(f"{self.kind}: {message}")


_lib = None


def lib() -> C.CDLL:
    """Load the CUDA library (raises if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} not built: run `python -c 'import __graft_entry__ as g; g.build()'`")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def check(status: int, info: int = -1) -> None:
    if status != OK:
        msg = lib().mp_last_error().decode(errors="replace")
        raise MPError(status, msg, info)
