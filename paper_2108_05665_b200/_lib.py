"""Loader for the in-tree engine library ``libmtcg.so`` (C ABI: include/mtcg.h).

The library is built by ``paper_2108_05665_b200/csrc/Makefile`` (nvcc,
sm_100a). There is no fallback: if it is missing and cannot be built, every
entry point raises.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading

from . import _abi as A

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
# MTCG_LIB_PATH loads another build of the library instead (A/B tuning runs)
LIB_PATH = os.environ.get("MTCG_LIB_PATH") or os.path.join(PKG_DIR, "libmtcg.so")
CSRC = os.path.join(PKG_DIR, "csrc")

_lib = None
_lock = threading.Lock()


class EngineLibraryMissing(RuntimeError):
    pass


def build(force: bool = False) -> str:
    """Compile libmtcg.so in-tree (make -C csrc)."""
    if force and os.path.exists(LIB_PATH):
        os.remove(LIB_PATH)
    subprocess.run(["make", "-s", "-C", CSRC, "-j4"], check=True)
    return LIB_PATH


def lib():
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                try:
                    build()
                except Exception as e:  # noqa: BLE001
                    raise EngineLibraryMissing(
                        f"{LIB_PATH} is missing and could not be built: {e}") from e
            L = C.CDLL(LIB_PATH)
            vp, cp, sz = C.c_void_p, C.c_char_p, C.c_size_t
            pp = C.POINTER(A.mtcg_problem)
            op = C.POINTER(A.mtcg_options)
            rp = C.POINTER(A.mtcg_result)
            ip = C.POINTER(A.mtcg_plan_info)
            u64p, i32p, dp = C.POINTER(C.c_uint64), C.POINTER(C.c_int32), C.POINTER(C.c_double)
            L.mtcg_version.restype = C.c_int
            L.mtcg_create.argtypes = [C.c_int, C.c_uint64, C.POINTER(vp), cp, sz]
            L.mtcg_create_multi.argtypes = [C.POINTER(C.c_int), C.c_int, C.c_uint64, C.POINTER(vp), cp, sz]
            L.mtcg_device_count.argtypes = [vp]
            L.mtcg_device_count.restype = C.c_int32
            L.mtcg_visible_devices.argtypes = []
            L.mtcg_visible_devices.restype = C.c_int32
            L.mtcg_run_slices_out.argtypes = [vp, C.c_uint64, C.c_uint64, vp, vp, cp, sz]
            L.mtcg_fold.argtypes = [vp, vp, C.c_uint64, vp, C.c_int, vp, cp, sz]
            L.mtcg_destroy.argtypes = [vp]
            L.mtcg_destroy.restype = None
            L.mtcg_eval.argtypes = [vp, pp, op, rp, cp, sz]
            L.mtcg_emulate.argtypes = [pp, op, C.c_uint64, ip, u64p, i32p, cp, sz]
            L.mtcg_linear_xeb.argtypes = [vp, C.c_int, dp, C.c_uint64, dp, cp, sz]
            L.mtcg_linear_xeb_amplitudes.argtypes = [vp, C.c_int, dp, C.c_uint64, dp, cp, sz]
            L.mtcg_compile.argtypes = [vp, pp, op, C.POINTER(vp), i32p, cp, sz]
            L.mtcg_plan_destroy.argtypes = [vp]
            L.mtcg_plan_destroy.restype = None
            L.mtcg_plan_get_info.argtypes = [vp, ip]
            L.mtcg_run.argtypes = [vp, C.c_uint64, C.c_uint64, vp, C.c_int, vp, cp, sz]
            L.mtcg_fetch.argtypes = [vp, vp, vp, rp, cp, sz]
            L.mtcg_xeb_device.argtypes = [vp, vp, C.c_int, vp, dp, cp, sz]
            L.mtcg_launch_count.argtypes = [vp]
            L.mtcg_launch_count.restype = C.c_uint64
            L.mtcg_plan_op_count.argtypes = [vp]
            L.mtcg_plan_op_count.restype = C.c_int32
            L.mtcg_plan_op_info.argtypes = [vp, C.c_int32, C.POINTER(A.mtcg_op_info)]
            L.mtcg_time_ops.argtypes = [vp, C.c_uint64, vp, C.c_int, vp, C.POINTER(C.c_float), cp, sz]
            L.mtcg_tuple_index_check.argtypes = [vp, pp, i32p, u64p, dp, dp, cp, sz]
            L.mtcg_read_samples.argtypes = [vp, C.c_uint64, C.c_int32, vp, C.c_uint64, u64p, i32p, cp, sz]
            L.mtcg_assign.argtypes = [vp, C.c_uint64, C.c_int32, C.c_int32, vp, vp, vp, vp, vp, vp,
                                      C.c_uint64, cp, sz]
            L.mtcg_write_amplitudes.argtypes = [cp, vp, C.c_uint64, C.c_int32, C.c_int32, vp, C.c_int32,
                                                u64p, cp, sz]
            _lib = L
        return _lib


# every symbol include/mtcg.h declares
EXPORTS = (
    "mtcg_version", "mtcg_create", "mtcg_destroy", "mtcg_eval", "mtcg_linear_xeb",
    "mtcg_linear_xeb_amplitudes", "mtcg_compile", "mtcg_plan_destroy",
    "mtcg_plan_get_info", "mtcg_run", "mtcg_fetch", "mtcg_xeb_device",
    "mtcg_emulate", "mtcg_launch_count", "mtcg_plan_op_count", "mtcg_plan_op_info",
    "mtcg_time_ops", "mtcg_create_multi", "mtcg_device_count", "mtcg_visible_devices",
    "mtcg_run_slices_out", "mtcg_fold", "mtcg_tuple_index_check",
    "mtcg_read_samples", "mtcg_assign", "mtcg_write_amplitudes",
)
