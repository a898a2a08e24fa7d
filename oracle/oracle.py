"""ORACLE TEST INFRASTRUCTURE — ctypes wrapper for the C restatement.

``oracle/liboracle.so`` (built from oracle/mtc_oracle.c by oracle/Makefile)
evaluates the same ``mtcg_problem`` the product consumes, in complex128 with
the reference's reduction order. Tests, smoke() and bench.py's CPU baseline
only — never the product path.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

from paper_2108_05665_b200._abi import ProblemArrays, mtcg_problem

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None


class OracleError(Exception):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


def build() -> None:
    subprocess.run(["make", "-s", "-C", _HERE, "oracle"], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = C.CDLL(LIB_PATH)
        u64p, dp, i32p = C.POINTER(C.c_uint64), C.POINTER(C.c_double), C.POINTER(C.c_int32)
        L.orc_eval.argtypes = [C.POINTER(mtcg_problem), C.c_int, dp, C.c_uint64, u64p,
                               u64p, i32p, i32p, C.c_char_p, C.c_size_t]
        L.orc_eval_slices.argtypes = [C.POINTER(mtcg_problem), C.c_int, C.c_uint64,
                                      C.c_uint64, dp, C.c_uint64, u64p, u64p, i32p, i32p,
                                      C.c_char_p, C.c_size_t]
        L.orc_linear_xeb.argtypes = [C.c_int, dp, C.c_uint64, dp, C.c_char_p, C.c_size_t]
        _lib = L
    return _lib


def eval_problem(p: ProblemArrays, mode: int = 0, slices=None):
    """-> (values[n_requests, 2^w] complex128, node_contractions, (mults, adds, rw),
    out_legs). slices=(s0, s1) folds only that slice range."""
    w = p.row_elems
    vals = np.zeros(2 * p.n_requests * w, dtype=np.float64)
    nc = np.zeros(max(p.n_nodes, 1), dtype=np.uint64)
    cnt = np.zeros(3, dtype=np.uint64)
    legs = np.zeros(64, dtype=np.int32)
    nlegs = C.c_int32(0)
    err = C.create_string_buffer(512)
    s0, s1 = slices if slices is not None else (0, 2 ** 64 - 1)
    rc = lib().orc_eval_slices(C.byref(p.struct()), mode, s0, s1,
                        vals.ctypes.data_as(C.POINTER(C.c_double)), p.n_requests * w,
                        nc.ctypes.data_as(C.POINTER(C.c_uint64)),
                        cnt.ctypes.data_as(C.POINTER(C.c_uint64)),
                        legs.ctypes.data_as(C.POINTER(C.c_int32)), C.byref(nlegs),
                        err, 512)
    if rc:
        raise OracleError(rc, err.value.decode())
    return (vals.view(np.complex128).reshape(p.n_requests, w), nc[:p.n_nodes],
            tuple(int(x) for x in cnt), legs[:nlegs.value].tolist())


def linear_xeb(n: int, probs) -> float:
    p = np.ascontiguousarray(probs, dtype=np.float64)
    out = C.c_double()
    err = C.create_string_buffer(256)
    rc = lib().orc_linear_xeb(n, p.ctypes.data_as(C.POINTER(C.c_double)), p.size,
                              C.byref(out), err, 256)
    if rc:
        raise OracleError(rc, err.value.decode())
    return out.value
