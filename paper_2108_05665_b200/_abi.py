"""ctypes mirror of include/mtcg.h (the C-ABI boundary) + problem packing.

`ProblemArrays` owns the numpy arrays behind one `mtcg_problem` so the
struct's borrowed pointers stay valid while it lives.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

MTCG_OK = 0
MTCG_ERR_INTERNAL = 1
MTCG_ERR_DATA = 2
MTCG_ERR_MEMORY_CAP = 3
MTCG_ERR_CUDA = 5
MTCG_ERR_ARGUMENT = 6
MTCG_ERR_NCCL = 7
MTCG_ERR_PARSE = 8

MTCG_C64 = 0
MTCG_C128 = 1

MTCG_EVAL_AUTO = 0
MTCG_EVAL_ALL = 1
MTCG_EVAL_SLICED = 2

_i32p = C.POINTER(C.c_int32)
_u32p = C.POINTER(C.c_uint32)
_u64p = C.POINTER(C.c_uint64)
_dp = C.POINTER(C.c_double)


class mtcg_problem(C.Structure):
    _fields_ = [
        ("n_nodes", C.c_int32),
        ("node_left", _i32p),
        ("node_right", _i32p),
        ("node_slot", _i32p),
        ("root", C.c_int32),
        ("n_sliced", C.c_int32),
        ("sliced", _u32p),
        ("n_legs", C.c_uint32),
        ("n_closed", C.c_uint32),
        ("leg_dims", _u32p),
        ("n_slots", C.c_int32),
        ("slot_n_values", _i32p),
        ("slot_leg_begin", _i32p),
        ("slot_legs", _u32p),
        ("values", _dp),
        ("n_requests", C.c_uint64),
        ("tuples", _u32p),
        ("n_batch_legs", C.c_int32),
        ("batch_legs", _u32p),
    ]


class mtcg_options(C.Structure):
    _fields_ = [
        ("eval_mode", C.c_int32),
        ("precision", C.c_int32),
        ("memory_cap_bytes", C.c_uint64),
        ("workers", C.c_int32),
        ("flags", C.c_int32),
        ("row_chunk", C.c_uint64),
    ]


class mtcg_result(C.Structure):
    _fields_ = [
        ("values", _dp),
        ("values_capacity", C.c_uint64),
        ("node_contractions", _u64p),
        ("mults", C.c_uint64),
        ("adds", C.c_uint64),
        ("rw", C.c_uint64),
        ("hbm_peak_bytes", C.c_uint64),
        ("cap_node", C.c_int32),
        ("n_out_legs", C.c_int32),
        ("out_legs", C.c_uint32 * 64),
    ]


class mtcg_op_info(C.Structure):
    """include/mtcg.h mtcg_op_info: one batched launch of a compiled slice."""
    _fields_ = [("node", C.c_int32), ("kernel", C.c_int32), ("fa", C.c_int32),
                ("fb", C.c_int32), ("kc", C.c_int32), ("batch", C.c_uint32),
                ("mults", C.c_uint64), ("bytes", C.c_uint64),
                ("compulsory_bytes", C.c_uint64)]


class mtcg_plan_info(C.Structure):
    _fields_ = [
        ("n_requests", C.c_uint64),
        ("n_rows", C.c_uint64),
        ("row_elems", C.c_uint64),
        ("n_slices", C.c_uint64),
        ("mults", C.c_uint64),
        ("adds", C.c_uint64),
        ("rw", C.c_uint64),
        ("contractions", C.c_uint64),
        ("hbm_arena_bytes", C.c_uint64),
        ("hbm_resident_bytes", C.c_uint64),
        ("precision", C.c_int32),
        ("n_kernels_per_slice", C.c_int32),
        ("prologue_ops", C.c_uint64),
        ("executed_contractions", C.c_uint64),
        ("fused_chains", C.c_uint64),
        ("fused_ops", C.c_uint64),
    ]


def _p(a: np.ndarray, ct):
    return a.ctypes.data_as(C.POINTER(ct))


@dataclass
class ProblemArrays:
    """The engine's inputs as flat arrays (field meaning: include/mtcg.h)."""

    node_left: np.ndarray
    node_right: np.ndarray
    node_slot: np.ndarray
    root: int
    sliced: np.ndarray
    n_closed: int
    leg_dims: np.ndarray
    slot_n_values: np.ndarray
    slot_leg_begin: np.ndarray
    slot_legs: np.ndarray
    values: np.ndarray          # complex128, flat
    tuples: np.ndarray          # (n_requests, n_slots) uint32
    batch_legs: np.ndarray
    _struct: Optional[mtcg_problem] = field(default=None, repr=False)

    def __post_init__(self):
        self.node_left = np.ascontiguousarray(self.node_left, dtype=np.int32)
        self.node_right = np.ascontiguousarray(self.node_right, dtype=np.int32)
        self.node_slot = np.ascontiguousarray(self.node_slot, dtype=np.int32)
        self.sliced = np.ascontiguousarray(self.sliced, dtype=np.uint32)
        self.leg_dims = np.ascontiguousarray(self.leg_dims, dtype=np.uint32)
        self.slot_n_values = np.ascontiguousarray(self.slot_n_values, dtype=np.int32)
        self.slot_leg_begin = np.ascontiguousarray(self.slot_leg_begin, dtype=np.int32)
        self.slot_legs = np.ascontiguousarray(self.slot_legs, dtype=np.uint32)
        self.values = np.ascontiguousarray(self.values, dtype=np.complex128).ravel()
        self.tuples = np.ascontiguousarray(self.tuples, dtype=np.uint32)
        if self.tuples.ndim != 2:
            self.tuples = self.tuples.reshape(-1, len(self.slot_n_values))
        self.batch_legs = np.ascontiguousarray(self.batch_legs, dtype=np.uint32)

    @property
    def n_nodes(self) -> int:
        return len(self.node_left)

    @property
    def n_slots(self) -> int:
        return len(self.slot_n_values)

    @property
    def n_requests(self) -> int:
        return self.tuples.shape[0]

    @property
    def n_legs(self) -> int:
        return len(self.leg_dims)

    @property
    def row_elems(self) -> int:
        return 1 << len(self.batch_legs)

    def struct(self) -> mtcg_problem:
        if self._struct is None:
            s = mtcg_problem()
            s.n_nodes = self.n_nodes
            s.node_left = _p(self.node_left, C.c_int32)
            s.node_right = _p(self.node_right, C.c_int32)
            s.node_slot = _p(self.node_slot, C.c_int32)
            s.root = self.root
            s.n_sliced = len(self.sliced)
            s.sliced = _p(self.sliced, C.c_uint32)
            s.n_legs = self.n_legs
            s.n_closed = self.n_closed
            s.leg_dims = _p(self.leg_dims, C.c_uint32)
            s.n_slots = self.n_slots
            s.slot_n_values = _p(self.slot_n_values, C.c_int32)
            s.slot_leg_begin = _p(self.slot_leg_begin, C.c_int32)
            s.slot_legs = _p(self.slot_legs, C.c_uint32)
            s.values = self.values.view(np.float64).ctypes.data_as(_dp)
            s.n_requests = self.n_requests
            s.tuples = _p(self.tuples, C.c_uint32)
            s.n_batch_legs = len(self.batch_legs)
            s.batch_legs = _p(self.batch_legs, C.c_uint32)
            self._struct = s
        return self._struct

    def with_plan(self, node_left, node_right, node_slot, root, sliced) -> "ProblemArrays":
        return ProblemArrays(node_left, node_right, node_slot, root, sliced,
                             self.n_closed, self.leg_dims, self.slot_n_values,
                             self.slot_leg_begin, self.slot_legs, self.values,
                             self.tuples, self.batch_legs)

    @staticmethod
    def build(plan_nodes: Sequence, root: int, sliced: Sequence[int], n_closed: int,
              leg_dims: Sequence[int], value_sets: Sequence, tuples,
              batch_legs: Sequence[int]) -> "ProblemArrays":
        """plan_nodes: [(left, right, slot)], value_sets: [(legs, data[nv, size])]."""
        nl = np.array([n[0] for n in plan_nodes], dtype=np.int32)
        nr = np.array([n[1] for n in plan_nodes], dtype=np.int32)
        ns = np.array([n[2] for n in plan_nodes], dtype=np.int32)
        nv, begin, legs, data = [], [0], [], []
        for lg, d in value_sets:
            d = np.asarray(d, dtype=np.complex128)
            d = d.reshape(-1, 1 << len(lg)) if len(lg) or d.size else d.reshape(-1, 1)
            nv.append(d.shape[0])
            legs.extend(lg)
            begin.append(len(legs))
            data.append(d.ravel())
        vals = np.concatenate(data) if data else np.zeros(0, np.complex128)
        t = np.asarray(tuples, dtype=np.uint32).reshape(-1, len(value_sets))
        return ProblemArrays(nl, nr, ns, root, list(sliced), n_closed, list(leg_dims),
                             nv, begin, legs, vals, t, sorted(batch_legs))
