"""ORACLE TEST INFRASTRUCTURE — ctypes driver for the UNMODIFIED reference.

Loads ``oracle/_ref/libmtcref.so`` (the reference ``mtc`` library compiled from
/root/reference/proj/src by ``oracle/Makefile`` plus the glue in
``oracle/ref_shim.cpp``). Only tests, golden-vector generators and the bench's
CPU-baseline leg may use this module; the product never imports it.

Everything here forwards to the reference's public API; see ref_shim.cpp for
the file:line of each entry point.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import List, Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_ref", "libmtcref.so")

_lib = None


def available() -> bool:
    return os.path.exists(LIB_PATH)


def lib():
    global _lib
    if _lib is None:
        if not available():
            raise RuntimeError(f"reference library not built: {LIB_PATH}")
        L = C.CDLL(LIB_PATH)
        vp, u32p, u64p, dp, ip = (C.c_void_p, C.POINTER(C.c_uint32),
                                  C.POINTER(C.c_uint64), C.POINTER(C.c_double),
                                  C.POINTER(C.c_int))
        L.ref_last_error.restype = C.c_char_p
        L.ref_free.argtypes = [vp]
        L.ref_problem_new.restype = vp
        L.ref_problem_new.argtypes = [C.c_char_p, C.c_int, C.c_char_p, C.c_char_p]
        L.ref_problem_free.argtypes = [vp]
        L.ref_read_samples.argtypes = [C.c_char_p, C.c_uint64, C.c_int, vp, C.c_uint64, u64p, ip]
        L.ref_format_amplitude_row.argtypes = [C.c_char_p, C.c_double, C.c_double, C.c_int, vp, C.c_uint64]
        L.ref_set_plan.argtypes = [vp, C.c_char_p]
        L.ref_plan_text.restype = vp
        L.ref_plan_text.argtypes = [vp]
        for name in ("ref_n_qubits", "ref_n_slots", "ref_plan_root"):
            getattr(L, name).argtypes = [vp]
        L.ref_n_closed.restype = C.c_uint32
        L.ref_n_closed.argtypes = [vp]
        L.ref_n_legs.restype = C.c_uint32
        L.ref_n_legs.argtypes = [vp]
        L.ref_slot_tensor.argtypes = [vp, C.c_int, u32p, dp]
        L.ref_slot_n_values.argtypes = [vp, C.c_int]
        L.ref_slot_values.argtypes = [vp, C.c_int, u32p, dp]
        L.ref_n_requests.restype = C.c_uint64
        L.ref_n_requests.argtypes = [vp]
        L.ref_tuples.argtypes = [vp, u32p]
        L.ref_batch_legs.argtypes = [vp, u32p]
        L.ref_plan_nodes.argtypes = [vp, ip, ip, ip]
        L.ref_plan_sliced.argtypes = [vp, u32p]
        L.ref_eval.argtypes = [vp, C.c_int, C.c_int, C.c_uint64, dp, u64p, u64p,
                               u64p, ip]
        L.ref_eval_slice.argtypes = [vp, C.c_uint64, dp]
        L.ref_eval_slices_parallel.argtypes = [vp, C.c_uint64, C.c_uint64, C.c_int]
        L.ref_emulate.argtypes = [vp, C.c_uint64, u64p, u64p, u64p]
        L.ref_exact_totals.argtypes = [vp, u64p, u64p, u64p, u64p, u64p]
        L.ref_grid_circuit.restype = vp
        L.ref_grid_circuit.argtypes = [C.c_int, C.c_int, C.c_int, C.c_uint64]
        L.ref_random_circuit.restype = vp
        L.ref_random_circuit.argtypes = [C.c_uint64, C.c_int, C.c_int]
        L.ref_random_bitstrings.restype = vp
        L.ref_random_bitstrings.argtypes = [C.c_uint64, C.c_int, C.c_int]
        L.ref_left_deep_plan.restype = vp
        L.ref_left_deep_plan.argtypes = [C.c_int]
        L.ref_anneal.restype = vp
        L.ref_anneal.argtypes = [vp, C.c_uint64, C.c_uint64, C.c_double, C.c_double,
                                 C.c_double, C.c_uint64, C.c_uint64, C.c_uint64,
                                 C.c_uint32, dp]
        L.ref_add_slices_greedy.argtypes = [vp, C.c_int, C.c_uint64, C.c_uint64,
                                            C.c_int]
        L.ref_sample_eval_time.argtypes = [vp, C.c_uint64, C.c_int, dp, dp, dp]
        L.ref_statevector.argtypes = [C.c_char_p, C.c_char_p, dp]
        L.ref_linear_xeb.argtypes = [C.c_int, dp, C.c_uint64, dp]
        L.ref_xeb_from_amplitudes.argtypes = [C.c_int, dp, C.c_uint64, dp]
        _lib = L
    return _lib


class RefError(Exception):
    def __init__(self, code: int, msg: str, node: int = -1):
        super().__init__(msg)
        self.code = code
        self.node = node


def _take_string(ptr) -> str:
    s = C.cast(ptr, C.c_char_p).value.decode()
    lib().ref_free(ptr)
    return s


def _ptr(a, ct):
    return a.ctypes.data_as(C.POINTER(ct))


def grid_circuit(rows: int, cols: int, layers: int, seed: int) -> str:
    return _take_string(lib().ref_grid_circuit(rows, cols, layers, seed))


def random_circuit(seed: int, n_qubits: int, n_gates: int) -> str:
    return _take_string(lib().ref_random_circuit(seed, n_qubits, n_gates))


def random_bitstrings(seed: int, n_qubits: int, count: int) -> List[str]:
    return _take_string(lib().ref_random_bitstrings(seed, n_qubits, count)).split()


def left_deep_plan(n_slots: int) -> str:
    return _take_string(lib().ref_left_deep_plan(n_slots))


def statevector(circuit: str, bits: Sequence[str]) -> np.ndarray:
    out = np.zeros(2 * len(bits), dtype=np.float64)
    rc = lib().ref_statevector(circuit.encode(), "\n".join(bits).encode(),
                               _ptr(out, C.c_double))
    if rc:
        raise RefError(rc, lib().ref_last_error().decode())
    return out.view(np.complex128)


def linear_xeb(n: int, probs: np.ndarray) -> float:
    p = np.ascontiguousarray(probs, dtype=np.float64)
    out = C.c_double()
    rc = lib().ref_linear_xeb(n, _ptr(p, C.c_double), p.size, C.byref(out))
    if rc:
        raise RefError(rc, lib().ref_last_error().decode())
    return out.value


def read_samples(text: bytes, order: int = 0) -> List[str]:
    """The reference's read_samples (formats.cpp:42-69); RefError(code 4 =
    ParseError) with its message on failure."""
    buf = C.create_string_buffer(max(len(text), 1))
    n, nq = C.c_uint64(0), C.c_int(0)
    rc = lib().ref_read_samples(text, len(text), order, buf, len(buf), C.byref(n), C.byref(nq))
    if rc:
        raise RefError(rc, lib().ref_last_error().decode())
    raw = buf.raw[: n.value * nq.value].decode()
    return [raw[i * nq.value:(i + 1) * nq.value] for i in range(n.value)]


def format_amplitude_row(bits: str, amp: complex, order: int = 0) -> str:
    out = C.create_string_buffer(len(bits) + 128)
    lib().ref_format_amplitude_row(bits.encode(), amp.real, amp.imag, order, out, len(out))
    return out.value.decode()


class RefProblem:
    """circuit text + fuse + bitstrings (+ plan text) -> reference objects."""

    def __init__(self, circuit: str, bits: Sequence[str], plan: Optional[str] = None,
                 fuse: bool = True):
        self.h = lib().ref_problem_new(circuit.encode(), int(fuse),
                                       "\n".join(bits).encode(),
                                       (plan or "").encode())
        if not self.h:
            raise RefError(2, lib().ref_last_error().decode())
        self.bits = list(bits)

    def __del__(self):
        if getattr(self, "h", None):
            lib().ref_problem_free(self.h)
            self.h = None

    def set_plan(self, plan: str) -> None:
        rc = lib().ref_set_plan(self.h, plan.encode())
        if rc:
            raise RefError(rc, lib().ref_last_error().decode())

    def plan_text(self) -> str:
        return _take_string(lib().ref_plan_text(self.h))

    @property
    def n_qubits(self) -> int:
        return lib().ref_n_qubits(self.h)

    @property
    def n_closed(self) -> int:
        return lib().ref_n_closed(self.h)

    @property
    def n_legs(self) -> int:
        return lib().ref_n_legs(self.h)

    @property
    def n_slots(self) -> int:
        return lib().ref_n_slots(self.h)

    @property
    def n_requests(self) -> int:
        return lib().ref_n_requests(self.h)

    def slot_tensor(self, j: int):
        L = lib()
        r = L.ref_slot_tensor(self.h, j, None, None)
        legs = np.zeros(max(r, 1), dtype=np.uint32)
        data = np.zeros(2 << r, dtype=np.float64)
        L.ref_slot_tensor(self.h, j, _ptr(legs, C.c_uint32), _ptr(data, C.c_double))
        return legs[:r].tolist(), data.view(np.complex128)

    def value_set(self, j: int):
        L = lib()
        r = L.ref_slot_values(self.h, j, None, None)
        nv = L.ref_slot_n_values(self.h, j)
        legs = np.zeros(max(r, 1), dtype=np.uint32)
        data = np.zeros(2 * nv << r, dtype=np.float64)
        L.ref_slot_values(self.h, j, _ptr(legs, C.c_uint32), _ptr(data, C.c_double))
        return legs[:r].tolist(), data.view(np.complex128).reshape(nv, 1 << r)

    def tuples(self) -> np.ndarray:
        t = np.zeros((self.n_requests, self.n_slots), dtype=np.uint32)
        if t.size:
            lib().ref_tuples(self.h, _ptr(t, C.c_uint32))
        return t

    def batch_legs(self) -> List[int]:
        L = lib()
        n = L.ref_batch_legs(self.h, None)
        b = np.zeros(max(n, 1), dtype=np.uint32)
        L.ref_batch_legs(self.h, _ptr(b, C.c_uint32))
        return b[:n].tolist()

    def plan_nodes(self):
        L = lib()
        n = L.ref_plan_nodes(self.h, None, None, None)
        l, r, s = (np.zeros(n, dtype=np.int32) for _ in range(3))
        L.ref_plan_nodes(self.h, _ptr(l, C.c_int), _ptr(r, C.c_int), _ptr(s, C.c_int))
        return l, r, s, L.ref_plan_root(self.h)

    def plan_sliced(self) -> List[int]:
        L = lib()
        n = L.ref_plan_sliced(self.h, None)
        b = np.zeros(max(n, 1), dtype=np.uint32)
        L.ref_plan_sliced(self.h, _ptr(b, C.c_uint32))
        return b[:n].tolist()

    def eval(self, mode: str = "auto", workers: int = 1, cap: int = 0):
        """mode: all | sliced | naive | auto. Returns (values, node_counts,
        counters(mults, adds, rw), peak_bytes)."""
        m = {"all": 0, "sliced": 1, "naive": 2, "auto": 3}[mode]
        w = len(self.batch_legs())
        vals = np.zeros(2 * self.n_requests << w, dtype=np.float64)
        n_nodes = len(self.plan_nodes()[0])
        nc = np.zeros(max(n_nodes, 1), dtype=np.uint64)
        cnt = np.zeros(3, dtype=np.uint64)
        peak = C.c_uint64()
        node = C.c_int(-1)
        rc = lib().ref_eval(self.h, m, workers, cap, _ptr(vals, C.c_double),
                            _ptr(nc, C.c_uint64), _ptr(cnt, C.c_uint64),
                            C.byref(peak), C.byref(node))
        if rc:
            raise RefError(rc, lib().ref_last_error().decode(), node.value)
        v = vals.view(np.complex128).reshape(self.n_requests, 1 << w)
        return v, nc[:n_nodes], tuple(int(x) for x in cnt), peak.value

    def eval_slice(self, idx: int) -> np.ndarray:
        w = len(self.batch_legs())
        vals = np.zeros(2 * self.n_requests << w, dtype=np.float64)
        rc = lib().ref_eval_slice(self.h, idx, _ptr(vals, C.c_double))
        if rc:
            raise RefError(rc, lib().ref_last_error().decode())
        return vals.view(np.complex128).reshape(self.n_requests, 1 << w)

    def eval_slices_parallel(self, first: int, n: int, threads: int) -> None:
        rc = lib().ref_eval_slices_parallel(self.h, first, n, threads)
        if rc:
            raise RefError(rc, lib().ref_last_error().decode())

    def emulate(self, cap: int = 0):
        n_nodes = len(self.plan_nodes()[0])
        nc = np.zeros(max(n_nodes, 1), dtype=np.uint64)
        cnt = np.zeros(3, dtype=np.uint64)
        peak = C.c_uint64()
        rc = lib().ref_emulate(self.h, cap, _ptr(cnt, C.c_uint64), C.byref(peak),
                               _ptr(nc, C.c_uint64))
        if rc:
            raise RefError(rc, lib().ref_last_error().decode())
        return tuple(int(x) for x in cnt), peak.value, nc[:n_nodes]

    def exact_totals(self):
        n_nodes = len(self.plan_nodes()[0])
        m, a, r = (np.zeros(2, dtype=np.uint64) for _ in range(3))
        kt = np.zeros(max(n_nodes, 1), dtype=np.uint64)
        sz = np.zeros(max(n_nodes, 1), dtype=np.uint64)
        rc = lib().ref_exact_totals(self.h, _ptr(m, C.c_uint64), _ptr(a, C.c_uint64),
                                    _ptr(r, C.c_uint64), _ptr(kt, C.c_uint64),
                                    _ptr(sz, C.c_uint64))
        if rc:
            raise RefError(rc, lib().ref_last_error().decode())
        j = lambda x: (int(x[0]) << 64) | int(x[1])
        return {"mults": j(m), "adds": j(a), "rw": j(r),
                "k_t": kt[:n_nodes], "size": sz[:n_nodes]}

    def sample_eval_time(self, budget: int = 1 << 24, threads: int = 1):
        """-> (single-thread-equivalent seconds of the full evaluation,
        sampling wall seconds, fraction of per-slice MACs actually executed)."""
        est, wall, frac = C.c_double(), C.c_double(), C.c_double()
        rc = lib().ref_sample_eval_time(self.h, budget, threads, C.byref(est),
                                        C.byref(wall), C.byref(frac))
        if rc:
            raise RefError(rc, lib().ref_last_error().decode())
        return est.value, wall.value, frac.value

    def add_slices_greedy(self, n: int, k: int, m_max: int = 8 << 30,
                          criterion: str = "cost") -> None:
        crit = {"memory": 0, "cost": 1}[criterion]
        rc = lib().ref_add_slices_greedy(self.h, n, k, m_max, crit)
        if rc:
            raise RefError(rc, lib().ref_last_error().decode())

    def anneal(self, k: int, m_max: int = 8 << 30, steps: int = 200000,
               slice_interval: int = 100000, seed: int = 0, chains: int = 1,
               alpha: float = 16.0, beta: float = 8.0, p: float = 4.0):
        obj = C.c_double()
        ptr = lib().ref_anneal(self.h, k, m_max, alpha, beta, p, steps,
                               slice_interval, seed, chains, C.byref(obj))
        if not ptr:
            raise RefError(2, lib().ref_last_error().decode())
        return _take_string(ptr), obj.value


def to_arrays(p: RefProblem):
    """The reference's (Plan, NetworkDiagram, AssignmentSet) as the flat
    mtcg_problem arrays both the product and the C oracle consume."""
    from paper_2108_05665_b200._abi import ProblemArrays

    l, r, s, root = p.plan_nodes()
    vs = [p.value_set(j) for j in range(p.n_slots)]
    return ProblemArrays.build(list(zip(l.tolist(), r.tolist(), s.tolist())), root,
                               p.plan_sliced(), p.n_closed, [2] * p.n_legs, vs,
                               p.tuples(), p.batch_legs())
