"""Python face of the B200 engine, mirroring the reference's hot-path API.

    eval_all(plan, d, as, opts)      multieval.hpp:62-63
    eval_sliced(plan, d, as, opts)   multieval.hpp:69-70
    emulate(plan, d, as, opts)       multieval.hpp:74-75 (host-side, exact counts)
    linear_xeb(n, probs)             xeb.hpp:38
    probs_from_amplitudes(amps)      xeb.hpp:42-43

Every call crosses the C ABI of ``libmtcg.so`` (include/mtcg.h); there is no
CPU fallback. `Engine` additionally exposes the staged API (compile once, run
slice ranges into a device accumulator, fetch / fused XEB) used by the bench
and the multi-GPU slice scheduler.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import List, Optional, Sequence

import numpy as np

from . import _abi as A
from ._lib import lib
from .errors import DataError, EngineError, MemoryCapError, ParseError

PRECISIONS = {"c64": A.MTCG_C64, "c128": A.MTCG_C128}


@dataclass
class Tensor:
    """A request's result tensor (tensor.hpp:55-87): row-major over `legs`
    (the batch legs, ascending; none for a single amplitude)."""

    legs: List[int]
    data: np.ndarray


@dataclass
class EvalOptions:
    """EvalOptions (multieval.hpp:26-29) plus the device precision."""

    memory_cap_bytes: int = 0
    workers: int = 1
    precision: str = "c64"
    tensor_cores: bool = True  # dense complex64 ops on tcgen05 (split-integer GEMM)
    # evaluate slice-invariant subtrees once per run instead of once per slice
    # (MTCG_FLAG_SLICE_REUSE; same values, reference counters)
    slice_reuse: bool = False
    # memo streaming: requests in lexicographic chunks of this many (one-shot
    # eval; 0 = all at once)
    row_chunk: int = 0
    # tuple index (plan.cpp:292-333): None = the GPU from 2^15 requests up,
    # else the host; True / False force the GPU (MTCG_FLAG_DEVICE_INDEX) / the
    # host (MTCG_FLAG_HOST_INDEX). Same rows, ranks and pairs either way.
    device_index: Optional[bool] = None


@dataclass
class OpCounters:
    mults: int = 0
    adds: int = 0
    rw: int = 0


class EvalResult:
    """EvalResult (multieval.hpp:36-41). `values[i]` is request i's tensor;
    `amplitudes` is the same data as an (n_requests, 2^w) array. The per-
    request Tensor objects are built on first access of `values` (10^4
    Python objects per fetch otherwise dominate — and, through GC, spike —
    the host side of an end-to-end evaluation)."""

    def __init__(self, out_legs: List[int], counters: OpCounters, peak_bytes: int,
                 node_contractions: np.ndarray, amplitudes: np.ndarray):
        self.out_legs = list(out_legs)
        self.counters = counters
        self.peak_bytes = peak_bytes
        self.node_contractions = node_contractions
        self.amplitudes = amplitudes
        self._values: Optional[List[Tensor]] = None

    @property
    def values(self) -> List[Tensor]:
        if self._values is None:
            self._values = [Tensor(list(self.out_legs), self.amplitudes[i])
                            for i in range(self.amplitudes.shape[0])]
        return self._values

    def __repr__(self) -> str:
        return (f"EvalResult(n={self.amplitudes.shape[0]}, counters={self.counters}, "
                f"peak_bytes={self.peak_bytes})")


@dataclass
class EmulateResult:
    counters: OpCounters
    peak_bytes: int
    node_contractions: np.ndarray
    contractions: int = 0
    plan_info: Optional[A.mtcg_plan_info] = None  # schedule facts (prologue, fused chains)


def _raise(status: int, err: C.Array, cap_node: int = -1):
    msg = err.value.decode(errors="replace")
    if status == A.MTCG_ERR_DATA:
        raise DataError(msg)
    if status == A.MTCG_ERR_MEMORY_CAP:
        raise MemoryCapError(msg, cap_node)
    if status == A.MTCG_ERR_PARSE:
        raise ParseError(msg)
    raise EngineError(f"mtcg status {status}: {msg}")


def problem_arrays(plan, d, assignments) -> A.ProblemArrays:
    """Pack reference-shaped inputs (a Plan, a NetworkDiagram and an
    AssignmentSet: plan.hpp:33-45, diagram.hpp:32-68 — e.g. workloads.network's
    restatements) into the C ABI's POD arrays."""
    vs = [(s[0].legs, np.stack([t.data for t in s])) for s in assignments.value_sets]
    nodes = list(zip(plan.left, plan.right, plan.slot))
    return A.ProblemArrays.build(nodes, plan.root, plan.sliced, d.n_closed, d.leg_dims, vs,
                                 assignments.tuples, assignments.batch_legs)


def _options(mode: int, opts: Optional[EvalOptions]) -> A.mtcg_options:
    opts = opts or EvalOptions()
    o = A.mtcg_options()
    o.eval_mode = mode
    if opts.precision not in PRECISIONS:
        raise DataError(f"unknown precision '{opts.precision}'")
    o.precision = PRECISIONS[opts.precision]
    o.memory_cap_bytes = int(opts.memory_cap_bytes)
    o.workers = int(opts.workers)
    o.flags = ((0 if opts.tensor_cores else 1) | (2 if opts.slice_reuse else 0)
               | {None: 0, True: 8, False: 4}[opts.device_index])  # MTCG_FLAG_*
    o.row_chunk = int(opts.row_chunk)
    return o


class CompiledProblem:
    """A problem compiled and resident on one device (mtcg_compile)."""

    def __init__(self, engine: "Engine", handle: C.c_void_p, problem: A.ProblemArrays):
        self.engine = engine
        self.h = handle
        self.problem = problem
        info = A.mtcg_plan_info()
        lib().mtcg_plan_get_info(self.h, C.byref(info))
        self.info = info

    def __del__(self):
        if getattr(self, "h", None):
            lib().mtcg_plan_destroy(self.h)
            self.h = None

    @property
    def n_slices(self) -> int:
        return int(self.info.n_slices)

    @property
    def complex_dtype_bytes(self) -> int:
        return 8 if self.info.precision == A.MTCG_C64 else 16

    def new_accumulator(self, device=None):
        """A zeroed torch device buffer for mtcg_run: (rows, 2^w, 2) reals."""
        import torch

        dt = torch.float32 if self.info.precision == A.MTCG_C64 else torch.float64
        dev = device if device is not None else torch.device("cuda", self.engine.device)
        return torch.zeros((max(int(self.info.n_rows), 1), int(self.info.row_elems), 2),
                           dtype=dt, device=dev)

    def run(self, slice_begin: int, slice_end: int, acc_ptr: int, accumulate: bool = False,
            stream: int = 0) -> None:
        err = C.create_string_buffer(1024)
        st = lib().mtcg_run(self.h, slice_begin, slice_end, C.c_void_p(acc_ptr),
                            int(accumulate), C.c_void_p(stream or None), err, 1024)
        if st:
            _raise(st, err)

    def fetch(self, acc_ptr: int, stream: int = 0, node_contractions: bool = True):
        p = self.problem
        w = int(self.info.row_elems)
        vals = np.zeros(2 * p.n_requests * w, dtype=np.float64)
        nc = np.zeros(max(p.n_nodes, 1), dtype=np.uint64)
        res = A.mtcg_result()
        res.values = vals.ctypes.data_as(C.POINTER(C.c_double))
        res.values_capacity = p.n_requests * w
        res.node_contractions = nc.ctypes.data_as(C.POINTER(C.c_uint64)) if node_contractions else None
        err = C.create_string_buffer(1024)
        st = lib().mtcg_fetch(self.h, C.c_void_p(acc_ptr), C.c_void_p(stream or None),
                              C.byref(res), err, 1024)
        if st:
            _raise(st, err)
        return _result_from(res, vals, nc[:p.n_nodes], p.n_requests, w)

    def run_slices_out(self, slice_begin: int, slice_end: int, out_ptr: int, stream: int = 0) -> None:
        """Each slice's root values (no fold) into consecutive blocks of
        out_ptr (new_accumulator-shaped blocks): the per-rank half of a
        deterministic multi-GPU evaluation (mtcg_run_slices_out)."""
        err = C.create_string_buffer(1024)
        st = lib().mtcg_run_slices_out(self.h, slice_begin, slice_end, C.c_void_p(out_ptr),
                                       C.c_void_p(stream or None), err, 1024)
        if st:
            _raise(st, err)

    def fold(self, parts_ptr: int, n_parts: int, acc_ptr: int, accumulate: bool = False,
             stream: int = 0) -> None:
        """acc = (acc if accumulate else parts[0]) + parts[1] + ... in order
        (mtcg_fold: the reference's slice fold)."""
        err = C.create_string_buffer(1024)
        st = lib().mtcg_fold(self.h, C.c_void_p(parts_ptr), n_parts, C.c_void_p(acc_ptr),
                             int(accumulate), C.c_void_p(stream or None), err, 1024)
        if st:
            _raise(st, err)

    def new_slice_buffer(self, n_slices: int):
        """Device buffer for n_slices per-slice root tensors."""
        import torch

        dt = torch.float32 if self.info.precision == A.MTCG_C64 else torch.float64
        return torch.zeros((max(n_slices, 1), max(int(self.info.n_rows), 1), int(self.info.row_elems), 2),
                           dtype=dt, device=torch.device("cuda", self.engine.device))

    def op_infos(self):
        """Per-op introspection (mtcg_plan_op_info), in launch order."""
        L = lib()
        out = []
        for i in range(L.mtcg_plan_op_count(self.h)):
            oi = A.mtcg_op_info()
            L.mtcg_plan_op_info(self.h, i, C.byref(oi))
            out.append(oi)
        return out

    def op_kernels(self):
        """Kernel configuration of every op (12: tcgen05 tensor-core GEMM)."""
        return [oi.kernel for oi in self.op_infos()]

    def xeb(self, acc_ptr: int, n_qubits: int, stream: int = 0) -> float:
        out = C.c_double()
        err = C.create_string_buffer(1024)
        st = lib().mtcg_xeb_device(self.h, C.c_void_p(acc_ptr), n_qubits,
                                   C.c_void_p(stream or None), C.byref(out), err, 1024)
        if st:
            _raise(st, err)
        return out.value


def _result_from(res: A.mtcg_result, vals: np.ndarray, nc: np.ndarray, n_req: int,
                 w: int) -> EvalResult:
    amps = vals.view(np.complex128).reshape(n_req, w)
    legs = [int(res.out_legs[i]) for i in range(res.n_out_legs)]
    return EvalResult(legs, OpCounters(int(res.mults), int(res.adds), int(res.rw)),
                      int(res.hbm_peak_bytes), nc.copy(), amps)


class Engine:
    """An mtcg handle bound to one CUDA device, or to several (``devices``:
    mtcg_create_multi — eval() then spreads slices over the first
    min(EvalOptions.workers, len(devices)) of them, bit-identical to one
    device; repeats share a GPU)."""

    def __init__(self, device: int = 0, hbm_cap_bytes: int = 0, devices=None):
        devs = list(devices) if devices is not None else [device]
        self.device = devs[0]
        self.devices = devs
        h = C.c_void_p()
        err = C.create_string_buffer(1024)
        arr = (C.c_int * len(devs))(*devs)
        st = lib().mtcg_create_multi(arr, len(devs), hbm_cap_bytes, C.byref(h), err, 1024)
        if st:
            _raise(st, err)
        self.h = h

    def __del__(self):
        if getattr(self, "h", None):
            lib().mtcg_destroy(self.h)
            self.h = None

    @property
    def launches(self) -> int:
        return int(lib().mtcg_launch_count(self.h))

    def eval(self, problem: A.ProblemArrays, mode: int = A.MTCG_EVAL_AUTO,
             opts: Optional[EvalOptions] = None) -> EvalResult:
        o = _options(mode, opts)
        w = problem.row_elems
        vals = np.zeros(2 * problem.n_requests * w, dtype=np.float64)
        nc = np.zeros(max(problem.n_nodes, 1), dtype=np.uint64)
        res = A.mtcg_result()
        res.values = vals.ctypes.data_as(C.POINTER(C.c_double))
        res.values_capacity = problem.n_requests * w
        res.node_contractions = nc.ctypes.data_as(C.POINTER(C.c_uint64))
        err = C.create_string_buffer(1024)
        st = lib().mtcg_eval(self.h, C.byref(problem.struct()), C.byref(o), C.byref(res),
                             err, 1024)
        if st:
            _raise(st, err, res.cap_node)
        return _result_from(res, vals, nc[:problem.n_nodes], problem.n_requests, w)

    def compile(self, problem: A.ProblemArrays, mode: int = A.MTCG_EVAL_AUTO,
                opts: Optional[EvalOptions] = None) -> CompiledProblem:
        o = _options(mode, opts)
        h = C.c_void_p()
        cap_node = C.c_int32(-1)
        err = C.create_string_buffer(1024)
        st = lib().mtcg_compile(self.h, C.byref(problem.struct()), C.byref(o), C.byref(h),
                                C.byref(cap_node), err, 1024)
        if st:
            _raise(st, err, cap_node.value)
        return CompiledProblem(self, h, problem)

    def tuple_index_check(self, problem: A.ProblemArrays):
        """Build the tuple index on the host and on this GPU and compare them
        (mtcg_tuple_index_check). Returns (equal, rows, host_ms, device_ms)."""
        eq, rows = C.c_int32(0), C.c_uint64(0)
        hm, dm = C.c_double(0), C.c_double(0)
        err = C.create_string_buffer(1024)
        st = lib().mtcg_tuple_index_check(self.h, C.byref(problem.struct()), C.byref(eq), C.byref(rows),
                                          C.byref(hm), C.byref(dm), err, 1024)
        if st:
            _raise(st, err)
        return bool(eq.value), int(rows.value), hm.value, dm.value

    def linear_xeb(self, n: int, probs) -> float:
        p = np.ascontiguousarray(probs, dtype=np.float64)
        out = C.c_double()
        err = C.create_string_buffer(1024)
        st = lib().mtcg_linear_xeb(self.h, n, p.ctypes.data_as(C.POINTER(C.c_double)),
                                   p.size, C.byref(out), err, 1024)
        if st:
            _raise(st, err)
        return out.value

    def linear_xeb_amplitudes(self, n: int, amps) -> float:
        a = np.ascontiguousarray(np.asarray(amps, dtype=np.complex128).ravel())
        out = C.c_double()
        err = C.create_string_buffer(1024)
        st = lib().mtcg_linear_xeb_amplitudes(
            self.h, n, a.view(np.float64).ctypes.data_as(C.POINTER(C.c_double)), a.size,
            C.byref(out), err, 1024)
        if st:
            _raise(st, err)
        return out.value


_default: Optional[Engine] = None


def default_engine() -> Engine:
    global _default
    if _default is None:
        _default = Engine(0)
    return _default


def eval_all(plan: Plan, d: NetworkDiagram, assignments: AssignmentSet,
             opts: Optional[EvalOptions] = None) -> EvalResult:
    return default_engine().eval(problem_arrays(plan, d, assignments), A.MTCG_EVAL_ALL, opts)


def eval_sliced(plan: Plan, d: NetworkDiagram, assignments: AssignmentSet,
                opts: Optional[EvalOptions] = None) -> EvalResult:
    return default_engine().eval(problem_arrays(plan, d, assignments), A.MTCG_EVAL_SLICED, opts)


def emulate_arrays(problem: A.ProblemArrays, opts: Optional[EvalOptions] = None,
                   mode: int = A.MTCG_EVAL_AUTO) -> EmulateResult:
    """Host-only schedule construction with exact counts (mtcg_emulate)."""
    o = _options(mode, opts)
    info = A.mtcg_plan_info()
    nc = np.zeros(max(problem.n_nodes, 1), dtype=np.uint64)
    cap_node = C.c_int32(-1)
    err = C.create_string_buffer(1024)
    st = lib().mtcg_emulate(C.byref(problem.struct()), C.byref(o),
                            int((opts or EvalOptions()).memory_cap_bytes), C.byref(info),
                            nc.ctypes.data_as(C.POINTER(C.c_uint64)), C.byref(cap_node),
                            err, 1024)
    if st:
        _raise(st, err, cap_node.value)
    r = EmulateResult(OpCounters(int(info.mults), int(info.adds), int(info.rw)),
                      int(info.hbm_arena_bytes + info.hbm_resident_bytes),
                      nc[:problem.n_nodes].copy(), int(info.contractions))
    r.plan_info = info  # the device schedule the same options would build
    return r


def emulate(plan: Plan, d: NetworkDiagram, assignments: AssignmentSet,
            opts: Optional[EvalOptions] = None) -> EmulateResult:
    return emulate_arrays(problem_arrays(plan, d, assignments), opts)


def probs_from_amplitudes(amps) -> np.ndarray:
    """|a|^2 per amplitude (xeb.cpp:67-73) — host helper."""
    a = np.asarray(amps, dtype=np.complex128)
    return a.real * a.real + a.imag * a.imag


def linear_xeb(n: int, probs: Sequence[float]) -> float:
    """linear_xeb (xeb.cpp:43-50) reduced on the device."""
    return default_engine().linear_xeb(n, probs)
