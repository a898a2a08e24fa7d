"""Paper-scale request ingestion through the C ABI:
sample files -> canonical sample matrix (read_samples, formats.cpp:42-69),
the per-slot value ranking of build_assignments (diagram.cpp:229-297) ->
the tuple matrix of mtcg_problem, and amplitude TSV output with '*'
expansion (formats.cpp:78-83, tools/main.cpp:161-179). Native and
multithreaded in libmtcg (csrc/ingest.cpp); no per-row Python."""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import List, Sequence, Union

import numpy as np

from ._lib import lib
from .engine import _raise

Q0_FIRST, Q0_LAST = 0, 1  # BitOrder (formats.hpp:28)


def read_samples(text: Union[bytes, str], order: int = Q0_FIRST) -> np.ndarray:
    """Samples text -> (n_rows, n_qubits) uint8 array of b'0' / b'1' / b'*',
    canonical (qubit 0 first)."""
    buf = text.encode() if isinstance(text, str) else bytes(text)
    out = np.empty(max(len(buf), 1), dtype=np.uint8)
    n, nq = C.c_uint64(0), C.c_int32(0)
    err = C.create_string_buffer(1024)
    st = lib().mtcg_read_samples(buf, len(buf), order, out.ctypes.data, out.size, C.byref(n), C.byref(nq),
                                 err, 1024)
    if st:
        _raise(st, err)
    return out[: n.value * nq.value].reshape(n.value, nq.value)


def read_samples_file(path: str, order: int = Q0_FIRST) -> np.ndarray:
    with open(path, "rb") as f:
        return read_samples(f.read(), order)


def sample_strings(m: np.ndarray) -> List[str]:
    return [bytes(r).decode() for r in m]


@dataclass
class Assignment:
    tuples: np.ndarray          # (n_rows, n_slots) uint32 (mtcg_problem.tuples)
    slot_n_values: np.ndarray   # (n_slots,)
    value_keys: List[np.ndarray]  # per slot: distinct fixed-bit tuples, ascending (packed, first bit MSB)
    fixed_qubits: List[List[int]]  # per slot: the non-batch qubits of its open legs


def assign(samples: np.ndarray, slot_qubits: Sequence[Sequence[int]]) -> Assignment:
    """slot_qubits[j]: the qubits of slot j's open legs in slot_open_legs
    order. Batch positions are the '*' columns of sample 0."""
    s = np.ascontiguousarray(samples, dtype=np.uint8)
    n, nq = (s.shape[0], s.shape[1]) if s.ndim == 2 else (0, 0)
    m = len(slot_qubits)
    begin = np.zeros(m + 1, dtype=np.int32)
    for j, qs in enumerate(slot_qubits):
        begin[j + 1] = begin[j] + len(qs)
    flat = np.array([q for qs in slot_qubits for q in qs] or [0], dtype=np.int32)
    tuples = np.empty((n, m), dtype=np.uint32)
    nv = np.zeros(max(m, 1), dtype=np.int32)
    kb = np.zeros(m + 1, dtype=np.uint64)
    cap = sum(min(max(n, 1), 1 << min(len(qs), 24)) for qs in slot_qubits) + m
    keys = np.zeros(max(cap, 1), dtype=np.uint32)
    err = C.create_string_buffer(1024)
    st = lib().mtcg_assign(s.ctypes.data if n else None, n, nq, m, begin.ctypes.data, flat.ctypes.data,
                           tuples.ctypes.data if n and m else None, nv.ctypes.data, kb.ctypes.data,
                           keys.ctypes.data, keys.size, err, 1024)
    if st:
        _raise(st, err)
    star = [bool(n) and s[0, q] == ord("*") for q in range(nq)]
    fixed = [[q for q in qs if not star[q]] for qs in slot_qubits]
    vk = [keys[int(kb[j]):int(kb[j + 1])].copy() for j in range(m)]
    return Assignment(tuples, nv[:m].copy(), vk, fixed)


def write_amplitudes(path: str, samples: np.ndarray, values: np.ndarray, order: int = Q0_FIRST) -> int:
    """values: (n_rows, 2^w) complex (EvalResult.amplitudes). Returns bytes."""
    s = np.ascontiguousarray(samples, dtype=np.uint8)
    v = np.ascontiguousarray(values, dtype=np.complex128)
    n, nq = s.shape
    w = int(round(np.log2(v.shape[1]))) if v.ndim == 2 and v.shape[1] else 0
    written = C.c_uint64(0)
    err = C.create_string_buffer(1024)
    st = lib().mtcg_write_amplitudes(path.encode(), s.ctypes.data if n else None, n, nq, order,
                                     v.view(np.float64).ctypes.data if n else None, w, C.byref(written),
                                     err, 1024)
    if st:
        _raise(st, err)
    return written.value
