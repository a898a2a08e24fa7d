"""GPU: the alternative launch/kernel paths of one workload agree.

* slice graph (captured once, replayed per slice after a set-slice kernel)
  vs direct launches (MTCG_NO_GRAPHS=1) — same kernels, bit-identical;
* concurrent (multi-stream DAG) capture vs the serial graph — bit-identical;
* grouped kernels (items sharing an A entry read it once: rows-grouped in
  complex128, grouped tcgen05 GEMM in complex64) vs ungrouped
  (MTCG_NO_GROUP=1) — complex128 bit-identical (same per-output reduction
  order), complex64 within the north-star tolerance;
* the leaf-operand slice projection resolved on the device for every slice
  (staged one-slice runs fold to the full run).
"""
import numpy as np
import pytest

from oracle import oracle as O
from paper_2108_05665_b200 import _abi as A
from paper_2108_05665_b200.engine import EvalOptions

from .helpers import random_instance, rel_err, workload

pytestmark = pytest.mark.gpu

TOL = 1e-4


def bits_equal(x, y) -> bool:
    return np.array_equal(np.asarray(x).view(np.float64), np.asarray(y).view(np.float64))


def run(engine, p, opts, runs=2):
    """Evaluate all slices `runs` times on one plan (the 2nd run replays the
    captured graph) and return the last result."""
    cp = engine.compile(p, A.MTCG_EVAL_AUTO, opts)
    acc = cp.new_accumulator()
    for _ in range(runs):
        cp.run(0, cp.n_slices, acc.data_ptr())
    return cp.fetch(acc.data_ptr()).amplitudes


@pytest.mark.parametrize("precision", ["c64", "c128"])
def test_graph_replay_matches_direct_launches(engine, monkeypatch, precision):
    p, c, bits = workload("cfg1")
    opts = EvalOptions(precision=precision)
    graphed = run(engine, p, opts)
    monkeypatch.setenv("MTCG_NO_GRAPHS", "1")
    direct = run(engine, p, opts)
    assert bits_equal(graphed, direct)


def test_multi_stream_capture_matches_serial(engine, monkeypatch):
    p, c, bits = workload("cfg1")
    opts = EvalOptions(precision="c64")
    serial = run(engine, p, opts)
    monkeypatch.setenv("MTCG_STREAMS", "6")
    concurrent = run(engine, p, opts)
    assert bits_equal(serial, concurrent)


@pytest.mark.parametrize("name", ["cfg1", "cfg2"])
def test_grouped_kernels_match_ungrouped(engine, monkeypatch, name):
    p, c, bits = workload(name)
    if name == "cfg2":  # complex64: grouped tcgen05 GEMM + grouped rows
        opts = EvalOptions(precision="c64")
        s1 = 1
    else:
        opts = EvalOptions(precision="c128")
        s1 = None

    def one(env):
        if env:
            monkeypatch.setenv("MTCG_NO_GROUP", "1")
        else:
            monkeypatch.delenv("MTCG_NO_GROUP", raising=False)
        cp = engine.compile(p, A.MTCG_EVAL_AUTO, opts)
        acc = cp.new_accumulator()
        cp.run(0, s1 or cp.n_slices, acc.data_ptr())
        return cp.fetch(acc.data_ptr()).amplitudes

    grouped, plain = one(False), one(True)
    if opts.precision == "c128":
        assert bits_equal(grouped, plain)
        ov, _, _, _ = O.eval_problem(p)
        assert bits_equal(grouped, ov)
    else:
        assert rel_err(grouped, plain, c.n_qubits) <= TOL
        assert np.linalg.norm(grouped - plain) / np.linalg.norm(plain) <= TOL


@pytest.mark.parametrize("seed", [0, 3, 6, 9])
def test_device_slice_offsets_every_slice(engine, seed):
    import torch

    p, c, bits = random_instance(seed)
    cp = engine.compile(p, A.MTCG_EVAL_AUTO, EvalOptions(precision="c128"))
    S = cp.n_slices
    acc = cp.new_accumulator()
    for s in range(S):  # one graph, replayed with a different device slice index
        cp.run(s, s + 1, acc.data_ptr(), accumulate=s > 0)
    torch.cuda.synchronize()
    ov, _, _, _ = O.eval_problem(p)
    assert bits_equal(cp.fetch(acc.data_ptr()).amplitudes, ov)


@pytest.mark.parametrize("name,precision", [("cfg2", "c64"), ("cfg2", "c128")])
def test_slice_reuse_bit_identical(engine, name, precision):
    """Cross-slice reuse (MTCG_FLAG_SLICE_REUSE): the
    slice-invariant subtrees evaluated once per run give bit-identical
    amplitudes (every op is deterministic; only the schedule changes), also
    for staged slice ranges (the prologue reruns on every run call)."""
    p, c, bits = workload(name)
    base = run(engine, p, EvalOptions(precision=precision))
    reuse = run(engine, p, EvalOptions(precision=precision, slice_reuse=True))
    assert bits_equal(base, reuse)
    cp = engine.compile(p, A.MTCG_EVAL_AUTO, EvalOptions(precision=precision, slice_reuse=True))
    assert cp.info.prologue_ops > 0
    assert cp.info.executed_contractions < cp.info.contractions
    capped = engine.compile(p, A.MTCG_EVAL_AUTO, EvalOptions(precision=precision, slice_reuse=True,
                                                               memory_cap_bytes=64 << 30))
    assert capped.info.prologue_ops == 0  # reference cap accounting: no resident tables
    del capped
    acc = cp.new_accumulator()
    S = cp.n_slices
    cp.run(0, S // 2, acc.data_ptr())
    cp.run(S // 2, S, acc.data_ptr(), accumulate=True)
    staged = cp.fetch(acc.data_ptr()).amplitudes
    # two partial folds: the same per-slice values, summed (c128 summation
    # order matches the single fold: slices accumulate in index order)
    if precision == "c128":
        assert bits_equal(staged, base)
    else:
        assert rel_err(staged, base, c.n_qubits) <= TOL


@pytest.mark.parametrize("seed", [0, 3, 6, 9, 12, 15])
def test_slice_reuse_random_instances(engine, seed):
    p, c, bits = random_instance(seed)
    cp = engine.compile(p, A.MTCG_EVAL_AUTO, EvalOptions(precision="c128", slice_reuse=True))
    acc = cp.new_accumulator()
    cp.run(0, cp.n_slices, acc.data_ptr())
    ov, _, _, _ = O.eval_problem(p)
    assert bits_equal(cp.fetch(acc.data_ptr()).amplitudes, ov)


def test_plan_survives_arena_growth(engine):
    """Plans share the handle's arena; compiling a larger plan moves it. An
    earlier plan must follow (re-resolve the arena, re-capture its graph)."""
    p1, c1, _ = workload("cfg1")
    opts = EvalOptions(precision="c128")
    cp1 = engine.compile(p1, A.MTCG_EVAL_AUTO, opts)
    acc1 = cp1.new_accumulator()
    cp1.run(0, cp1.n_slices, acc1.data_ptr())  # graph captured on the current arena
    first = cp1.fetch(acc1.data_ptr()).amplitudes
    p2, _, _ = workload("cfg2")
    cp2 = engine.compile(p2, A.MTCG_EVAL_AUTO, EvalOptions(precision="c64", slice_reuse=True))
    acc2 = cp2.new_accumulator()
    cp2.run(0, 1, acc2.data_ptr())
    cp1.run(0, cp1.n_slices, acc1.data_ptr())
    assert bits_equal(cp1.fetch(acc1.data_ptr()).amplitudes, first)


def _op_kernels(cp):
    import ctypes as C

    from paper_2108_05665_b200._lib import lib

    from paper_2108_05665_b200._abi import mtcg_op_info as OpInfo  # the one ABI struct

    L = lib()
    L.mtcg_plan_op_count.restype = C.c_int32
    L.mtcg_plan_op_count.argtypes = [C.c_void_p]
    L.mtcg_plan_op_info.argtypes = [C.c_void_p, C.c_int32, C.POINTER(OpInfo)]
    out = []
    for i in range(L.mtcg_plan_op_count(cp.h)):
        oi = OpInfo()
        L.mtcg_plan_op_info(cp.h, i, C.byref(oi))
        out.append((oi.node, oi.kernel))
    return out


@pytest.mark.parametrize("name,precision", [("cfg1", "c128"), ("cfg2", "c128"), ("cfg2", "c64")])
def test_fused_chains_match_unfused(engine, monkeypatch, name, precision):
    """Fused operand chains (consecutive skinny ops evaluated in shared memory,
    planner.hpp Chain) keep every step's reduction order: bit-identical to
    the op-by-op path in both precisions; and they are in use (cfg2: nodes
    301 -> 302 -> 304 -> 305)."""
    p, c, bits = workload(name)
    opts = EvalOptions(precision=precision)
    cp = engine.compile(p, A.MTCG_EVAL_AUTO, opts)
    fused_nodes = [n for n, k in _op_kernels(cp) if k == 16]
    assert fused_nodes, "no fused chains"
    if name == "cfg2":
        assert {301, 302, 304, 305} <= set(fused_nodes)
    del cp
    fused = run(engine, p, opts)
    monkeypatch.setenv("MTCG_NO_CHAIN", "1")
    plain = run(engine, p, opts)
    assert bits_equal(fused, plain)
    if precision == "c128" and name == "cfg1":
        ov, _, _, _ = O.eval_problem(p)
        assert bits_equal(fused, ov)


@pytest.mark.parametrize("seed", list(range(0, 40, 3)))
def test_fused_chains_random_instances(engine, seed):
    p, c, bits = random_instance(seed)
    cp = engine.compile(p, A.MTCG_EVAL_AUTO, EvalOptions(precision="c128"))
    acc = cp.new_accumulator()
    cp.run(0, cp.n_slices, acc.data_ptr())
    ov, _, _, _ = O.eval_problem(p)
    assert bits_equal(cp.fetch(acc.data_ptr()).amplitudes, ov)
