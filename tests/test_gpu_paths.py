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
