"""cfg3 (BASELINE configs[2]: 53-qubit Sycamore m=12, plans/cfg3.plan, 2^20
slices) on the GPU against the unmodified reference's own per-slice
amplitudes (tests/golden/cfg3_reference.npz: run_slice, multieval.cpp:465-476,
on the first 10 bitstrings, slices 0 and 1): complex128 bit-identical,
complex64 within BASELINE §3's amplitude tolerance. The complex64 schedule
runs the tensor-core GEMMs and the long-K kernel (node 619: 16 x 16 x 16384
per item)."""
import os

import numpy as np
import pytest

from paper_2108_05665_b200.engine import EvalOptions

from .helpers import ROOT

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(ROOT, "tests", "golden", "cfg3_reference.npz")


def _subset():
    import bench
    g = np.load(GOLDEN)
    p, circ, _, _ = bench.load_workload("cfg3", int(g["subset"]))
    return g, p, circ


@pytest.mark.parametrize("prec", ["c128", "c64"])
def test_cfg3_slices_against_reference(engine, prec):
    g, p, circ = _subset()
    cp = engine.compile(p, 0, EvalOptions(precision=prec))
    acc = cp.new_accumulator()
    got = []
    for s in g["slices"]:
        cp.run(int(s), int(s) + 1, acc.data_ptr())
        got.append(cp.fetch(acc.data_ptr()).amplitudes.reshape(-1))
    got = np.stack(got)
    want = g["slice_amplitudes"]
    if prec == "c128":
        assert np.array_equal(got.view(np.float64), want.view(np.float64))
    else:
        floor = 2.0 ** (-circ.n_qubits / 2)
        assert np.max(np.abs(got - want) / np.maximum(np.abs(want), floor)) <= 1e-4
        kinds = set(cp.op_kernels())
        assert 12 in kinds and 17 in kinds  # tcgen05 GEMM, long-K kernel
