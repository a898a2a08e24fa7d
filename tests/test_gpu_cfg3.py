"""cfg3 / cfg4 (BASELINE configs[2-3]: 53-qubit Sycamore m=12 / 14,
plans/cfg3.plan / cfg4.plan, 2^20 / 2^24 slices) on the GPU against the
unmodified reference's own per-slice amplitudes
(tests/golden/<cfg>_reference.npz: run_slice, multieval.cpp:465-476, on the
first 10 bitstrings, slices 0 and 1): complex128 bit-identical,
complex64 within BASELINE §3's amplitude tolerance. The complex64 schedule
runs the tensor-core GEMMs and the long-K kernel (node 619: 16 x 16 x 16384
per item)."""
import os

import numpy as np
import pytest

from paper_2108_05665_b200.engine import EvalOptions

from .helpers import ROOT

pytestmark = pytest.mark.gpu

def _subset(name):
    import bench
    path = os.path.join(ROOT, "tests", "golden", f"{name}_reference.npz")
    if not os.path.exists(path):
        pytest.skip(f"{path} not generated (tests/golden/make_sycamore_reference.py --config {name})")
    g = np.load(path)
    p, circ, _, _ = bench.load_workload(name, int(g["subset"]))
    return g, p, circ


@pytest.mark.parametrize("name", ["cfg3", "cfg4"])
@pytest.mark.parametrize("prec", ["c128", "c64"])
def test_cfg3_slices_against_reference(engine, prec, name):
    g, p, circ = _subset(name)
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
        assert 12 in kinds  # tcgen05 GEMM
        if name == "cfg3":
            assert 17 in kinds  # long-K kernel
