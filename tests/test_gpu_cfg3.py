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


def test_long_k_gather_tiles_against_complex128(engine):
    """Gather-mode tensor-core tiles for long-K per-item ops (M = 64, one item
    per 128-row tile, K = 4096): a traffic-heavier cfg3 tree
    (tests/golden/cfg3_longk_gather.plan, from plans/sycamore_plan.py with
    alpha = 30) has such a node (598: 64 x 64 x 4096 per request) once the
    batch passes 1,024 requests. Slice 0 on 1,100 requests: complex64 on the
    tensor cores within BASELINE §3's tolerance of complex128."""
    import bench
    from workloads import network as N
    from paper_2108_05665_b200.engine import problem_arrays

    c = N.sycamore_circuit(12, 2024)
    d = N.to_diagram(c, True)
    bits = N.random_bitstrings(N.Rng(99), 53, 1100)
    plan = N.parse_plan(open(os.path.join(ROOT, "tests", "golden", "cfg3_longk_gather.plan")).read())
    p = problem_arrays(plan, d, N.build_assignments(d, bits, []))
    cp = engine.compile(p, 0, EvalOptions(precision="c64"))
    ga = [o for o in cp.op_infos() if o.kernel == 12 and o.fa in (5, 6) and o.kc >= 9]
    assert ga, "no long-K gather op in this schedule"
    acc = cp.new_accumulator()
    cp.run(0, 1, acc.data_ptr())
    got = cp.fetch(acc.data_ptr()).amplitudes
    c2 = engine.compile(p, 0, EvalOptions(precision="c128"))
    acc2 = c2.new_accumulator()
    c2.run(0, 1, acc2.data_ptr())
    want = c2.fetch(acc2.data_ptr()).amplitudes
    floor = 2.0 ** (-c.n_qubits / 2)
    assert np.max(np.abs(got - want) / np.maximum(np.abs(want), floor)) <= 1e-4
