"""GPU parity: the CUDA path (through the C ABI) against the C oracle and the
reference's golden vectors.

C128 mode must be bit-identical to the oracle (which is bit-identical to the
reference, tests/test_oracle.py); C64 mode must satisfy the north-star
tolerance |a_gpu - a_ref| <= 1e-4 * max(|a_ref|, 2^(-n/2)) per amplitude and
relative L2 <= 1e-4 over the batch.
"""
import math
import os

import numpy as np
import pytest

from oracle import oracle as O
from paper_2108_05665_b200 import _abi as A
from paper_2108_05665_b200.engine import EvalOptions
from paper_2108_05665_b200.errors import DataError, MemoryCapError

from .helpers import GHZ_CIRCUIT, GHZ_PLAN, GOLDEN_AMP, ROOT, build, random_instance, rel_err, workload

pytestmark = pytest.mark.gpu

C64 = EvalOptions(precision="c64")
C128 = EvalOptions(precision="c128")
TOL = 1e-4


def bits_equal(x: np.ndarray, y: np.ndarray) -> bool:
    return np.array_equal(np.asarray(x).view(np.float64), np.asarray(y).view(np.float64))


def test_worked_example_golden(engine):
    p, _ = build(GHZ_CIRCUIT, ["000", "100", "111"], GHZ_PLAN, fuse=False)
    for opts in (C64, C128):
        r = engine.eval(p, A.MTCG_EVAL_ALL, opts)
        assert np.allclose(r.amplitudes.ravel(), GOLDEN_AMP, rtol=0, atol=1e-7)
        nc = r.node_contractions
        assert int(nc.sum()) == 13  # multieval_test.cpp:112
        assert sorted(int(x) for x in nc if x) == [1, 1, 1, 1, 2, 2, 2, 3]
        assert int(nc[p.root]) == 3
    r = engine.eval(p, A.MTCG_EVAL_ALL, C128)
    assert np.all(np.abs(r.amplitudes - GOLDEN_AMP) < 1e-12)  # multieval_test.cpp:85
    ov, onc, ocnt, _ = O.eval_problem(p)
    assert bits_equal(r.amplitudes, ov)
    assert (r.counters.mults, r.counters.adds, r.counters.rw) == ocnt


@pytest.mark.parametrize("seed", range(0, 240))
def test_random_instances_c128_bit_exact_and_c64_tolerance(engine, seed):
    p, c, bits = random_instance(seed)
    ov, onc, ocnt, olegs = O.eval_problem(p)
    r = engine.eval(p, A.MTCG_EVAL_AUTO, C128)
    assert bits_equal(r.amplitudes, ov), np.max(np.abs(r.amplitudes - ov))
    assert np.array_equal(r.node_contractions, onc)
    assert (r.counters.mults, r.counters.adds, r.counters.rw) == ocnt
    assert [int(x) for x in r.values[0].legs] == olegs if len(bits) else True
    r64 = engine.eval(p, A.MTCG_EVAL_AUTO, C64)
    assert rel_err(r64.amplitudes, ov, c.n_qubits) <= TOL
    assert np.array_equal(r64.node_contractions, onc)


def test_sliced_single_leg_two_tensor_network(engine):
    # multieval_test.cpp:285-299: <0|H|0> with its only closed leg sliced
    p, _ = build("1\n0 h 0\n", ["0"], "0 1\nslice: 0\n", fuse=False)
    for opts in (C64, C128):
        r = engine.eval(p, A.MTCG_EVAL_SLICED, opts)
        assert abs(r.amplitudes[0, 0] - 1 / math.sqrt(2)) < 1e-7
    with pytest.raises(DataError, match="use eval_sliced"):
        engine.eval(p, A.MTCG_EVAL_ALL, C64)
    p2, _ = build("1\n0 h 0\n", ["0"], "0 1\nslice: 0 0\n", fuse=False)
    with pytest.raises(DataError, match="sliced twice"):
        engine.eval(p2, A.MTCG_EVAL_SLICED, C64)
    p3, _ = build("1\n0 h 0\n", ["0"], "0 1\n", fuse=False)
    with pytest.raises(DataError, match="no sliced legs"):
        engine.eval(p3, A.MTCG_EVAL_SLICED, C64)


def test_batch_legs_expand_like_state_vector(engine):
    # multieval_test.cpp:186-200 circuit, requests 0*0 and 1*1
    circ = "3\n0 h 0\n0 h 2\n1 cx 0 1\n2 fs 1 2 0.7 0.3\n"
    p, d = build(circ, ["0*0", "1*1"], None, fuse=False)
    ov, _, _, olegs = O.eval_problem(p)
    r = engine.eval(p, A.MTCG_EVAL_ALL, C128)
    assert bits_equal(r.amplitudes, ov)
    assert [int(x) for x in r.values[0].legs] == olegs == [d.open_legs[1]]


def test_duplicate_requests_evaluated_once(engine):
    p1, _ = build(GHZ_CIRCUIT, ["101"], GHZ_PLAN, fuse=False)
    p3, _ = build(GHZ_CIRCUIT, ["101", "101", "101"], GHZ_PLAN, fuse=False)
    r1 = engine.eval(p1, A.MTCG_EVAL_ALL, C128)
    r3 = engine.eval(p3, A.MTCG_EVAL_ALL, C128)
    assert np.array_equal(r3.node_contractions, r1.node_contractions)
    assert all(bits_equal(r3.amplitudes[i], r1.amplitudes[0]) for i in range(3))


def test_memory_cap_reports_node(engine):
    from workloads import network as N

    rng = N.Rng(77)
    c = N.random_circuit(rng, 5, 20)
    bits = N.random_bitstrings(rng, 5, 3)
    p, _ = build(N.format_circuit(c), bits, None, fuse=False)
    with pytest.raises(MemoryCapError) as ei:
        engine.eval(p, A.MTCG_EVAL_ALL, EvalOptions(memory_cap_bytes=256))
    assert "memory cap exceeded" in str(ei.value)
    assert ei.value.node >= 0


def test_empty_request_set_and_lone_leaf(engine):
    p, _ = build(GHZ_CIRCUIT, [], GHZ_PLAN, fuse=False)
    r = engine.eval(p, A.MTCG_EVAL_ALL, C64)
    assert r.amplitudes.shape[0] == 0 and int(r.node_contractions.sum()) == 0
    # one-qubit network with no gates: the root is the |0> leaf
    p1, _ = build("1\n", ["0", "1"], "(0)\n", fuse=False)
    r1 = engine.eval(p1, A.MTCG_EVAL_ALL, C128)
    assert np.array_equal(r1.amplitudes.ravel(), np.array([1, 0], dtype=np.complex128))


@pytest.mark.parametrize("precision", ["c64", "c128"])
def test_cfg1_full_workload(engine, precision):
    p, c, bits = workload("cfg1")
    ov, onc, ocnt, _ = O.eval_problem(p)
    r = engine.eval(p, A.MTCG_EVAL_AUTO, EvalOptions(precision=precision))
    assert np.array_equal(r.node_contractions, onc)
    assert (r.counters.mults, r.counters.adds, r.counters.rw) == ocnt
    if precision == "c128":
        assert bits_equal(r.amplitudes, ov)
    else:
        assert rel_err(r.amplitudes, ov, c.n_qubits) <= TOL
        assert np.linalg.norm(r.amplitudes - ov) / np.linalg.norm(ov) <= TOL


def test_staged_api_slice_ranges_sum_to_full_run(engine):
    import torch

    p, c, bits = random_instance(3)  # sliced instance (seed % 3 == 0)
    cp = engine.compile(p, A.MTCG_EVAL_AUTO, C128)
    S = cp.n_slices
    assert S >= 2
    acc = cp.new_accumulator()
    cp.run(0, S, acc.data_ptr(), accumulate=False)
    full = cp.fetch(acc.data_ptr()).amplitudes
    acc2 = cp.new_accumulator()
    for s in range(S):  # one slice at a time, folded in order
        cp.run(s, s + 1, acc2.data_ptr(), accumulate=s > 0)
    torch.cuda.synchronize()
    assert bits_equal(cp.fetch(acc2.data_ptr()).amplitudes, full)
    ov, _, _, _ = O.eval_problem(p)
    assert bits_equal(full, ov)


def test_xeb_device_matches_oracle(engine):
    p, c, bits = workload("cfg1")
    cp = engine.compile(p, A.MTCG_EVAL_AUTO, C128)
    acc = cp.new_accumulator()
    cp.run(0, cp.n_slices, acc.data_ptr())
    f_dev = cp.xeb(acc.data_ptr(), c.n_qubits)
    ov, _, _, _ = O.eval_problem(p)
    f_ref = O.linear_xeb(c.n_qubits, (np.abs(ov) ** 2).ravel())
    assert abs(f_dev - f_ref) <= 1e-12 * max(1.0, abs(f_ref))
    probs = (np.abs(ov) ** 2).ravel()
    assert abs(engine.linear_xeb(c.n_qubits, probs) - f_ref) <= 1e-12 * max(1.0, abs(f_ref))
    assert abs(engine.linear_xeb_amplitudes(c.n_qubits, ov) - f_ref) <= 1e-12 * max(1.0, abs(f_ref))
    with pytest.raises(DataError, match="negative probability"):
        engine.linear_xeb(3, np.array([0.1, -0.2]))
    with pytest.raises(DataError, match="at least one sample"):
        engine.linear_xeb(3, np.array([]))
    # xeb_test.cpp:26-40: uniform -> 0; single p = 2^(1-n) -> 1
    assert abs(engine.linear_xeb(4, np.full(16, 1 / 16))) < 1e-15
    assert abs(engine.linear_xeb(4, np.array([2.0 ** -3])) - 1.0) < 1e-15


GOLDEN_CFG2 = os.path.join(ROOT, "tests", "golden", "cfg2_reference.npz")


@pytest.mark.skipif(not os.path.exists(GOLDEN_CFG2), reason="cfg2 golden not generated")
@pytest.mark.parametrize("tensor_cores", [True, False])
def test_cfg2_full_size_against_reference_golden(engine, tensor_cores):
    """The bench workload at full size (30 qubits, 10^4 bitstrings, 16
    slices) against the reference's own complex128 amplitudes
    (tests/golden/cfg2_reference.npz, a full eval_sliced run).

    Amplitudes: |a - a_ref| <= 1e-4 max(|a_ref|, 2^-n/2), L2 <= 1e-4; F_XEB:
    SURVEY §8c / BASELINE §3's |dF| <= 1e-4 (|F| + 1/sqrt(k)) — in both modes
    (the tensor-core path accumulates split-integer digits exactly, so it
    carries no systematic scale error; tools/bias_sweep.sh)."""
    g = np.load(GOLDEN_CFG2)
    p, c, bits = workload("cfg2")
    cp = engine.compile(p, A.MTCG_EVAL_AUTO, EvalOptions(precision="c64", tensor_cores=tensor_cores))
    acc = cp.new_accumulator()
    cp.run(0, cp.n_slices, acc.data_ptr())
    r = cp.fetch(acc.data_ptr())
    want = g["amplitudes"].reshape(r.amplitudes.shape)
    assert np.array_equal(r.node_contractions, g["node_contractions"])
    assert (r.counters.mults, r.counters.adds, r.counters.rw) == tuple(int(x) for x in g["counters"])
    assert rel_err(r.amplitudes, want, c.n_qubits) <= TOL
    assert np.linalg.norm(r.amplitudes - want) / np.linalg.norm(want) <= TOL
    f_ref = O.linear_xeb(c.n_qubits, (np.abs(want) ** 2).ravel())
    f_dev = cp.xeb(acc.data_ptr(), c.n_qubits)
    scale = np.vdot(want, r.amplitudes).real / np.vdot(want, want).real - 1.0
    print(f"cfg2 full size, tensor_cores={tensor_cores}: max rel "
          f"{rel_err(r.amplitudes, want, c.n_qubits):.2e}, L2 "
          f"{np.linalg.norm(r.amplitudes - want) / np.linalg.norm(want):.2e}, scale bias {scale:.2e}, "
          f"F {f_dev:.6f} vs {f_ref:.6f} (dF {f_dev - f_ref:.2e})")
    assert abs(f_dev - f_ref) <= TOL * (abs(f_ref) + 1 / math.sqrt(len(bits)))


def test_cfg1_statevector_sampled_xeb(engine):
    """cfg1 with 1,000 bitstrings sampled from the exact output distribution
    (SURVEY §8(d)): c128 amplitudes bit-identical to the oracle, and the fused
    device XEB within 5 sigma of the target 2^n sum p^2 - 1 while uniform
    bitstrings (the cfg1 workload) sit within 5 sigma of 0 — the reference's
    XEB criterion (tests/acceptance_main.cpp:400-428) on cfg1."""
    from .helpers import statevector_samples

    p, c, bits, probs, target = statevector_samples("cfg1", 1000, 411)
    want, _, _, _ = O.eval_problem(p)
    cp = engine.compile(p, A.MTCG_EVAL_AUTO, EvalOptions(precision="c128"))
    acc = cp.new_accumulator()
    cp.run(0, cp.n_slices, acc.data_ptr())
    got = cp.fetch(acc.data_ptr())
    assert bits_equal(got.amplitudes, want)
    assert np.allclose((np.abs(want.reshape(-1)) ** 2), probs, rtol=1e-12, atol=0)
    sigma = 1.0 / math.sqrt(len(bits))
    f = cp.xeb(acc.data_ptr(), c.n_qubits)
    assert abs(f - target) < 5 * sigma and target > 10 * sigma
    pu, cu, _ = workload("cfg1")
    cpu = engine.compile(pu, A.MTCG_EVAL_AUTO, EvalOptions(precision="c128"))
    accu = cpu.new_accumulator()
    cpu.run(0, cpu.n_slices, accu.data_ptr())
    assert abs(cpu.xeb(accu.data_ptr(), cu.n_qubits)) < 5 * sigma
