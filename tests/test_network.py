"""Input producers (network.py) pinned to the reference: diagram structure
golden facts (diagram_test.cpp), generators, plan format, and bit-exact
equality with the reference's diagrams/assignments in this container."""
import numpy as np
import pytest

from oracle import refimpl
from paper_2108_05665_b200 import network as N
from paper_2108_05665_b200.errors import DataError, ParseError

from .helpers import GHZ_CIRCUIT, GHZ_PLAN


def test_worked_example_diagram():
    # diagram_test.cpp:38-60: 9 slots, open legs 8/9/10, |0> slots first
    d = N.to_diagram(N.parse_circuit(GHZ_CIRCUIT), False)
    assert d.slot_count == 9
    assert d.n_closed == 8 and d.open_legs == [8, 9, 10]
    for q in range(3):
        assert np.array_equal(d.slot_tensors[q].data, [1, 0])


def test_fusion_keeps_single_network_norm():
    # fused and unfused diagrams describe the same state; |amp|^2 sums to 1
    from paper_2108_05665_b200.engine import problem_arrays
    from oracle import oracle as O

    rng = N.Rng(5)
    c = N.random_circuit(rng, 4, 14)
    bits = [format(i, "04b") for i in range(16)]
    amps = []
    for fuse in (False, True):
        d = N.to_diagram(c, fuse)
        p = problem_arrays(N.left_deep_plan(d.slot_count), d, N.build_assignments(d, bits, []))
        amps.append(O.eval_problem(p)[0].ravel())
    assert np.allclose(amps[0], amps[1], atol=1e-12)
    assert abs(np.sum(np.abs(amps[0]) ** 2) - 1) < 1e-12


def test_plan_format_round_trip_and_errors():
    p = N.parse_plan(GHZ_PLAN)
    assert N.format_plan(p) == GHZ_PLAN
    assert N.parse_plan("0 1\nslice: 3 1\n").sliced == [3, 1]
    assert N.format_plan(N.parse_plan("(0)")) == "(0)\nslice:\n"
    for bad in ("", "(0 1", "0 1)", "0 1\nslices: 2\n", "0 x"):
        with pytest.raises(ParseError):
            N.parse_plan(bad)


def test_assignment_errors():
    d = N.to_diagram(N.parse_circuit(GHZ_CIRCUIT), False)
    with pytest.raises(DataError, match="has length"):
        N.build_assignments(d, ["00"], [])
    with pytest.raises(DataError, match="invalid character"):
        N.build_assignments(d, ["0x0"], [])
    with pytest.raises(DataError, match="batch position"):
        N.build_assignments(d, ["0*0"], [])


def test_circuit_parse_errors():
    for bad, msg in [("", "empty circuit"), ("x\n", "qubit count"), ("2\n0 foo 0\n", "unknown gate"),
                     ("2\n0 cz 0\n", "needs two qubits"), ("2\n1 h 0\n0 h 1\n", "non-decreasing"),
                     ("2\n0 h 0\n0 x 0\n", "used twice"), ("2\n0 h 5\n", "out of range")]:
        with pytest.raises(ParseError, match=msg):
            N.parse_circuit(bad)


@pytest.mark.skipif(not refimpl.available(), reason="reference build absent (GPU box)")
@pytest.mark.parametrize("seed", range(40))
def test_bit_exact_against_reference_producers(seed):
    rng = N.Rng(seed)
    n = 2 + rng.uniform_index(6)
    c = N.random_circuit(rng, n, 24)
    circ = N.format_circuit(c)
    bits = N.random_bitstrings(rng, n, 1 + rng.uniform_index(12))
    if seed % 4 == 1:
        q = rng.uniform_index(n)
        bits = [b[:q] + "*" + b[q + 1:] for b in bits]
    fuse = seed % 2 == 0
    rp = refimpl.RefProblem(circ, bits, None, fuse=fuse)
    d = N.to_diagram(N.parse_circuit(circ), fuse)
    assert d.n_closed == rp.n_closed and d.slot_count == rp.n_slots
    for j in range(d.slot_count):
        legs, data = rp.slot_tensor(j)
        assert legs == d.slot_tensors[j].legs
        assert np.array_equal(data.view(np.float64), d.slot_tensors[j].data.view(np.float64))
    asg = N.build_assignments(d, bits, N.batch_legs_of(d, bits))
    assert np.array_equal(asg.tuples, rp.tuples())
    for j in range(d.slot_count):
        legs, data = rp.value_set(j)
        assert legs == asg.value_sets[j][0].legs
        assert np.array_equal(np.stack([t.data for t in asg.value_sets[j]]), data)


@pytest.mark.skipif(not refimpl.available(), reason="reference build absent (GPU box)")
def test_generators_match_reference():
    for args in [(3, 4, 8, 12345), (5, 6, 12, 12345), (2, 3, 5, 7)]:
        assert refimpl.grid_circuit(*args) == N.format_circuit(N.grid_circuit(*args))
    assert refimpl.random_bitstrings(99, 30, 64) == N.random_bitstrings(N.Rng(99), 30, 64)
    for s in range(20):
        assert refimpl.random_circuit(s, 5, 18) == N.format_circuit(N.random_circuit(N.Rng(s), 5, 18))
