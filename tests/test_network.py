"""Input producers (network.py) pinned to the reference: diagram structure
golden facts (diagram_test.cpp), generators, plan format, and bit-exact
equality with the reference's diagrams/assignments in this container."""
import numpy as np
import pytest

from oracle import refimpl
from workloads import network as N
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


def test_sycamore_layout_and_cycle_pattern():
    # BASELINE configs 3-5: the 53-qubit Sycamore layout (86 couplers; 88 with
    # all 54 sites), layers A-D partition the couplers into matchings, cycle i
    # uses layer ABCDCDAB[i % 8], fSim(pi/2, pi/6), single-qubit gates never
    # repeat on a qubit, and a final single-qubit moment closes the circuit
    for n, n_couplers in [(53, 86), (54, 88)]:
        sites = N.sycamore_sites(n)
        assert len(sites) == n == len(set(sites))
        layers = {p: N.sycamore_layer(sites, p) for p in "ABCD"}
        every = [tuple(sorted(e)) for p in "ABCD" for e in layers[p]]
        assert len(every) == len(set(every)) == n_couplers
        for p, pairs in layers.items():
            used = [q for e in pairs for q in e]
            assert len(used) == len(set(used)), p  # a matching
            for a, b in pairs:
                (ra, ca), (rb, cb) = sites[a], sites[b]
                assert abs(ra - rb) + abs(ca - cb) == 1
    with pytest.raises(DataError):
        N.sycamore_sites(50)
    m = 12
    c = N.sycamore_circuit(m, 12345)
    assert c.n_qubits == 53
    sites = N.sycamore_sites(53)
    moments = {}
    for g in c.gates:
        moments.setdefault(g.moment, []).append(g)
    assert sorted(moments) == list(range(2 * m + 1))
    prev = [None] * 53
    for t in range(2 * m + 1):
        gs = moments[t]
        if t % 2 == 0:  # single-qubit moment over every qubit
            assert sorted(g.q0 for g in gs) == list(range(53))
            for g in gs:
                assert g.name in ("x_1_2", "y_1_2", "hz_1_2") and g.name != prev[g.q0]
                prev[g.q0] = g.name
        else:
            want = N.sycamore_layer(sites, "ABCDCDAB"[(t // 2) % 8])
            assert [(g.q0, g.q1) for g in gs] == want
            assert all(g.name == "fs" and g.p0 == pytest.approx(np.pi / 2) and
                       g.p1 == pytest.approx(np.pi / 6) for g in gs)
    # round trip through the reference's circuit text format
    assert N.format_circuit(N.parse_circuit(N.format_circuit(c))) == N.format_circuit(c)
    # deterministic in the seed
    assert N.format_circuit(N.sycamore_circuit(m, 12345)) == N.format_circuit(c)
    assert N.format_circuit(N.sycamore_circuit(m, 1)) != N.format_circuit(c)


@pytest.mark.skipif(not refimpl.available(), reason="reference build absent (GPU box)")
def test_sycamore_circuit_consumed_by_reference():
    # the reference's loader builds the same fused 53-qubit network (311
    # slots, 516 closed legs at m = 12) and the same leaves, bit for bit
    c = N.format_circuit(N.sycamore_circuit(12, 12345))
    bits = N.random_bitstrings(N.Rng(99), 53, 8)
    rp = refimpl.RefProblem(c, bits, None, fuse=True)
    d = N.to_diagram(N.parse_circuit(c), True)
    assert (d.slot_count, d.n_closed) == (rp.n_slots, rp.n_closed) == (311, 516)
    for j in range(d.slot_count):
        legs, data = rp.slot_tensor(j)
        assert legs == d.slot_tensors[j].legs
        assert np.array_equal(data.view(np.float64), d.slot_tensors[j].data.view(np.float64))
