"""The C oracle pinned to the reference: golden vectors from the reference's own
tests, fixtures produced by the reference itself (tests/golden/
reference_cases.json, made by tests/golden/make_golden.py from oracle/_ref) —
bit-exact complex128 — and, in this container, live reference runs."""
import json
import math
import os

import numpy as np
import pytest

from oracle import oracle as O
from oracle import refimpl
from paper_2108_05665_b200 import _abi as A
from workloads import network as N
from paper_2108_05665_b200.engine import problem_arrays

from .helpers import GHZ_CIRCUIT, GHZ_PLAN, GOLDEN_AMP, ROOT, random_instance

CASES = json.load(open(os.path.join(ROOT, "tests", "golden", "reference_cases.json")))
MODES = {"auto": A.MTCG_EVAL_AUTO, "all": A.MTCG_EVAL_ALL, "sliced": A.MTCG_EVAL_SLICED}


def problem_of(case):
    c = N.parse_circuit(case["circuit"])
    d = N.to_diagram(c, case["fuse"])
    asg = N.build_assignments(d, case["bits"], N.batch_legs_of(d, case["bits"]))
    return problem_arrays(N.parse_plan(case["plan"]), d, asg), c


def unhex(pairs):
    return np.array([complex(float.fromhex(a), float.fromhex(b)) for a, b in pairs],
                    dtype=np.complex128)


@pytest.mark.parametrize("case", CASES["cases"], ids=lambda c: c["name"])
def test_oracle_matches_reference_fixture(case):
    try:
        p, _ = problem_of(case)
    except Exception as e:  # noqa: BLE001 — plan parse errors etc. must match too
        assert case["status"] != 0, e
        return
    if case["status"]:
        with pytest.raises(O.OracleError) as ei:
            O.eval_problem(p, MODES[case["mode"]])
        assert ei.value.code == case["status"]
        assert str(ei.value) == case["message"]
        return
    v, nc, cnt, legs = O.eval_problem(p, MODES[case["mode"]])
    want = unhex(case["amplitudes"])
    assert np.array_equal(v.ravel().view(np.float64), want.view(np.float64))
    assert [int(x) for x in nc] == case["node_contractions"]
    assert list(cnt) == case["counters"]


def test_worked_example_golden_vector():
    # multieval_test.cpp:74-116: amplitudes 1/(2 sqrt 2), node counts 1/2/3, 13 total
    c = N.parse_circuit(GHZ_CIRCUIT)
    d = N.to_diagram(c, False)
    p = problem_arrays(N.parse_plan(GHZ_PLAN), d, N.build_assignments(d, ["000", "100", "111"], []))
    v, nc, cnt, _ = O.eval_problem(p, A.MTCG_EVAL_ALL)
    assert np.all(np.abs(v - GOLDEN_AMP) < 1e-12)
    assert int(nc.sum()) == 13 and int(nc[p.root]) == 3


def test_sliced_h_golden_vector():
    # multieval_test.cpp:285-294
    c = N.parse_circuit("1\n0 h 0\n")
    d = N.to_diagram(c, False)
    p = problem_arrays(N.parse_plan("0 1\nslice: 0\n"), d, N.build_assignments(d, ["0"], []))
    v, _, _, _ = O.eval_problem(p, A.MTCG_EVAL_SLICED)
    assert abs(v[0, 0] - 1 / math.sqrt(2)) < 1e-12


def test_linear_xeb_known_answers():
    x = {k: float.fromhex(v) for k, v in CASES["xeb"].items()}
    assert O.linear_xeb(4, [1 / 16] * 16) == x["uniform_n4"]
    assert O.linear_xeb(4, [2.0 ** -3]) == x["single_p_2^(1-n)_n4"]
    cfg1 = [c for c in CASES["cases"] if c["name"] == "cfg1"][0]
    amps = unhex(cfg1["amplitudes"])
    probs = [a.real * a.real + a.imag * a.imag for a in amps]
    assert O.linear_xeb(12, probs) == x["cfg1_probs"]
    with pytest.raises(O.OracleError):
        O.linear_xeb(3, [])
    with pytest.raises(O.OracleError):
        O.linear_xeb(3, [0.5, -0.1])


def test_slice_ranges_partition_the_fold():
    p, _, _ = random_instance(3)
    full = O.eval_problem(p)[0]
    S = 1 << len(p.sliced)
    parts = sum(O.eval_problem(p, slices=(s, s + 1))[0] for s in range(S))
    assert np.max(np.abs(parts - full)) <= 1e-14


@pytest.mark.skipif(not refimpl.available(), reason="reference build absent (GPU box)")
@pytest.mark.parametrize("seed", range(60))
def test_oracle_bit_exact_against_live_reference(seed):
    p, c, bits = random_instance(seed + 1000)
    circ = N.format_circuit(c)
    plan = N.format_plan(N.Plan(list(p.node_left), list(p.node_right), list(p.node_slot),
                                int(p.root), [int(x) for x in p.sliced]))
    fuse = (seed + 1000) % 2 == 0
    rp = refimpl.RefProblem(circ, bits, plan, fuse=fuse)
    rv, rnc, rcnt, _ = rp.eval("auto")
    # re-pack from the plan text so node numbering is the parser's, as in the reference
    d = N.to_diagram(N.parse_circuit(circ), fuse)
    p = problem_arrays(N.parse_plan(plan), d, N.build_assignments(d, bits, N.batch_legs_of(d, bits)))
    v, nc, cnt, _ = O.eval_problem(p)
    assert np.array_equal(rv.view(np.float64), v.view(np.float64))
    assert np.array_equal(rnc, nc) and tuple(rcnt) == cnt
