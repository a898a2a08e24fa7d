"""Generate the golden fixtures from the UNMODIFIED reference (oracle/_ref).

Each case stores its inputs in the reference's own text formats (circuit,
bitstrings, plan, fuse flag) and the reference's outputs: eval_all /
eval_sliced amplitudes (complex128, exact via float.hex), node_contractions
and OpCounters, plus the reference's validation errors for malformed inputs.
tests/test_oracle.py pins the C oracle (and network.py) to these files; the GPU
box never needs /root/reference.

Usage: python tests/golden/make_golden.py
"""
from __future__ import annotations

import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import refimpl as R  # noqa: E402
from workloads import network as N  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden", "reference_cases.json")


def hexc(z) -> list:
    return [float(z.real).hex(), float(z.imag).hex()]


def case(name, circuit, bits, plan, fuse, mode="auto"):
    p = R.RefProblem(circuit, bits, plan, fuse=fuse)
    out = {"name": name, "circuit": circuit, "bits": bits, "plan": plan, "fuse": fuse,
           "mode": mode}
    try:
        v, nc, cnt, peak = p.eval(mode)
        out.update(status=0, amplitudes=[hexc(z) for z in v.ravel()],
                   node_contractions=[int(x) for x in nc], counters=list(cnt),
                   batch_legs=p.batch_legs(), peak_bytes=int(peak))
    except R.RefError as e:
        out.update(status=e.code, message=str(e))
    return out


def random_case(seed):
    rng = N.Rng(seed * 7919 + 17)
    n = 2 + rng.uniform_index(5)
    c = N.random_circuit(rng, n, 18)
    fuse = seed % 2 == 0
    d = N.to_diagram(c, fuse)
    k = 1 + rng.uniform_index(10)
    bits = N.random_bitstrings(rng, n, k)
    if seed % 5 == 1:
        q = rng.uniform_index(n)
        bits = [b[:q] + "*" + b[q + 1:] for b in bits]
    plan = N.random_plan(rng, d.slot_count)
    if seed % 3 == 0 and d.n_closed > 0:
        ns = 1 + rng.uniform_index(3)
        legs = []
        while len(legs) < min(ns, d.n_closed):
            leg = rng.uniform_index(d.n_closed)
            if leg not in legs:
                legs.append(leg)
        plan.sliced = legs
    return case(f"random_{seed}", N.format_circuit(c), bits, N.format_plan(plan), fuse)


def main():
    ghz = "3\n0 h 0\n0 t 2\n1 cx 0 1\n2 cx 1 2\n3 h 0\n3 h 1\n"
    ghz_plan = "(((0 3) (1 5)) ((2 4) (6 8))) 7\nslice:\n"
    cases = [
        case("worked_example", ghz, ["000", "100", "111"], ghz_plan, False, "all"),
        case("duplicates", ghz, ["101", "101", "101"], ghz_plan, False, "all"),
        case("sliced_h", "1\n0 h 0\n", ["0"], "0 1\nslice: 0\n", False, "sliced"),
        case("batch", "3\n0 h 0\n0 h 2\n1 cx 0 1\n2 fs 1 2 0.7 0.3\n", ["0*0", "1*1"],
             N.format_plan(N.left_deep_plan(7)), False, "all"),
        case("empty_requests", ghz, [], ghz_plan, False, "all"),
        case("lone_leaf", "1\n", ["0", "1"], "(0)\n", False, "all"),
        # reference error behaviour (multieval.cpp:284-348, plan.cpp:201-259)
        case("err_sliced_in_eval_all", "1\n0 h 0\n", ["0"], "0 1\nslice: 0\n", False, "all"),
        case("err_unsliced_in_eval_sliced", "1\n0 h 0\n", ["0"], "0 1\n", False, "sliced"),
        case("err_sliced_twice", "1\n0 h 0\n", ["0"], "0 1\nslice: 0 0\n", False, "sliced"),
        case("err_open_leg_sliced", "1\n0 h 0\n", ["0"], "0 1\nslice: 1\n", False, "sliced"),
        case("err_missing_leg_sliced", "1\n0 h 0\n", ["0"], "0 1\nslice: 7\n", False, "sliced"),
        case("err_slot_twice", ghz, ["000"], "(((0 3) (1 5)) ((2 4) (6 8))) 0\n", False, "all"),
        case("err_slot_range", ghz, ["000"], "(((0 3) (1 5)) ((2 4) (6 8))) 9\n", False, "all"),
        case("err_missing_slot", ghz, ["000"], "(((0 3) (1 5)) ((2 4) (6 8)))\n", False, "all"),
    ]
    cases += [random_case(s) for s in range(40)]
    c1 = N.format_circuit(N.grid_circuit(3, 4, 8, 12345))
    bits1 = N.random_bitstrings(N.Rng(99), 12, 1000)
    cases.append(case("cfg1", c1, bits1, open(os.path.join(ROOT, "plans", "cfg1.plan")).read(),
                      True, "auto"))
    # linear_xeb known answers (xeb_test.cpp:26-66)
    xeb = {
        "uniform_n4": R.linear_xeb(4, [1 / 16] * 16),
        "single_p_2^(1-n)_n4": R.linear_xeb(4, [2.0 ** -3]),
        "cfg1_probs": R.linear_xeb(12, [float.fromhex(a) ** 2 + float.fromhex(b) ** 2
                                        for a, b in cases[-1]["amplitudes"]]),
    }
    with open(OUT, "w") as f:
        json.dump({"generator": "tests/golden/make_golden.py (oracle/_ref = reference "
                                "/root/reference/proj compiled by oracle/Makefile)",
                   "cases": cases, "xeb": {k: float(v).hex() for k, v in xeb.items()}}, f)
    print(f"{len(cases)} cases -> {OUT} ({os.path.getsize(OUT) / 1e3:.0f} kB)")


if __name__ == "__main__":
    main()
