"""Instance builders shared by the tests (no reference needed at run time)."""
from __future__ import annotations

import os
from typing import List, Optional, Tuple

import numpy as np

from workloads import network as N
from paper_2108_05665_b200._abi import ProblemArrays
from paper_2108_05665_b200.engine import problem_arrays

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

GHZ_CIRCUIT = "3\n0 h 0\n0 t 2\n1 cx 0 1\n2 cx 1 2\n3 h 0\n3 h 1\n"  # gen.cpp:109-112
GHZ_PLAN = "(((0 3) (1 5)) ((2 4) (6 8))) 7\nslice:\n"              # gen.cpp:114
GOLDEN_AMP = 0.35355339059327373                                    # multieval_test.cpp:74


def build(circuit: str, bits: List[str], plan: Optional[str] = None, fuse: bool = True,
          plan_obj: Optional[N.Plan] = None) -> Tuple[ProblemArrays, N.NetworkDiagram]:
    c = N.parse_circuit(circuit)
    d = N.to_diagram(c, fuse)
    asg = N.build_assignments(d, bits, N.batch_legs_of(d, bits))
    if plan_obj is None:
        plan_obj = N.parse_plan(plan) if plan else N.left_deep_plan(d.slot_count)
    return problem_arrays(plan_obj, d, asg), d


def random_instance(seed: int, max_qubits: int = 6, gates: int = 18, slices: bool = True,
                    batch: bool = True):
    """Random circuit + random plan + random bitstrings (+ sliced legs, batch
    leg), the pattern of multieval_test.cpp:118-283 / acceptance crit. 1-6."""
    rng = N.Rng(seed * 7919 + 17)
    n = 2 + rng.uniform_index(max_qubits - 1)
    c = N.random_circuit(rng, n, gates)
    d = N.to_diagram(c, seed % 2 == 0)
    k = 1 + rng.uniform_index(10)
    bits = N.random_bitstrings(rng, n, k)
    if batch and seed % 5 == 1:
        q = rng.uniform_index(n)
        bits = [b[:q] + "*" + b[q + 1:] for b in bits]
    asg = N.build_assignments(d, bits, N.batch_legs_of(d, bits))
    plan = N.random_plan(rng, d.slot_count)
    if slices and seed % 3 == 0 and d.n_closed > 0:
        ns = 1 + rng.uniform_index(3)
        legs: List[int] = []
        while len(legs) < min(ns, d.n_closed):
            leg = rng.uniform_index(d.n_closed)
            if leg not in legs:
                legs.append(leg)
        plan.sliced = legs
    return problem_arrays(plan, d, asg), c, bits


def workload(name: str) -> Tuple[ProblemArrays, N.Circuit, List[str]]:
    """cfg1 / cfg2 of BASELINE.json with the committed reference-annealed plans."""
    cfgs = {"cfg1": (3, 4, 8, 1000), "cfg2": (5, 6, 12, 10000)}
    r, cc, layers, k = cfgs[name]
    c = N.grid_circuit(r, cc, layers, 12345)
    bits = N.random_bitstrings(N.Rng(99), r * cc, k)
    d = N.to_diagram(c, True)
    asg = N.build_assignments(d, bits, [])
    plan = N.parse_plan(open(os.path.join(ROOT, "plans", f"{name}.plan")).read())
    return problem_arrays(plan, d, asg), c, bits


def rel_err(got: np.ndarray, want: np.ndarray, n_qubits: int) -> float:
    """max |a_gpu - a_ref| / max(|a_ref|, 2^(-n/2))."""
    floor = 2.0 ** (-n_qubits / 2)
    return float(np.max(np.abs(got - want) / np.maximum(np.abs(want), floor))) if want.size else 0.0


def statevector_samples(name: str, k: int, seed: int):
    """cfg1-style workload with k bitstrings sampled from the circuit's exact
    output distribution (the pattern of the reference's XEB
    criterion, tests/acceptance_main.cpp:400-428: cumulative |amp|^2 over the
    bitstrings in index order, qubit 0 = most significant bit
    (support/oracle.cpp:162-167), u = uniform_real01 * total, lower_bound).
    The distribution is the C oracle's evaluation of all 2^n bitstrings.
    Returns (problem, circuit, bits, probs_of_bits, target F)."""
    from oracle import oracle as O

    cfgs = {"cfg1": (3, 4, 8)}
    r, cc, layers = cfgs[name]
    n = r * cc
    c = N.grid_circuit(r, cc, layers, 12345)
    d = N.to_diagram(c, True)
    plan = N.parse_plan(open(os.path.join(ROOT, "plans", f"{name}.plan")).read())
    every = [format(i, f"0{n}b") for i in range(1 << n)]
    amps, _, _, _ = O.eval_problem(problem_arrays(plan, d, N.build_assignments(d, every, [])))
    dist = (np.abs(amps.reshape(-1)) ** 2).astype(np.float64)
    cum = np.cumsum(dist)
    rng = N.Rng(seed)
    idx = [min(int(np.searchsorted(cum, rng.uniform_real01() * cum[-1], side="left")), len(dist) - 1)
           for _ in range(k)]
    bits = [every[i] for i in idx]
    target = float((1 << n) * np.sum(dist * dist) - 1.0)
    p = problem_arrays(plan, d, N.build_assignments(d, bits, []))
    return p, c, bits, dist[idx], target
