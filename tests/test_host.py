"""Host side of the C ABI, no GPU: the library loads and exports every symbol
include/mtcg.h declares; mtcg_emulate (validation + tuple index + schedule)
reproduces the reference's counts, node_contractions and error behaviour."""
import ctypes as C
import json
import os
import re

import numpy as np
import pytest

from paper_2108_05665_b200 import _abi as A
from paper_2108_05665_b200._lib import EXPORTS, LIB_PATH, lib
from paper_2108_05665_b200.engine import EvalOptions, emulate_arrays
from paper_2108_05665_b200.errors import DataError, MemoryCapError

from .helpers import ROOT, random_instance, workload
from .test_oracle import CASES, MODES, problem_of


def test_library_loads_and_exports_every_declared_symbol():
    L = lib()
    header = open(os.path.join(ROOT, "include", "mtcg.h")).read()
    declared = set(re.findall(r"\b(mtcg_[a-z_]+)\s*\(", header))
    assert declared, "no declarations parsed"
    for sym in sorted(declared):
        assert hasattr(L, sym), sym
    assert set(EXPORTS) <= declared | {"mtcg_version"}
    assert L.mtcg_version() == 2


def test_library_is_an_in_tree_sm100a_build():
    import subprocess

    assert LIB_PATH.startswith(ROOT)
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


@pytest.mark.parametrize("case", [c for c in CASES["cases"]], ids=lambda c: c["name"])
def test_emulate_matches_reference_counts_and_errors(case):
    try:
        p, _ = problem_of(case)
    except Exception:  # noqa: BLE001
        assert case["status"] != 0
        return
    if case["status"]:
        with pytest.raises(DataError) as ei:
            emulate_arrays(p, mode=MODES[case["mode"]])
        assert str(ei.value) == case["message"]
        return
    em = emulate_arrays(p, mode=MODES[case["mode"]])
    assert [int(x) for x in em.node_contractions] == case["node_contractions"]
    assert [em.counters.mults, em.counters.adds, em.counters.rw] == case["counters"]


def test_emulate_cfg2_counts_match_reference_totals():
    # exact-mode CostedPlan totals of the bench workload (769,600
    # contractions, 1.585e12 complex MACs with the survey's annealed plan)
    p, _, _ = workload("cfg2")
    em = emulate_arrays(p)
    assert em.contractions == 769600
    assert em.counters.mults == 1584552545792  # CostedPlan exact total_mults
    golden = os.path.join(ROOT, "tests", "golden", "cfg2_reference.npz")
    if os.path.exists(golden):
        g = np.load(golden)
        assert np.array_equal(em.node_contractions, g["node_contractions"])
        assert (em.counters.mults, em.counters.adds, em.counters.rw) == tuple(int(x) for x in g["counters"])


def test_memory_cap_names_a_node():
    p, _, _ = random_instance(0)
    with pytest.raises(MemoryCapError) as ei:
        emulate_arrays(p, EvalOptions(memory_cap_bytes=64))
    assert "memory cap exceeded at node" in str(ei.value)
    assert 0 <= ei.value.node < p.n_nodes


def test_unsupported_bond_dimension_is_a_data_error():
    p, _, _ = random_instance(2)
    dims = np.array(p.leg_dims)
    dims[0] = 3
    q = A.ProblemArrays(p.node_left, p.node_right, p.node_slot, p.root, p.sliced, p.n_closed,
                        dims, p.slot_n_values, p.slot_leg_begin, p.slot_legs, p.values,
                        p.tuples, p.batch_legs)
    with pytest.raises(DataError, match="bond dimension"):
        emulate_arrays(q)


def test_request_tuple_out_of_range():
    p, _, _ = random_instance(4)
    t = p.tuples.copy()
    t[0, 0] = 99
    q = A.ProblemArrays(p.node_left, p.node_right, p.node_slot, p.root, p.sliced, p.n_closed,
                        p.leg_dims, p.slot_n_values, p.slot_leg_begin, p.slot_legs, p.values,
                        t, p.batch_legs)
    with pytest.raises(DataError, match="indexes past slot 0's value set"):
        emulate_arrays(q)


def test_device_entry_points_fail_loudly_without_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2108_05665_b200.engine import Engine
    from paper_2108_05665_b200.errors import EngineError

    with pytest.raises(EngineError):
        Engine(0)


# ---- device schedule built on the host (no GPU): slice reuse, fused chains ----


def test_slice_reuse_schedule_keeps_reference_counts():
    """MTCG_FLAG_SLICE_REUSE reorders the schedule (slice-invariant prologue)
    but every reference count is unchanged; cfg2 executes fewer contractions."""
    p, c, bits = workload("cfg2")
    base = emulate_arrays(p, EvalOptions())
    reuse = emulate_arrays(p, EvalOptions(slice_reuse=True))
    assert np.array_equal(base.node_contractions, reuse.node_contractions)
    assert base.counters == reuse.counters and base.contractions == reuse.contractions
    assert base.plan_info.prologue_ops == 0
    assert base.plan_info.executed_contractions == base.contractions
    assert reuse.plan_info.prologue_ops > 0
    assert reuse.plan_info.executed_contractions < reuse.contractions


def test_fused_chains_planned_and_switchable(monkeypatch):
    """cfg2's spine runs (e.g. nodes 301-305) become fused chains; counts are
    unaffected; MTCG_NO_CHAIN=1 turns them off; unsliced cfg1 has runs too."""
    p, c, bits = workload("cfg2")
    r = emulate_arrays(p, EvalOptions())
    assert r.plan_info.fused_chains >= 5
    assert r.plan_info.fused_ops >= 2 * r.plan_info.fused_chains
    monkeypatch.setenv("MTCG_NO_CHAIN", "1")
    off = emulate_arrays(p, EvalOptions())
    assert off.plan_info.fused_chains == 0 and off.plan_info.fused_ops == 0
    assert np.array_equal(off.node_contractions, r.node_contractions)
    assert off.counters == r.counters
    monkeypatch.delenv("MTCG_NO_CHAIN")
    p1, _, _ = workload("cfg1")
    assert emulate_arrays(p1, EvalOptions()).plan_info.fused_chains >= 1


@pytest.mark.parametrize("seed", range(0, 60, 7))
def test_schedule_flags_never_change_counts_on_random_instances(seed):
    p, c, bits = random_instance(seed)
    a = emulate_arrays(p, EvalOptions())
    b = emulate_arrays(p, EvalOptions(slice_reuse=True))
    assert np.array_equal(a.node_contractions, b.node_contractions)
    assert a.counters == b.counters
    assert b.plan_info.executed_contractions <= b.contractions


def test_memory_cap_accounting_differs_from_the_reference_as_documented():
    """the device arena counts 8 B per complex64 element over
    its own static schedule (leaves, tables, accumulators), the reference's
    Session 16 B per scalar over its recursion, so the smallest cap that runs
    differs between them. Pinned on cfg1: each side's threshold is found by
    bisection; below both, both raise MemoryCapError; between them, exactly
    the side with the larger threshold raises; above both, neither does."""
    from oracle import refimpl as R

    if not R.available():
        pytest.skip("reference library not built")
    from workloads import network as N
    from paper_2108_05665_b200.engine import problem_arrays

    c = N.grid_circuit(3, 4, 8, 12345)
    bits = N.random_bitstrings(N.Rng(99), 12, 1000)
    plan_text = open(os.path.join(os.path.dirname(__file__), "..", "plans", "cfg1.plan")).read()
    d = N.to_diagram(c, True)
    p = problem_arrays(N.parse_plan(plan_text), d, N.build_assignments(d, bits, []))
    ref = R.RefProblem(N.format_circuit(c), bits, plan_text, fuse=True)

    def dev_raises(cap):
        try:
            emulate_arrays(p, EvalOptions(precision="c64", memory_cap_bytes=cap))
            return False
        except MemoryCapError:
            return True

    def ref_raises(cap):
        try:
            ref.emulate(cap)
            return False
        except R.RefError as e:
            assert e.code == 3
            return True

    def threshold(raises):  # smallest cap that runs
        lo, hi = 1, 1 << 40
        assert raises(lo) and not raises(hi)
        while hi - lo > 1:
            mid = (lo + hi) // 2
            lo, hi = (mid, hi) if raises(mid) else (lo, mid)
        return hi

    t_dev, t_ref = threshold(dev_raises), threshold(ref_raises)
    assert t_dev != t_ref
    lo, hi = sorted((t_dev, t_ref))
    assert dev_raises(lo - 1) and ref_raises(lo - 1)
    mid = (lo + hi) // 2
    assert dev_raises(mid) == (t_dev > mid) and ref_raises(mid) == (t_ref > mid)
    assert not dev_raises(hi) and not ref_raises(hi)


def test_maximum_sizes_are_rejected_with_the_references_messages():
    """SURVEY §8(c) edge cases at the size limits: more than 2^24 slices is
    the reference's own DataError (multieval.cpp:345); an intermediate of
    order above 32 (the engine's 32-bit table offsets) is rejected up front
    instead of wrapping; exactly 2^24 slices is accepted."""
    from workloads import network as N
    from paper_2108_05665_b200.engine import problem_arrays

    c = N.grid_circuit(5, 6, 12, 12345)
    d = N.to_diagram(c, True)
    bits = N.random_bitstrings(N.Rng(99), 30, 4)
    plan = N.parse_plan(open(os.path.join(os.path.dirname(__file__), "..", "plans", "cfg2.plan")).read())
    asg = N.build_assignments(d, bits, [])
    plan.sliced = list(range(25))
    with pytest.raises(DataError) as e:
        emulate_arrays(problem_arrays(plan, d, asg), EvalOptions(precision="c64"))
    assert str(e.value) == "slice list expands to more than 2^24 slices"
    plan.sliced = list(range(24))
    info = emulate_arrays(problem_arrays(plan, d, asg), EvalOptions(precision="c64")).plan_info
    assert info.n_slices == 1 << 24
    # a left-deep tree over the 53-qubit m=12 network builds order > 32 nodes
    c53 = N.sycamore_circuit(12, 2024)
    d53 = N.to_diagram(c53, True)
    b53 = N.random_bitstrings(N.Rng(1), 53, 2)
    p53 = problem_arrays(N.left_deep_plan(d53.slot_count), d53, N.build_assignments(d53, b53, []))
    with pytest.raises(DataError) as e:
        emulate_arrays(p53, EvalOptions(precision="c64"))
    assert "order above 32" in str(e.value)
