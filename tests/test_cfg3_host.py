"""cfg3's / cfg4's exact algorithmic totals: the engine's shape replay
(mtcg_emulate) of the whole 10^4- / 10^5-bitstring evaluation equals the unmodified reference's
CostedPlan totals recorded with the golden amplitudes
(tests/golden/make_sycamore_reference.py; plan.cpp:497-502)."""
import os

import numpy as np
import pytest

from paper_2108_05665_b200.engine import EvalOptions, emulate_arrays

from .helpers import ROOT


@pytest.mark.parametrize("name", ["cfg3", "cfg4"])
def test_cfg3_counts_equal_reference(name):
    import bench
    path = os.path.join(ROOT, "tests", "golden", f"{name}_reference.npz")
    if not os.path.exists(path):
        pytest.skip(f"{path} not generated")
    g = np.load(path)
    p, _, _, _ = bench.load_workload(name)
    r = emulate_arrays(p, EvalOptions(precision="c128"))
    assert str(r.counters.mults) == str(g["mults_str"])
    assert str(r.counters.adds) == str(g["adds_str"])
    assert str(r.counters.rw) == str(g["rw_str"])
