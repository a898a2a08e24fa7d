"""The reference's own types and test patterns with eval_all / eval_sliced /
linear_xeb swapped for the device engine through include/mtcg_mtc.hpp
(oracle/dropin_test.cpp, built against the reference in the dev container by
`make -C oracle dropin`; the binary travels to the GPU box)."""
import os
import subprocess

import pytest

from .helpers import ROOT

pytestmark = pytest.mark.gpu

BIN = os.path.join(ROOT, "oracle", "_ref", "dropin_test")


@pytest.mark.skipif(not os.path.exists(BIN), reason="drop-in binary not built")
def test_reference_tests_through_the_drop_in_header():
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "all drop-in criteria passed" in r.stdout
