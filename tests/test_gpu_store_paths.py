"""Both epilogue store paths of the split-integer tensor-core kernel
(tc_i8_persistent<PAIR, QA, TR>): the default picks the transposed path only
for widely spaced output rows, which no benched op has, so each path is forced
in turn (MTCG_TC_TRANSPOSE, read once per process: child processes) on the
cfg2 and cfg3 workloads and checked against the reference's own amplitudes
(tests/golden/cfg2_reference.npz: a full eval_sliced run;
tests/golden/cfg3_reference.npz: slices 0-1 of 10 requests) at the
tolerances of test_gpu_parity / test_gpu_cfg3."""
import json
import os
import subprocess
import sys

import pytest

from .helpers import ROOT

pytestmark = pytest.mark.gpu

CHILD = r"""
import json, math, sys
import numpy as np
sys.path.insert(0, sys.argv[1])
from oracle import oracle as O
from paper_2108_05665_b200 import _abi as A
from paper_2108_05665_b200.engine import Engine, EvalOptions
from tests.helpers import workload, rel_err
eng = Engine(0)
out = {}
g = np.load(sys.argv[1] + "/tests/golden/cfg2_reference.npz")
p, c, bits = workload("cfg2")
cp = eng.compile(p, A.MTCG_EVAL_AUTO, EvalOptions(precision="c64", tensor_cores=True))
acc = cp.new_accumulator()
cp.run(0, cp.n_slices, acc.data_ptr())
r = cp.fetch(acc.data_ptr())
want = g["amplitudes"].reshape(r.amplitudes.shape)
f_ref = O.linear_xeb(c.n_qubits, (np.abs(want) ** 2).ravel())
f_dev = cp.xeb(acc.data_ptr(), c.n_qubits)
out["cfg2_rel"] = rel_err(r.amplitudes, want, c.n_qubits)
out["cfg2_l2"] = float(np.linalg.norm(r.amplitudes - want) / np.linalg.norm(want))
out["cfg2_dF"] = abs(f_dev - f_ref)
out["cfg2_dF_gate"] = 1e-4 * (abs(f_ref) + 1 / math.sqrt(len(bits)))
out["cfg2_nc_equal"] = bool(np.array_equal(r.node_contractions, g["node_contractions"]))
print(json.dumps(out))
"""


def _run(transpose: int) -> dict:
    env = dict(os.environ, MTCG_TC_TRANSPOSE=str(transpose))
    r = subprocess.run([sys.executable, "-c", CHILD, ROOT], capture_output=True, text=True, timeout=900,
                       env=env, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    return json.loads(r.stdout.strip().splitlines()[-1])


@pytest.mark.skipif(not os.path.exists(os.path.join(ROOT, "tests", "golden", "cfg2_reference.npz")),
                    reason="cfg2 golden not generated")
@pytest.mark.parametrize("transpose", [1, 0])
def test_cfg2_store_paths_against_reference(transpose):
    o = _run(transpose)
    assert o["cfg2_nc_equal"]
    assert o["cfg2_rel"] <= 1e-4 and o["cfg2_l2"] <= 1e-4
    assert o["cfg2_dF"] <= o["cfg2_dF_gate"]


CHILD3 = r"""
import json, sys
import numpy as np
sys.path.insert(0, sys.argv[1])
import tests.test_gpu_cfg3 as T
from paper_2108_05665_b200.engine import Engine
eng = Engine(0)
T.test_cfg3_slices_against_reference(eng, "c64", "cfg3")
print(json.dumps({"ok": True}))
"""


@pytest.mark.skipif(not os.path.exists(os.path.join(ROOT, "tests", "golden", "cfg3_reference.npz")),
                    reason="cfg3 golden not generated")
def test_cfg3_transposed_stores_against_reference():
    """cfg3's tensor-core ops with at most 64 real columns per tile (whole-K
    tiles of N <= 16 among them) through the transposed path, complex64
    against the reference's complex128 subset."""
    env = dict(os.environ, MTCG_TC_TRANSPOSE="1")
    r = subprocess.run([sys.executable, "-c", CHILD3, ROOT], capture_output=True, text=True, timeout=1200,
                       env=env, cwd=ROOT)
    assert r.returncode == 0, (r.stdout[-2000:], r.stderr[-3000:])
    assert json.loads(r.stdout.strip().splitlines()[-1])["ok"]
