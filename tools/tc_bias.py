"""Relative error / bias of the complex64 device path against the bit-exact
complex128 path on cfg2 slices [0, 2): max relative error, relative L2 and
the mean of Re(a64 / a128) - 1 (a systematic scale error shows up there)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2108_05665_b200.engine import Engine, EvalOptions  # noqa: E402
from tests.helpers import rel_err, workload  # noqa: E402


def run(eng, p, opts):
    cp = eng.compile(p, 0, opts)
    acc = cp.new_accumulator()
    cp.run(0, 2, acc.data_ptr())
    return cp.fetch(acc.data_ptr()).amplitudes.ravel()


if __name__ == "__main__":
    p, c, _ = workload("cfg2")
    eng = Engine(0)
    exact = run(eng, p, EvalOptions(precision="c128"))
    got = run(eng, p, EvalOptions(precision="c64", tensor_cores=os.environ.get("TC", "1") == "1"))
    big = np.abs(exact) > 2.0 ** (-c.n_qubits / 2)
    ratio = got[big] / exact[big]
    print(f"{os.environ.get('MTCG_TC_ONLY', 'all')}: max rel {rel_err(got, exact, c.n_qubits):.3e} "
          f"L2 {np.linalg.norm(got - exact) / np.linalg.norm(exact):.3e} "
          f"bias {np.mean(ratio.real) - 1:+.3e} (std {np.std(ratio.real):.2e})")
