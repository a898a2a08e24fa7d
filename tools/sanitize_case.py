"""Small cases for compute-sanitizer (memcheck / racecheck / synccheck):
the worked example and cfg1 (every CUDA-core kernel class, complex64 and
complex128), then one slice of cfg2 with the tensor-core path restricted to
the ops listed in MTCG_TC_ONLY (default: 311, a whole-K split-integer GEMM;
279, the pre-quantized CTA-pair GEMM). Exits non-zero on a parity failure.

    compute-sanitizer --tool memcheck python tools/sanitize_case.py
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("MTCG_TC_ONLY", "311,279")
os.environ.setdefault("MTCG_NO_GRAPHS", "1")  # launch kernels directly (per-launch reports)

from oracle import oracle as O  # noqa: E402
from paper_2108_05665_b200 import _abi as A  # noqa: E402
from paper_2108_05665_b200.engine import Engine, EvalOptions  # noqa: E402
from tests.helpers import rel_err, workload  # noqa: E402

eng = Engine(0)
p1, c1, _ = workload("cfg1")
want1 = O.eval_problem(p1)[0]
for prec in ("c64", "c128"):
    got = eng.eval(p1, A.MTCG_EVAL_AUTO, EvalOptions(precision=prec)).amplitudes
    e = rel_err(got, want1, c1.n_qubits)
    print(f"cfg1 {prec}: max rel {e:.2e}")
    assert e <= (1e-4 if prec == "c64" else 1e-12)
p2, c2, _ = workload("cfg2")
cp = eng.compile(p2, A.MTCG_EVAL_AUTO, EvalOptions(precision="c64"))
tc = [oi.node for oi in cp.op_infos() if oi.kernel == 12]
acc = cp.new_accumulator()
cp.run(0, 1, acc.data_ptr())
got = cp.fetch(acc.data_ptr()).amplitudes
cx = eng.compile(p2, A.MTCG_EVAL_AUTO, EvalOptions(precision="c128"))
accx = cx.new_accumulator()
cx.run(0, 1, accx.data_ptr())
want = cx.fetch(accx.data_ptr()).amplitudes
e = rel_err(got, want, c2.n_qubits)
print(f"cfg2 slice 0, tensor-core ops {tc}: max rel {e:.2e}")
assert e <= 1e-4 and tc
print("sanitize case ok")
