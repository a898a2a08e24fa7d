"""The tcgen05 3xTF32 complex-GEMM path on the bench workload's dense nodes:
complex64 results (tensor cores on / off) against the bit-exact complex128
path over a slice range, and evidence that the tensor-core kernel ran."""
import ctypes as C

import numpy as np
import pytest

from paper_2108_05665_b200 import _abi as A
from paper_2108_05665_b200._lib import lib
from paper_2108_05665_b200.engine import EvalOptions

from .helpers import rel_err, workload

pytestmark = pytest.mark.gpu


from paper_2108_05665_b200._abi import mtcg_op_info as OpInfo  # the one ABI struct


def op_kernels(cp):
    L = lib()
    L.mtcg_plan_op_count.restype = C.c_int32
    L.mtcg_plan_op_count.argtypes = [C.c_void_p]
    L.mtcg_plan_op_info.argtypes = [C.c_void_p, C.c_int32, C.POINTER(OpInfo)]
    out = []
    for i in range(L.mtcg_plan_op_count(cp.h)):
        oi = OpInfo()
        L.mtcg_plan_op_info(cp.h, i, C.byref(oi))
        out.append((oi.node, oi.kernel, oi.fa, oi.fb, oi.kc))
    return out


def run_range(engine, p, opts, s0, s1):
    cp = engine.compile(p, A.MTCG_EVAL_AUTO, opts)
    acc = cp.new_accumulator()
    cp.run(s0, s1, acc.data_ptr())
    return cp, cp.fetch(acc.data_ptr()).amplitudes


def test_cfg2_tensor_core_path_matches_exact_path(engine):
    p, c, bits = workload("cfg2")
    cp_tc, tc = run_range(engine, p, EvalOptions(precision="c64"), 0, 2)
    kinds = op_kernels(cp_tc)
    tc_nodes = [k for k in kinds if k[1] == 12]
    assert any(k[0] == 279 for k in tc_nodes), "node 279 (M=2^15 N=2^11 K=2^10) not on tensor cores"
    _, cuda = run_range(engine, p, EvalOptions(precision="c64", tensor_cores=False), 0, 2)
    _, exact = run_range(engine, p, EvalOptions(precision="c128"), 0, 2)
    e_tc = rel_err(tc, exact, c.n_qubits)
    e_cuda = rel_err(cuda, exact, c.n_qubits)
    l2 = np.linalg.norm(tc - exact) / np.linalg.norm(exact)
    print(f"tensor cores: max rel {e_tc:.2e}, L2 {l2:.2e}; CUDA cores: max rel {e_cuda:.2e}")
    assert e_tc <= 1e-4 and l2 <= 1e-4
    assert e_cuda <= 1e-4


def test_gather_mode_matches_cuda_cores(engine, monkeypatch):
    """Tensor-core gather mode (node 349: 9,992 items of 32 x 32 x 128 sharing
    128 B entries, stacked 4 items per 128-row tile) against the same op on
    the CUDA-core tile kernel (MTCG_NO_GATHER=1), over a slice range."""
    p, c, bits = workload("cfg2")
    cp, ga = run_range(engine, p, EvalOptions(precision="c64"), 0, 2)
    assert any(k[0] == 349 and k[1] == 12 for k in op_kernels(cp)), "node 349 not in gather mode"
    monkeypatch.setenv("MTCG_NO_GATHER", "1")
    cp2, plain = run_range(engine, p, EvalOptions(precision="c64"), 0, 2)
    assert not any(k[0] == 349 and k[1] == 12 for k in op_kernels(cp2))
    _, exact = run_range(engine, p, EvalOptions(precision="c128"), 0, 2)
    e_ga, e_plain = rel_err(ga, exact, c.n_qubits), rel_err(plain, exact, c.n_qubits)
    print(f"gather mode: max rel {e_ga:.2e}; CUDA-core tile: {e_plain:.2e}")
    assert e_ga <= 1e-4 and np.linalg.norm(ga - exact) / np.linalg.norm(exact) <= 1e-4
