"""Memo streaming (EvalOptions.row_chunk, mtcg_options.row_chunk): requests
in lexicographic chunks, request-independent subtrees once per slice for all
chunks (the reference bounds its memory with
a one-entry left cache and per-node right dictionaries, multieval.cpp:213-274).
Values must not depend on the chunking: complex128 bit-identical to the C
oracle (= the reference) for every chunk size; counters / node_contractions
are the whole evaluation's; a plan whose memo tables exceed a memory cap runs
chunked where the unchunked schedule raises MemoryCapError."""
import numpy as np
import pytest

from oracle import oracle as O
from paper_2108_05665_b200 import _abi as A
from paper_2108_05665_b200.engine import EvalOptions, emulate_arrays
from paper_2108_05665_b200.errors import MemoryCapError

from .helpers import random_instance, rel_err, workload

pytestmark = pytest.mark.gpu


def bits_equal(a, b):
    return np.array_equal(np.ascontiguousarray(a).view(np.float64), np.ascontiguousarray(b).view(np.float64))


@pytest.mark.parametrize("seed", [0, 1, 3, 6, 9, 11, 12, 15])
@pytest.mark.parametrize("chunk", [1, 2, 3])
def test_chunked_random_instances_c128(engine, seed, chunk):
    p, _, _ = random_instance(seed)
    want, want_nc, want_cnt, _ = O.eval_problem(p)
    got = engine.eval(p, A.MTCG_EVAL_AUTO, EvalOptions(precision="c128", row_chunk=chunk))
    assert bits_equal(got.amplitudes, want)
    assert np.array_equal(got.node_contractions, want_nc)


@pytest.mark.parametrize("chunk", [1, 37, 250, 999])
def test_chunked_cfg1_c128_matches_oracle(engine, chunk):
    p, c, _ = workload("cfg1")
    want, want_nc, _, _ = O.eval_problem(p)
    got = engine.eval(p, A.MTCG_EVAL_AUTO, EvalOptions(precision="c128", row_chunk=chunk))
    assert bits_equal(got.amplitudes, want)
    assert np.array_equal(got.node_contractions, want_nc)


def test_chunked_cfg2_c64(engine):
    p, c, _ = workload("cfg2")
    base = engine.eval(p, A.MTCG_EVAL_AUTO, EvalOptions(precision="c64"))
    got = engine.eval(p, A.MTCG_EVAL_AUTO, EvalOptions(precision="c64", row_chunk=2500))
    assert rel_err(got.amplitudes, base.amplitudes, c.n_qubits) <= 1e-4
    assert np.array_equal(got.node_contractions, base.node_contractions)
    assert (got.counters.mults, got.counters.rw) == (base.counters.mults, base.counters.rw)


def test_chunking_runs_under_a_cap_the_whole_schedule_exceeds(engine):
    p, c, _ = workload("cfg1")
    info = emulate_arrays(p, EvalOptions(precision="c128")).plan_info
    # the whole schedule's need: arena + leaves + the root accumulators
    need = int(info.hbm_arena_bytes) + int(info.hbm_resident_bytes) + 2 * int(info.n_rows * info.row_elems) * 16
    cap = None
    for frac in [1 - 0.02 * i for i in range(1, 40)]:  # the largest cap the whole schedule exceeds
        try:
            engine.eval(p, A.MTCG_EVAL_AUTO, EvalOptions(precision="c128", memory_cap_bytes=int(need * frac)))
        except MemoryCapError:
            cap = int(need * frac)
            break
    assert cap is not None
    want, _, _, _ = O.eval_problem(p)
    got = engine.eval(p, A.MTCG_EVAL_AUTO, EvalOptions(precision="c128", memory_cap_bytes=cap, row_chunk=10))
    assert bits_equal(got.amplitudes, want)


@pytest.mark.parametrize("seed", [3, 6, 15])
def test_chunked_staged_api(engine, seed):
    """mtcg_compile with row_chunk: run slice ranges into one accumulator
    (chunks back to back), fetch, fused XEB — as the unchunked plan."""
    p, c, _ = random_instance(seed)
    want, want_nc, _, _ = O.eval_problem(p)
    cp = engine.compile(p, A.MTCG_EVAL_AUTO, EvalOptions(precision="c128", row_chunk=2))
    S = cp.n_slices
    acc = cp.new_accumulator()
    cp.run(0, S // 2 if S > 1 else S, acc.data_ptr())
    if S > 1:
        cp.run(S // 2, S, acc.data_ptr(), accumulate=True)
    r = cp.fetch(acc.data_ptr())
    assert bits_equal(r.amplitudes, want)
    assert np.array_equal(r.node_contractions, want_nc)
    f = cp.xeb(acc.data_ptr(), c.n_qubits)
    f_ref = O.linear_xeb(c.n_qubits, (np.abs(want) ** 2).ravel())
    assert abs(f - f_ref) <= 1e-12 * max(1.0, abs(f_ref))
