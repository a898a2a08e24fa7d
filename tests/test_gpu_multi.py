"""Multi-GPU behind the C ABI, on one GPU (the reference's
workers contract, multieval.hpp:64-68, multieval_test.cpp:277-281):

* mtcg_run_slices_out + mtcg_fold (the per-rank half and the root half of
  the deterministic multi-GPU step) reproduce mtcg_run bit for bit;
* an mtcg_create_multi handle over 1, 2, 3 and 4 "virtual" devices (one GPU
  listed repeatedly: the same per-device schedule, device-to-device copies in
  place of NCCL) evaluates bit-identically to a single-device handle, and in
  complex128 bit-identically to the C oracle (= the reference);
* EvalOptions.workers caps the devices used.
"""
import numpy as np
import pytest
import torch

from oracle import oracle as O
from paper_2108_05665_b200 import _abi as A
from paper_2108_05665_b200.engine import Engine, EvalOptions

from .helpers import random_instance, workload

pytestmark = pytest.mark.gpu


def bits_equal(a, b):
    return np.array_equal(np.ascontiguousarray(a).view(np.float64), np.ascontiguousarray(b).view(np.float64))


@pytest.mark.parametrize("precision", ["c64", "c128"])
def test_slices_out_then_fold_equals_run(engine, precision):
    p, c, _ = workload("cfg2")
    cp = engine.compile(p, A.MTCG_EVAL_AUTO, EvalOptions(precision=precision))
    S = cp.n_slices
    acc = cp.new_accumulator()
    cp.run(0, S, acc.data_ptr())
    want = cp.fetch(acc.data_ptr()).amplitudes
    parts = cp.new_slice_buffer(S)
    cp.run_slices_out(0, S, parts.data_ptr())
    acc2 = cp.new_accumulator()
    cp.fold(parts.data_ptr(), S, acc2.data_ptr())
    assert bits_equal(cp.fetch(acc2.data_ptr()).amplitudes, want)
    # two halves folded into one accumulator (accumulate=True) — same bits
    acc3 = cp.new_accumulator()
    cp.fold(parts.data_ptr(), S // 2, acc3.data_ptr())
    half = parts[S // 2:].contiguous()
    cp.fold(half.data_ptr(), S - S // 2, acc3.data_ptr(), accumulate=True)
    assert bits_equal(cp.fetch(acc3.data_ptr()).amplitudes, want)
    # one slice's values are the slice alone
    one = cp.new_accumulator()
    cp.run(3, 4, one.data_ptr())
    assert torch.equal(one, parts[3])


@pytest.mark.parametrize("n_dev", [2, 3, 4])
def test_multi_device_handle_bit_identical(engine, n_dev):
    p, c, _ = workload("cfg2")
    single = engine.eval(p, A.MTCG_EVAL_AUTO, EvalOptions(precision="c64"))
    multi = Engine(devices=[0] * n_dev)
    got = multi.eval(p, A.MTCG_EVAL_AUTO, EvalOptions(precision="c64", workers=0))
    assert bits_equal(got.amplitudes, single.amplitudes)
    assert np.array_equal(got.node_contractions, single.node_contractions)
    assert (got.counters.mults, got.counters.rw) == (single.counters.mults, single.counters.rw)


@pytest.mark.parametrize("seed", [0, 3, 6, 9, 12])
def test_multi_device_c128_matches_oracle(seed):
    p, _, _ = random_instance(seed)
    want = O.eval_problem(p)[0]
    multi = Engine(devices=[0, 0, 0])
    for workers in (0, 1, 2):
        got = multi.eval(p, A.MTCG_EVAL_AUTO, EvalOptions(precision="c128", workers=workers))
        assert bits_equal(got.amplitudes, want), workers


def test_device_count_and_bad_device():
    from paper_2108_05665_b200._lib import lib
    from paper_2108_05665_b200.errors import DataError

    m = Engine(devices=[0, 0])
    assert lib().mtcg_device_count(m.h) == 2
    assert lib().mtcg_visible_devices() >= 1
    with pytest.raises(DataError, match="not visible"):
        Engine(devices=[0, 999])


@pytest.mark.parametrize("n_dev", [2, 4])
def test_fewer_slices_than_devices_split_requests(engine, n_dev):
    """S < devices (cfg1: one slice): the requests are split over the devices
    in lexicographic blocks (SURVEY §8e fallback) — complex128 bit-identical
    to the oracle, counts and node_contractions the whole evaluation's;
    complex64 within tolerance of one device."""
    p, c, _ = workload("cfg1")
    want, want_nc, want_cnt, _ = O.eval_problem(p)
    multi = Engine(devices=[0] * n_dev)
    got = multi.eval(p, A.MTCG_EVAL_AUTO, EvalOptions(precision="c128", workers=0))
    assert bits_equal(got.amplitudes, want)
    assert np.array_equal(got.node_contractions, want_nc)
    assert (got.counters.mults, got.counters.adds, got.counters.rw) == tuple(int(x) for x in want_cnt)
    single = engine.eval(p, A.MTCG_EVAL_AUTO, EvalOptions(precision="c64"))
    g64 = multi.eval(p, A.MTCG_EVAL_AUTO, EvalOptions(precision="c64", workers=0))
    floor = 2.0 ** (-c.n_qubits / 2)
    assert np.max(np.abs(g64.amplitudes - single.amplitudes) / np.maximum(np.abs(single.amplitudes), floor)) <= 1e-5
