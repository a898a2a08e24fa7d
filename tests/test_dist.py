"""Multi-process slice scheduling on CPU (gloo, world_size 1, 2 and 3): the
same SliceScheduler the bench uses on NVLink/NCCL — contiguous slice blocks
per rank, then either one all-gather of per-slice values and an ordered fold
on rank 0 (default; bit-identical for every world size, the reference's
workers contract, multieval.hpp:64-68) or one reduce of per-rank partials —
with the C oracle standing in for each rank's device (per-slice values /
block folds; the GPU tests run the engine's own mtcg_run_slices_out +
mtcg_fold and the in-library multi-device handle).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2108_05665_b200.scheduler import SliceScheduler, slice_range


def test_slice_ranges_cover_every_slice_once():
    for S in (1, 2, 16, 17, 1 << 10):
        for world in (1, 2, 3, 8):
            seen = []
            for r in range(world):
                s0, s1 = slice_range(S, r, world)
                seen.extend(range(s0, s1))
            assert seen == list(range(S))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, seed, out, mode="reduce"):
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from oracle import oracle as O
    from tests.helpers import random_instance

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    p, _, _ = random_instance(seed)
    S = 1 << len(p.sliced)

    def run_partial(s0, s1, acc):
        v = O.eval_problem(p, slices=(s0, s1))[0]
        acc.copy_(torch.from_numpy(np.ascontiguousarray(v).view(np.float64).reshape(acc.shape)))

    def run_out(s0, s1, parts):
        for i, sl in enumerate(range(s0, s1)):
            v = O.eval_problem(p, slices=(sl, sl + 1))[0]
            parts[i].copy_(torch.from_numpy(np.ascontiguousarray(v).view(np.float64).reshape(parts[i].shape)))

    def fold(parts, n, acc):
        a = parts[0].clone()
        for i in range(1, n):
            a = a + parts[i]  # one rounded add per slice, in slice order
        acc.copy_(a)

    acc = torch.zeros((p.n_requests, p.row_elems, 2), dtype=torch.float64)
    SliceScheduler(S, rank, world, run_partial, run_out=run_out, fold=fold, mode=mode).step(acc)
    if rank == 0:
        np.save(out, acc.numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sliced_partials_reduce_to_full_result(tmp_path, world):
    from oracle import oracle as O
    from tests.helpers import random_instance

    seed = 6  # sliced instance (seed % 3 == 0) with 2^k slices
    p, _, _ = random_instance(seed)
    assert len(p.sliced) >= 1
    out = str(tmp_path / "acc.npy")
    mp.spawn(_worker, args=(world, _free_port(), seed, out), nprocs=world, join=True)
    got = np.load(out).view(np.complex128).reshape(p.n_requests, p.row_elems)
    want = O.eval_problem(p)[0]
    assert np.max(np.abs(got - want)) <= 1e-14 * max(1.0, np.max(np.abs(want)))


@pytest.mark.parametrize("world", [1, 2, 3])
@pytest.mark.parametrize("seed", [6, 9])
def test_gather_fold_bit_identical_for_every_world_size(tmp_path, world, seed):
    """Gather mode: per-slice values all-gathered, folded on rank 0 in slice
    order — bit-identical to the single-process sequential fold for any rank
    count (the reference's workers=4 == workers=1 test,
    multieval_test.cpp:277-281)."""
    from oracle import oracle as O
    from tests.helpers import random_instance

    p, _, _ = random_instance(seed)
    assert len(p.sliced) >= 1
    out = str(tmp_path / "acc.npy")
    mp.spawn(_worker, args=(world, _free_port(), seed, out, "gather"), nprocs=world, join=True)
    got = np.load(out).view(np.complex128).reshape(p.n_requests, p.row_elems)
    want = O.eval_problem(p)[0]
    assert np.array_equal(got.view(np.float64), np.ascontiguousarray(want).view(np.float64))
