"""The engine across processes: two ranks (torch.multiprocessing, gloo over
the host, both on cuda:0 — the box has one GPU, and gloo keeps the ranks'
kernels independent of each other) run the bench's SliceScheduler with the
engine's own mtcg_run_slices_out per rank and mtcg_fold on rank 0. The folded
amplitudes must be bit-identical (c128) to one process's mtcg_run over all
slices and to the oracle — the reference's workers contract
(multieval.hpp:64-68) through the real device path."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, seed, out):
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from paper_2108_05665_b200.engine import Engine, EvalOptions
    from paper_2108_05665_b200.scheduler import SliceScheduler
    from tests.helpers import random_instance

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    p, _, _ = random_instance(seed)
    eng = Engine(0)
    cp = eng.compile(p, 0, EvalOptions(precision="c128"))
    S = cp.n_slices
    dev_acc = cp.new_accumulator()

    def run_out(s0, s1, parts):
        buf = cp.new_slice_buffer(s1 - s0)
        cp.run_slices_out(s0, s1, buf.data_ptr())
        torch.cuda.synchronize()
        parts[: s1 - s0].copy_(buf.cpu())

    def fold(parts, n, acc):
        d = parts[:n].cuda()
        cp.fold(d.data_ptr(), n, dev_acc.data_ptr())
        torch.cuda.synchronize()
        acc.copy_(dev_acc.cpu())

    acc = torch.zeros(tuple(dev_acc.shape), dtype=torch.float64)
    SliceScheduler(S, rank, world, run_out=run_out, fold=fold, mode="gather").step(acc)
    if rank == 0:
        np.save(out, acc.numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("seed", [6, 9, 12])
def test_engine_gather_fold_across_processes(tmp_path, seed):
    from oracle import oracle as O
    from paper_2108_05665_b200.engine import Engine, EvalOptions
    from tests.helpers import random_instance

    p, _, _ = random_instance(seed)
    assert len(p.sliced) >= 1
    out = str(tmp_path / "acc.npy")
    mp.spawn(_worker, args=(2, _free_port(), seed, out), nprocs=2, join=True)
    got = np.load(out)
    cp = Engine(0).compile(p, 0, EvalOptions(precision="c128"))
    acc = cp.new_accumulator()
    cp.run(0, cp.n_slices, acc.data_ptr())
    torch.cuda.synchronize()
    one = acc.cpu().numpy()
    assert np.array_equal(got, one)
    want = O.eval_problem(p)[0]
    assert np.array_equal(got.view(np.complex128).reshape(want.shape).view(np.float64),
                          np.ascontiguousarray(want).view(np.float64))
