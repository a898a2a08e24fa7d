"""Slice scheduler across GPUs: one process per GPU, one NCCL collective.

The reference folds per-slice results in slice-index order on one host
(multieval.cpp:478-513, worker w takes idx = w, w+W, ...). Here slices are
split into contiguous blocks, one per rank; each rank folds its block in
increasing slice index into a device accumulator (mtcg_run) and the partial
amplitudes are summed by a single reduce to rank 0 (NCCL over NVLink on the
GPU box; any torch.distributed backend works — the CPU tests use gloo). Rank 0
then runs the fused |amp|^2 -> XEB reduction on the summed accumulator.
"""
from __future__ import annotations

from typing import Callable, Optional, Tuple


def slice_range(n_slices: int, rank: int, world: int) -> Tuple[int, int]:
    """Contiguous, balanced block of [0, n_slices) owned by `rank`."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    return n_slices * rank // world, n_slices * (rank + 1) // world


class SliceScheduler:
    """Runs one rank's share of a compiled problem and combines partials.

    `run_partial(s0, s1, acc)` fills `acc` (a torch tensor) with the fold of
    slices [s0, s1) — CompiledProblem.run on a GPU, or any host callable in
    tests. `acc` must be zero-filled-by-overwrite semantics: the first slice
    of the range overwrites it; an empty range leaves zeros.
    """

    def __init__(self, n_slices: int, rank: int = 0, world: int = 1,
                 run_partial: Optional[Callable] = None, group=None):
        self.n_slices = n_slices
        self.rank, self.world = rank, world
        self.s0, self.s1 = slice_range(n_slices, rank, world)
        self.run_partial = run_partial
        self.group = group

    def step(self, acc) -> None:
        if self.s1 > self.s0:
            self.run_partial(self.s0, self.s1, acc)
        else:
            acc.zero_()
        if self.world > 1:
            import torch.distributed as dist

            dist.reduce(acc, dst=0, group=self.group)

    @staticmethod
    def for_compiled(cp, rank: int = 0, world: int = 1, stream: int = 0, group=None):
        def run(s0, s1, acc):
            cp.run(s0, s1, acc.data_ptr(), accumulate=False, stream=stream)

        return SliceScheduler(cp.n_slices, rank, world, run, group)
