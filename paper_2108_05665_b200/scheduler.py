"""Slice scheduler across GPUs: one process per GPU, one collective per step.

The reference folds per-slice results in slice-index order on one host
(multieval.cpp:478-513: worker w takes idx = w, w+W, ...; by_row =
per_slice[0], then add_into for idx = 1 .. S-1) and guarantees values that do
not depend on the worker count (multieval.hpp:64-68). Here the slices are
split into contiguous blocks, one per rank, and

  mode "gather" (default, deterministic): each rank writes its block's
    per-slice root values (mtcg_run_slices_out), one all-gather (NCCL over
    NVLink on the GPU box; gloo in the CPU tests) brings every slice to every
    rank, and rank 0 folds them in slice order (mtcg_fold) — the reference's
    fold, so the amplitudes are bit-identical for 1, 2, 4 or 8 GPUs;
  mode "reduce": each rank folds its own block into a partial accumulator
    (mtcg_run) and one reduce sums the partials on rank 0 — fewer bytes on
    the wire, but the grouping of the sum depends on the rank count.

Rank 0 then runs the fused |amp|^2 -> XEB reduction on the folded values.
The in-process multi-GPU handle (mtcg_create_multi, used by mtcg_eval and the
C++ drop-in) implements the same gather + ordered fold with NCCL
point-to-point inside libmtcg.
"""
from __future__ import annotations

from typing import Callable, Optional, Tuple


def slice_range(n_slices: int, rank: int, world: int) -> Tuple[int, int]:
    """Contiguous, balanced block of [0, n_slices) owned by `rank`."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    return n_slices * rank // world, n_slices * (rank + 1) // world


def max_block(n_slices: int, world: int) -> int:
    return max(slice_range(n_slices, r, world)[1] - slice_range(n_slices, r, world)[0]
               for r in range(world))


class SliceScheduler:
    """Runs one rank's share of a compiled problem and combines the ranks.

    gather mode: `run_out(s0, s1, parts)` writes slice s0 + i's root values
    into parts[i] (parts: (max_block, *acc.shape)); `fold(parts, n, acc)`
    sets acc = parts[0] + ... + parts[n - 1] in order.
    reduce mode: `run_partial(s0, s1, acc)` folds the block into acc (the
    first slice overwrites; an empty range leaves zeros).
    """

    def __init__(self, n_slices: int, rank: int = 0, world: int = 1,
                 run_partial: Optional[Callable] = None, group=None,
                 run_out: Optional[Callable] = None, fold: Optional[Callable] = None,
                 mode: str = "gather"):
        if mode not in ("gather", "reduce"):
            raise ValueError(f"unknown mode {mode}")
        self.n_slices = n_slices
        self.rank, self.world = rank, world
        self.s0, self.s1 = slice_range(n_slices, rank, world)
        self.run_partial = run_partial
        self.run_out, self.fold = run_out, fold
        self.group = group
        self.mode = mode
        self.block = max_block(n_slices, world)
        self._parts = None
        self._all = None

    def _buffers(self, acc):
        import torch

        if self._parts is None or self._parts.shape[1:] != acc.shape:
            self._parts = torch.zeros((self.block,) + tuple(acc.shape), dtype=acc.dtype, device=acc.device)
            self._all = (torch.zeros((self.world * self.block,) + tuple(acc.shape), dtype=acc.dtype,
                                     device=acc.device) if self.world > 1 else self._parts)
        return self._parts, self._all

    def step(self, acc) -> None:
        if self.mode == "reduce":
            if self.s1 > self.s0:
                self.run_partial(self.s0, self.s1, acc)
            else:
                acc.zero_()
            if self.world > 1:
                import torch.distributed as dist

                dist.reduce(acc, dst=0, group=self.group)
            return
        parts, allp = self._buffers(acc)
        if self.s1 > self.s0:
            self.run_out(self.s0, self.s1, parts)
        if self.world > 1:
            import torch.distributed as dist

            dist.all_gather_into_tensor(allp, parts, group=self.group)
        if self.rank != 0:
            return
        if self.world > 1:
            import torch

            # rank blocks are contiguous in slice order; drop each block's padding
            idx = [r * self.block + i for r in range(self.world)
                   for i in range(slice_range(self.n_slices, r, self.world)[1]
                                  - slice_range(self.n_slices, r, self.world)[0])]
            ordered = allp[torch.tensor(idx, device=allp.device)] if idx else allp[:0]
        else:
            ordered = parts[: self.s1 - self.s0]
        if self.n_slices:
            self.fold(ordered.contiguous(), self.n_slices, acc)
        else:
            acc.zero_()

    @staticmethod
    def for_compiled(cp, rank: int = 0, world: int = 1, stream: int = 0, group=None,
                     mode: str = "gather"):
        def run_partial(s0, s1, acc):
            cp.run(s0, s1, acc.data_ptr(), accumulate=False, stream=stream)

        def run_out(s0, s1, parts):
            cp.run_slices_out(s0, s1, parts.data_ptr(), stream=stream)

        def fold(parts, n, acc):
            cp.fold(parts.data_ptr(), n, acc.data_ptr(), accumulate=False, stream=stream)

        return SliceScheduler(cp.n_slices, rank, world, run_partial, group, run_out, fold, mode)
