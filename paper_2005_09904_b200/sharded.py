"""Multi-GPU BiQGEMM: weight rows sharded across ranks.

One process per GPU (torch.distributed; NCCL over NVLink on the B200 box).
The output dimension m is split into contiguous, 32-row-aligned blocks
(row tiles never straddle ranks, so every output's reduction tree -- and
therefore y -- is bitwise identical for any number of ranks).  Each rank
holds only its rows' packed keys and alphas, receives x by broadcast from
rank 0, runs the fused kernel on its rows, and the row blocks are assembled
with an all-gather.  Rows are independent (per-row alpha, paper Eq. 2), so no
reduction is ever needed; that is also why the reference partitions rows
across its worker threads (kernel.hpp:80-82,165-173).

The per-rank compute is pluggable only so the CPU (gloo) tests can exercise
the sharding/collective logic without a GPU; production code always passes
the CUDA path (``device_compute``), which fails loudly if the library is not
built.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Callable

import torch
import torch.distributed as dist

ROW_ALIGN = 32


def shard_bounds(m: int, world: int, align: int = ROW_ALIGN) -> list[int]:
    """Contiguous row blocks, boundaries on multiples of `align` (the last
    block absorbs the ragged tail).  len = world + 1, bounds[0] = 0,
    bounds[-1] = m; a rank may own zero rows when m is small."""
    tiles = (m + align - 1) // align
    out = []
    for r in range(world + 1):
        out.append(min(m, (tiles * r // world) * align))
    out[-1] = m
    return out


@dataclass
class ShardPlan:
    m: int
    world: int
    bounds: list[int]

    @classmethod
    def make(cls, m: int, world: int) -> "ShardPlan":
        return cls(m, world, shard_bounds(m, world))

    def rows(self, rank: int) -> tuple[int, int]:
        return self.bounds[rank], self.bounds[rank + 1]

    @property
    def max_rows(self) -> int:
        return max(self.bounds[r + 1] - self.bounds[r] for r in range(self.world))


class ShardedBiQGEMM:
    """Row-sharded y = sum_i alpha_i o (B_i . x) across a process group.

    compute(x_dev, y_local) must fill y_local [rows, b] for this rank's rows.
    """

    def __init__(self, plan: ShardPlan, rank: int, compute: Callable, group=None, device=None):
        self.plan = plan
        self.rank = rank
        self.compute = compute
        self.group = group
        self.device = device if device is not None else torch.device("cpu")

    def forward(self, x: torch.Tensor | None, n: int, b: int) -> torch.Tensor:
        """x: [n, b] on rank 0 (ignored elsewhere).  Returns the full y [m, b]
        on every rank."""
        world = self.plan.world
        xb = x.to(self.device).contiguous() if (self.rank == 0 and x is not None) else torch.empty(
            (n, b), dtype=torch.float32, device=self.device)
        if world > 1:
            dist.broadcast(xb, src=0, group=self.group)
        lo, hi = self.plan.rows(self.rank)
        R = self.plan.max_rows
        y_pad = torch.zeros((R, b), dtype=torch.float32, device=self.device)
        if hi > lo:
            self.compute(xb, y_pad[: hi - lo])
        if world == 1:
            return y_pad[: self.plan.m].clone()
        gathered = torch.empty((world * R, b), dtype=torch.float32, device=self.device)
        dist.all_gather_into_tensor(gathered, y_pad, group=self.group)
        parts = [gathered[r * R: r * R + (self.plan.bounds[r + 1] - self.plan.bounds[r])] for r in range(world)]
        return torch.cat(parts, dim=0)


def device_compute(layer, pdl: bool = False):
    """The production per-rank compute: the fused CUDA kernel on this rank's
    PackedLinear shard (paper_2005_09904_b200.biqgemm.PackedLinear)."""

    def run(x_dev: torch.Tensor, y_local: torch.Tensor):
        layer.forward_device(x_dev, y_local, pdl=pdl)

    return run
