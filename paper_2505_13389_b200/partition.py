# SPDX-License-Identifier: Apache-2.0
"""Batch x head partition of one VSA problem across GPUs.

Every stage of the operator is independent per (b, h) unit: the coarse stage per
(b, h) (coarse.hpp:95,143), the fine stage per (b, h, q-cube) and (b, h, k-cube)
(fine.hpp:65,129,172). One problem's B*H units are therefore split into contiguous
ranges, one per rank, with no data-path collective: rank r runs the operator on
units [u0, u1) of the head-major [B*H, S, d] tensors (a contiguous slice) and owns
those rows of every output. Each unit is computed by exactly one rank with the same
kernels in the same order as on one GPU, so the union of the ranks' results is
bitwise identical to the single-GPU result (tests/test_partition_gloo.py,
tests/test_gpu_partition.py).

Balance: sizes differ by at most one unit. Wan2.1-1.3B (12 heads) on 8 GPUs gives
2 units on 4 ranks and 1 on 4 (a 1.5 / 2 = 75% ceiling on the step time); the DiT
batch (128 units) and the sweep (16 heads) split evenly.

Sub-split (SubSplitVsa, SURVEY.md §8e "sub-split by q-cube ranges (forward, dQ) and k-cube
ranges (dK/dV)"): the B*H*nc (unit, cube) tasks are split into contiguous ranges, so a
head can be shared by two ranks (Wan2.1-1.3B on 8 GPUs: 1.5 heads each). A rank replicates
the K1 / coarse stages of the units it touches and runs the fine forward for its query
cubes, the dQ pass for the same query cubes and the dK/dV pass for the key cubes of the
same range. The one exchange is of the per-row softmax statistics of the shared units:
lse after the forward and delta after the backward prologue (an all-reduce of each rank's
own rows, a few MB), since a key cube's dK/dV reads every query row that selected it.
"""
from __future__ import annotations

from typing import List, Tuple

import torch


def partition_units(units: int, world: int) -> List[Tuple[int, int]]:
    """Contiguous unit ranges [u0, u1) for ranks 0..world-1 (sizes differ by <= 1)."""
    if units < 1 or world < 1:
        raise ValueError("partition: units and world must be >= 1")
    return [(units * r // world, units * (r + 1) // world) for r in range(world)]


def shard_units(x: torch.Tensor, u0: int, u1: int) -> torch.Tensor:
    """Head-major [B, H, S, d] -> this rank's units as a [1, u1-u0, S, d] view (contiguous)."""
    B, H, S, d = x.shape
    return x.reshape(1, B * H, S, d)[:, u0:u1]


class PartitionedVsa:
    """The rank's share of one VSA problem: a VsaOp over its contiguous unit range.

    forward / backward take the rank's shard ([1, n, S, d], e.g. ``shard_units`` of the
    full tensors, or tensors built for those units only) and return that shard of the
    outputs. Ranks with no unit (world > B*H) hold no operator and return None."""

    def __init__(self, layout, B: int, H: int, d: int, top_k: int, rank: int, world: int, **op_kwargs):
        from .api import VsaOp

        self.units = B * H
        self.u0, self.u1 = partition_units(self.units, world)[rank]
        self.n = self.u1 - self.u0
        self.op = VsaOp(layout, 1, self.n, d, top_k, **op_kwargs) if self.n else None

    def forward(self, q, k, v, gc, gf=None, **kw):
        return None if self.op is None else self.op.forward(q, k, v, gc, gf, **kw)

    def backward(self, dout, *outs, **kw):
        return None if self.op is None else self.op.backward(dout, *outs, **kw)


def partition_tasks(units: int, nc: int, world: int) -> List[Tuple[int, int]]:
    """Contiguous (unit, cube) task ranges [t0, t1) over units*nc tasks (sizes differ by <= 1)."""
    return partition_units(units * nc, world)


def _all_reduce_sum(t: torch.Tensor) -> None:
    import torch.distributed as dist

    dist.all_reduce(t)


class SubSplitVsa:
    """A rank's share of one problem split by (unit, cube) task ranges.

    The rank's operator covers the units [ua, ub) its task range touches (inputs: those
    units' full [1, ub-ua, S, d] tensors) with task_range = its tasks relative to ua*nc.
    forward/backward exchange the lse / delta rows of the shared units through
    ``exchange`` (an in-place sum over ranks of a [B*H*Lp] fp32 buffer holding each rank's
    own rows; all_reduce over torch.distributed by default). Each rank owns the output rows
    of its task range: out / dq rows of its query cubes, dk / dv rows of its key cubes."""

    def __init__(self, layout, B: int, H: int, d: int, top_k: int, rank: int, world: int, exchange=None, **op_kwargs):
        from .api import VsaOp

        self.layout, self.units, self.nc, self.cube = layout, B * H, layout.num_cubes, layout.cube_size
        self.t0, self.t1 = partition_tasks(self.units, self.nc, world)[rank]
        self.ua = self.t0 // self.nc
        self.ub = -(-self.t1 // self.nc) if self.t1 > self.t0 else self.ua
        self.n = self.ub - self.ua
        self.exchange = exchange or _all_reduce_sum
        rel = (self.t0 - self.ua * self.nc, self.t1 - self.ua * self.nc)
        self.op = (VsaOp(layout, 1, self.n, d, top_k, task_range=rel, bwd_workspace=False, **op_kwargs)
                   if self.t1 > self.t0 else None)

    def shard(self, x: torch.Tensor) -> torch.Tensor:
        """Full head-major [B, H, S, d] -> this rank's units [1, ub-ua, S, d] (a view)."""
        return shard_units(x, self.ua, self.ub)

    # rows of this rank's tasks in the op's tiled [n * Lp] per-row statistics
    def _own(self):
        return (self.t0 - self.ua * self.nc) * self.cube, (self.t1 - self.ua * self.nc) * self.cube

    def _complete(self, stat: torch.Tensor, device) -> None:
        Lp = self.layout.seq_padded
        buf = torch.zeros(self.units * Lp, dtype=torch.float32, device=device)
        if self.op is not None:
            lo, hi = self._own()
            flat = stat.reshape(-1)
            buf[self.ua * Lp + lo:self.ua * Lp + hi] = flat[lo:hi]
        self.exchange(buf)
        if self.op is not None:
            stat.reshape(-1).copy_(buf[self.ua * Lp:self.ub * Lp])

    def forward(self, q, k, v, gc, gf=None, **kw):
        out = self.op.forward(q, k, v, gc, gf, **kw) if self.op is not None else None
        self._complete(self.op.lse if self.op is not None else None, q.device if q is not None else "cuda")
        return out

    def backward(self, dout, *outs, **kw):
        if self.op is None:
            self._complete(None, "cuda")
            return None
        return self.op.backward(dout, *outs, before_finish=lambda: self._complete(self.op.delta, dout.device), **kw)
