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
