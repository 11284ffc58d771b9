# SPDX-License-Identifier: Apache-2.0
"""Ulysses sequence parallelism for the VSA operator.

The reference is single-process (its only parallelism is OpenMP over (b, h)
work items, parallel.hpp:15-23); the build's sequence-parallel config shards the
raster sequence across P ranks. Attention needs whole sequences, so the one real
exchange step is a sequence -> head all-to-all before the op and head -> sequence
after it (and the mirror in backward):

    rank r holds   x_r  [B, S/P, H, d]            (its sequence shard, all heads)
    pack           send [P, B, S/P, H/P, d]       (block transpose, our kernel)
    all-to-all     recv [P, B, S/P, H/P, d]       = the full sequence of heads
                                                    r*H/P .. (r+1)*H/P, chunk j
                                                    being rank j's shard
    VSA            VsaOp(io="bshd", seq_chunks=P) reads/writes this chunked
                   layout IN PLACE (no unpack): its output is already the send
                   buffer of the return all-to-all
    all-to-all     [P, B, S/P, H/P, d]            head group j of my shard
    unpack         y_r  [B, S/P, H, d]            (block transpose)

Every (b, h) unit is computed by exactly one rank with the same kernels as the
single-GPU op, so results are bitwise identical to it. Collectives go through
torch.distributed (NCCL over NVLink on the GPU box, gloo in the CPU tests); the
gate exchange is issued asynchronously and overlaps K1-K3 (tile/pool/coarse),
which do not read the gates.
"""
from __future__ import annotations

import ctypes as C
from typing import Callable, Optional, Sequence

import torch
import torch.distributed as dist

from . import _lib as L


def transpose_blocks_cuda(src: torch.Tensor, dst: torch.Tensor, n0: int, n1: int, block_elems: int) -> None:
    """dst[i1][i0] = src[i0][i1] over [n0][n1] blocks (vsa_transpose_blocks)."""
    if not (src.is_cuda and dst.is_cuda):
        raise ValueError("transpose_blocks: CUDA tensors required")
    rc = L.lib().vsa_transpose_blocks(C.c_void_p(src.data_ptr()), C.c_void_p(dst.data_ptr()), n0, n1,
                                      block_elems * src.element_size(),
                                      C.c_void_p(torch.cuda.current_stream().cuda_stream))
    if rc != 0:
        raise (ValueError if rc < 0 else L.VsaError)(L.lib().vsa_last_error().decode())


class UlyssesExchange:
    """The two all-to-all reshardings of one sequence-parallel group.

    ``to_heads(x)``: [B, S/P, H, d] shard -> [P, B, S/P, H/P, d] (full sequence, local heads).
    ``to_seq(y)``  : [P, B, S/P, H/P, d] -> [B, S/P, H, d].
    ``transpose_blocks`` is the pack/unpack kernel (the CUDA C-ABI by default).
    """

    def __init__(self, B: int, S: int, H: int, d: int, group=None,
                 transpose_blocks: Callable = transpose_blocks_cuda, host_staged: bool = False):
        self.group = group
        self.P = dist.get_world_size(group) if dist.is_available() and dist.is_initialized() else 1
        if H % self.P or S % self.P:
            raise ValueError(f"Ulysses: heads ({H}) and sequence ({S}) must divide by the group size {self.P}")
        self.B, self.S, self.H, self.d = B, S, H, d
        self.Sc, self.Hl = S // self.P, H // self.P
        self.tb = transpose_blocks
        # host_staged: the all-to-all runs on host copies (for a CPU-only process group, e.g.
        # gloo with several ranks sharing one GPU in tests); the default exchanges the
        # device buffers directly (NCCL over NVLink)
        self.host_staged = host_staged

    def _all_to_all(self, recv, send, async_op=False):
        if not self.host_staged:
            return dist.all_to_all_single(recv, send, group=self.group, async_op=async_op)
        r = torch.empty(recv.shape, dtype=recv.dtype)
        dist.all_to_all_single(r, send.cpu(), group=self.group)
        recv.copy_(r)
        return None

    @property
    def shard_shape(self):
        return (self.B, self.Sc, self.H, self.d)

    @property
    def head_shape(self):
        return (self.P, self.B, self.Sc, self.Hl, self.d)

    @staticmethod
    def _norm(shape):  # [1, B, S, H, d] (one chunk) == [B, S, H, d]
        shape = tuple(shape)
        return shape[1:] if len(shape) == 5 and shape[0] == 1 else shape

    def _check(self, t: torch.Tensor, shape, name: str) -> None:
        if self._norm(t.shape) != self._norm(shape) or not t.is_contiguous():
            raise ValueError(f"{name}: expected a contiguous {tuple(shape)} tensor, got {tuple(t.shape)}")

    def to_heads(self, x: torch.Tensor, async_op: bool = False):
        self._check(x, self.shard_shape, "Ulysses.to_heads")
        if self.P == 1:  # [B, S, H, d] is the chunked layout with one chunk
            recv = x.view(self.head_shape)
            return (recv, None) if async_op else recv
        recv = torch.empty(self.head_shape, dtype=x.dtype, device=x.device)
        send = torch.empty_like(recv)
        self.tb(x, send, self.B * self.Sc, self.P, self.Hl * self.d)
        work = self._all_to_all(recv, send, async_op=async_op)
        return (recv, work) if async_op else recv

    def to_seq(self, y: torch.Tensor) -> torch.Tensor:
        self._check(y, self.head_shape, "Ulysses.to_seq")
        if self.P == 1:
            return y.view(self.shard_shape)
        out = torch.empty(self.shard_shape, dtype=y.dtype, device=y.device)
        recv = torch.empty_like(y)
        self._all_to_all(recv, y)
        self.tb(recv, out, self.P, self.B * self.Sc, self.Hl * self.d)
        return out


class UlyssesVsa:
    """Sequence-parallel VSA forward/backward on sequence shards [B, S/P, H, d].

    Each rank runs VsaOp on H/P heads over the whole sequence, reading the
    all-to-all receive buffers in place (io="bshd", seq_chunks=P)."""

    def __init__(self, layout, B: int, H: int, d: int, top_k: int, group=None, dtype=torch.bfloat16,
                 host_staged: bool = False, **op_kwargs):
        from .api import VsaOp

        self.x = UlyssesExchange(B, layout.seq_len, H, d, group, host_staged=host_staged)
        self.op = VsaOp(layout, B, self.x.Hl, d, top_k, dtype=dtype, io="bshd", seq_chunks=self.x.P, **op_kwargs)

    def forward(self, q, k, v, gc, gf=None) -> torch.Tensor:
        x = self.x
        qh, kh, vh = (x.to_heads(t) for t in (q, k, v))
        pending = []
        gch, w = x.to_heads(gc, async_op=True)
        pending.append(w)
        gfh = None
        if gf is not None:
            gfh, w = x.to_heads(gf, async_op=True)
            pending.append(w)

        def gates_ready():
            for w in pending:
                if w is not None:
                    w.wait()

        out = self.op.forward(qh, kh, vh, gch, gfh, before_fine=gates_ready)
        return x.to_seq(out)

    def backward(self, dout) -> Sequence[torch.Tensor]:
        grads = self.op.backward(self.x.to_heads(dout))
        return tuple(self.x.to_seq(g) for g in grads)
