# SPDX-License-Identifier: Apache-2.0
"""Multi-rank paths of the operator on the GPU, on one B200.

* Batch x head partition: every rank's PartitionedVsa (the product partitioner) on
  its unit shard, run one after another on the device; the concatenated results
  must be bitwise equal to one VsaOp on the whole problem.
* Ulysses sequence parallelism with 2 real ranks (two processes sharing cuda:0,
  gloo with host-staged all-to-alls, since NCCL needs one GPU per rank): the pack
  kernel, the chunked in-place layout of VsaOp and the unpack kernel, forward and
  backward, against a single-process VsaOp on the unsharded sequence — bitwise."""
import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def vsa():
    import paper_2505_13389_b200 as v

    v.lib()
    return v


@pytest.mark.parametrize("world", [2, 4, 8])
def test_bh_partition_bitwise(vsa, world):
    from paper_2505_13389_b200.partition import PartitionedVsa, shard_units

    L = vsa.TileLayout(8, 12, 12, pad=True)
    B, H, d, k = 2, 3, 64, 5
    g = torch.Generator(device="cuda").manual_seed(11)
    xs = [torch.randn((B, H, L.seq_len, d), generator=g, device="cuda").bfloat16() for _ in range(6)]
    full = vsa.VsaOp(L, B, H, d, k)
    ref = [full.forward(*xs[:5]).clone()] + [t.clone() for t in full.backward(xs[5])]
    flat = lambda t: t.reshape(B * H, L.seq_len, d)
    got = [[] for _ in ref]
    for rank in range(world):
        part = PartitionedVsa(L, B, H, d, k, rank, world)
        if part.op is None:
            continue
        sh = [shard_units(x, part.u0, part.u1).contiguous() for x in xs]
        outs = [part.forward(*sh[:5])] + list(part.backward(sh[5]))
        for i, o in enumerate(outs):
            got[i].append(o.reshape(part.n, L.seq_len, d))
    for i, r in enumerate(ref):
        assert torch.equal(torch.cat(got[i]), flat(r)), f"output {i}: partitioned != whole problem"


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


GRID, B_, H_, D_, K_ = (8, 16, 16), 1, 4, 128, 4


def _inputs(S):
    g = torch.Generator(device="cuda").manual_seed(21)
    return [torch.randn((B_, S, H_, D_), generator=g, device="cuda").bfloat16() for _ in range(6)]  # [B,S,H,d]


def _ulysses_worker(rank, world, port, q):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        sys.path.insert(0, ROOT)
        torch.cuda.set_device(0)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import paper_2505_13389_b200 as vsa

        L = vsa.TileLayout(*GRID, pad=True)
        S = L.seq_len
        xs = _inputs(S)
        Sc = S // world
        shard = [x[:, rank * Sc:(rank + 1) * Sc].contiguous() for x in xs]
        u = vsa.UlyssesVsa(L, B_, H_, D_, K_, host_staged=True)
        assert u.x.P == world
        out = u.forward(*shard[:5])
        grads = u.backward(shard[5])
        res = [out] + list(grads)
        # the unsharded reference: one VsaOp over all heads, sequence-major I/O
        full = vsa.VsaOp(L, B_, H_, D_, K_, io="bshd")
        fo = full.forward(*xs[:5])
        fg = full.backward(xs[5])
        for i, (a, b) in enumerate(zip(res, [fo] + list(fg))):
            want = b[:, rank * Sc:(rank + 1) * Sc]
            assert torch.equal(a, want), f"rank {rank} output {i}: Ulysses != single op"
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover - reported to the parent
        import traceback

        q.put((rank, traceback.format_exc() + repr(e)))


def test_ulysses_two_ranks_bitwise():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_ulysses_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=300) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    for r in range(2):
        assert res[r] == "ok", res[r]


class _SimExchange:
    """In-process stand-in for the all-reduce of SubSplitVsa (threads share one GPU):
    every rank adds its [units*Lp] buffer into one accumulator, waits for all, reads it back."""

    def __init__(self, world):
        import threading

        self.world, self.acc, self.lock = world, None, threading.Lock()
        self.b1, self.b2 = threading.Barrier(world, timeout=300), threading.Barrier(world, timeout=300)

    def __call__(self, buf):
        torch.cuda.synchronize()
        with self.lock:
            self.acc = buf.clone() if self.acc is None else self.acc + buf
        self.b1.wait()
        torch.cuda.synchronize()
        buf.copy_(self.acc)
        torch.cuda.synchronize()
        if self.b2.wait() == 0:  # one thread resets the accumulator once everyone has read it
            self.acc = None


@pytest.mark.parametrize("world", [2, 5, 8])
def test_cube_subsplit_bitwise(vsa, world):
    """SubSplitVsa (heads shared between ranks, lse / delta exchanged): every rank's rows of
    out (its query cubes), dq (its query cubes), dk / dv (its key cubes) are bitwise equal to
    one operator on the whole problem (the recompute-dQ backward, which the sub-split uses)."""
    import threading

    from paper_2505_13389_b200.partition import SubSplitVsa

    L = vsa.TileLayout(8, 16, 16)  # nc = 32, tile order: a task's rows are contiguous
    B, H, d, k = 1, 3, 128, 6
    g = torch.Generator(device="cuda").manual_seed(12)
    xs = [torch.randn((B, H, L.seq_padded, d), generator=g, device="cuda").bfloat16() for _ in range(6)]
    full = vsa.VsaOp(L, B, H, d, k, raster=False, bwd_workspace=False)
    ref = [full.forward(*xs[:5]).clone()] + [t.clone() for t in full.backward(xs[5])]
    torch.cuda.synchronize()
    ex = _SimExchange(world)
    parts = [SubSplitVsa(L, B, H, d, k, r, world, exchange=ex, raster=False) for r in range(world)]
    res = [None] * world

    def run(r):
        p = parts[r]
        sh = [p.shard(x).contiguous() for x in xs]
        out = p.forward(*sh[:5])
        grads = p.backward(sh[5])
        torch.cuda.synchronize()
        res[r] = [out] + list(grads)

    th = [threading.Thread(target=run, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    Lp, nc = L.seq_padded, L.num_cubes
    flat_ref = [x.reshape(-1, d) for x in ref]
    covered = 0
    for p, r in zip(parts, res):
        lo, hi = p.t0 * 64, p.t1 * 64  # global tiled rows of this rank's tasks
        off = p.ua * Lp
        for i in (0, 1, 2, 3):  # out, dq (query cubes) and dk, dv (key cubes) of the range
            got = r[i].reshape(-1, d)[lo - off:hi - off]
            assert torch.equal(got, flat_ref[i][lo:hi]), f"rank tasks [{p.t0},{p.t1}) output {i}"
        covered += hi - lo
        assert p.n <= 2
    assert covered == B * H * Lp
    # the shared heads really are split: some rank starts mid-head
    assert any(p.t0 % nc for p in parts)
