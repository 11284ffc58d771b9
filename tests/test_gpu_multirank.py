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
