# SPDX-License-Identifier: Apache-2.0
"""Batch x head partition on CPU: world_size 2 and 4 over gloo.

Each rank takes its contiguous unit range from the product partitioner
(paper_2505_13389_b200.partition.partition_units / shard_units), runs the ORACLE
VSA forward + backward (test infrastructure) on that shard only, and the gathered
results must equal the oracle on the unsharded problem bit for bit: every (b, h)
unit is computed by exactly one rank, no data-path collective. World 4 over 6
units gives ranks of 1 and 2 units (the uneven Wan2.1-1.3B-on-8-GPUs case)."""
import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GRID, B, H, D, TOPK = (4, 8, 8), 2, 3, 16, 2


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _problem():
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as orc

    rng = orc.Rng(9)
    S = GRID[0] * GRID[1] * GRID[2]
    return orc, [orc.randn(rng, B, H, S, D, np.float32) for _ in range(6)]  # q k v gc gf dO


def _oracle_vsa(orc, q, k, v, gc, gf, do):
    L = orc.TileLayout(*GRID, 4, 4, 4)
    t = lambda x: orc.tile(L, np.ascontiguousarray(x))
    qt, kt, vt, gct, gft, dot = (t(x) for x in (q, k, v, gc, gf, do))
    art = orc.coarse_forward_select(L, qt, kt, vt, TOPK)
    fo, _, lse = orc.fine_forward(L, qt, kt, vt, art.sel)
    cdq, cdk, cdv = orc.coarse_backward(art, L, dot * gct, qt, kt, vt)
    fdq, fdk, fdv = orc.fine_backward(L, qt, kt, vt, art.sel, dot * gft, lse)
    u = lambda x: orc.untile(L, x)
    return [u(art.oc * gct + fo * gft), u(cdq + fdq), u(cdk + fdk), u(cdv + fdv), u(dot * art.oc), u(dot * fo)]


def _worker(rank, world, port, q):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        sys.path.insert(0, ROOT)
        from paper_2505_13389_b200.partition import partition_units, shard_units

        orc, xs = _problem()
        parts = partition_units(B * H, world)
        u0, u1 = parts[rank]
        assert parts[0][0] == 0 and parts[-1][1] == B * H
        assert all(a[1] == b[0] for a, b in zip(parts[:-1], parts[1:]))
        assert max(b - a for a, b in parts) - min(b - a for a, b in parts) <= 1
        mine = [shard_units(torch.from_numpy(x), u0, u1).numpy() for x in xs]  # [1, n, S, d]
        res = _oracle_vsa(orc, *mine) if u1 > u0 else []
        gathered = [None] * world
        dist.all_gather_object(gathered, (u0, u1, [r.tobytes() for r in res]))
        if rank == 0:
            full = _oracle_vsa(orc, *xs)
            S = xs[0].shape[2]
            for i, f in enumerate(full):
                flat = f.reshape(B * H, S, D)
                got = np.concatenate([np.frombuffer(g[2][i], np.float32).reshape(g[1] - g[0], S, D)
                                      for g in gathered if g[1] > g[0]])
                assert np.array_equal(got, flat), f"output {i}: partitioned != unsharded"
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover - reported to the parent
        import traceback

        q.put((rank, traceback.format_exc() + repr(e)))


@pytest.mark.parametrize("world", [2, 4])
def test_bh_partition_gloo(world, orc):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=240) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    for r in range(world):
        assert res[r] == "ok", res[r]


def test_partition_units_contract():
    sys.path.insert(0, ROOT)
    from paper_2505_13389_b200.partition import partition_units

    assert partition_units(12, 8) == [(0, 1), (1, 3), (3, 4), (4, 6), (6, 7), (7, 9), (9, 10), (10, 12)]
    assert partition_units(128, 8)[3] == (48, 64)
    assert partition_units(2, 4) == [(0, 0), (0, 1), (1, 1), (1, 2)]
    with pytest.raises(ValueError):
        partition_units(0, 2)
