# SPDX-License-Identifier: Apache-2.0
"""Ulysses sequence parallelism on CPU: world_size 2 over gloo.

The exchange protocol (pack -> all-to-all -> chunked head layout -> all-to-all ->
unpack) is exercised with a torch block-transpose standing in for the CUDA pack
kernel (test double; the product default is vsa_transpose_blocks). End to end,
each rank runs the ORACLE VSA forward+backward (test infrastructure) on its
H/P heads of the full sequence, read from the all-to-all receive layout, and the
resharded results must equal the oracle on the unsharded problem bit for bit
(every (b, h) unit is computed by exactly one rank).
"""
import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def torch_transpose_blocks(src, dst, n0, n1, block_elems):
    dst.view(n1, n0, block_elems).copy_(src.reshape(n0, n1, block_elems).transpose(0, 1))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


GRID, B, H, D, TOPK = (4, 8, 8), 2, 4, 16, 2


def _problem():
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as orc

    rng = orc.Rng(5)
    S = GRID[0] * GRID[1] * GRID[2]
    xs = [orc.randn(rng, B, H, S, D, np.float32) for _ in range(6)]  # q k v gc gf dO, [B,H,S,d]
    return orc, xs


def _oracle_vsa(orc, q, k, v, gc, gf, do):
    """Full VSA fwd+bwd on raster [B,H,S,d] fp32 arrays (grid divisible: no padding)."""
    L = orc.TileLayout(*GRID, 4, 4, 4)
    t = lambda x: orc.tile(L, np.ascontiguousarray(x))
    qt, kt, vt, gct, gft, dot = (t(x) for x in (q, k, v, gc, gf, do))
    art = orc.coarse_forward_select(L, qt, kt, vt, TOPK)
    fo, _, lse = orc.fine_forward(L, qt, kt, vt, art.sel)
    out = art.oc * gct + fo * gft
    cdq, cdk, cdv = orc.coarse_backward(art, L, dot * gct, qt, kt, vt)
    fdq, fdk, fdv = orc.fine_backward(L, qt, kt, vt, art.sel, dot * gft, lse)
    u = lambda x: orc.untile(L, x)
    return [u(out), u(cdq + fdq), u(cdk + fdk), u(cdv + fdv), u(dot * art.oc), u(dot * fo)]


def _worker(rank, world, port, q):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        sys.path.insert(0, ROOT)
        from paper_2505_13389_b200.ulysses import UlyssesExchange

        orc, xs = _problem()
        S = xs[0].shape[2]
        Sc, Hl = S // world, H // world
        ex = UlyssesExchange(B, S, H, D, transpose_blocks=torch_transpose_blocks)
        assert ex.P == world and ex.Sc == Sc and ex.Hl == Hl
        # my sequence shard of every tensor, [B, S/P, H, d]
        shard = [torch.from_numpy(np.ascontiguousarray(x.transpose(0, 2, 1, 3)[:, rank * Sc:(rank + 1) * Sc]))
                 for x in xs]
        heads = [ex.to_heads(t) for t in shard]  # [P, B, S/P, H/P, d]
        # layout check: chunk j = rank j's shard, heads of this rank
        for x, hx in zip(xs, heads):
            want = x[:, rank * Hl:(rank + 1) * Hl].transpose(0, 2, 1, 3).reshape(B, world, Sc, Hl, D)
            assert np.array_equal(hx.numpy(), want.transpose(1, 0, 2, 3, 4)), "to_heads layout"
        # inverse exchange restores the shard
        back = ex.to_seq(heads[0])
        assert torch.equal(back, shard[0]), "to_seq(to_heads(x)) != x"
        # oracle VSA on the local heads, reading the chunked receive layout
        as_bhsd = lambda hx: np.ascontiguousarray(hx.numpy().transpose(1, 3, 0, 2, 4).reshape(B, Hl, S, D))
        res = _oracle_vsa(orc, *(as_bhsd(hx) for hx in heads))
        to_chunked = lambda r: torch.from_numpy(np.ascontiguousarray(
            r.reshape(B, Hl, world, Sc, D).transpose(2, 0, 3, 1, 4)))
        got = [ex.to_seq(to_chunked(r)) for r in res]
        full = _oracle_vsa(orc, *xs)
        for g, f in zip(got, full):
            want = f.transpose(0, 2, 1, 3)[:, rank * Sc:(rank + 1) * Sc]
            assert np.array_equal(g.numpy(), want), "Ulysses result differs from the unsharded oracle"
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover - reported to the parent
        import traceback

        q.put((rank, traceback.format_exc() + repr(e)))


@pytest.mark.parametrize("world", [2])
def test_ulysses_exchange_gloo(world, orc):
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


def test_exchange_rejects_indivisible():
    sys.path.insert(0, ROOT)
    from paper_2505_13389_b200.ulysses import UlyssesExchange

    ex = UlyssesExchange(1, 12, 4, 8, transpose_blocks=torch_transpose_blocks)  # not initialised: P = 1
    assert ex.P == 1
    x = torch.randn(1, 12, 4, 8)
    assert ex.to_heads(x).data_ptr() == x.data_ptr()  # one chunk: the shard IS the head layout
    with pytest.raises(ValueError):
        ex.to_heads(torch.randn(1, 11, 4, 8))
