# SPDX-License-Identifier: Apache-2.0
"""GPU: sequence-major raster I/O (DiT-native [B,S,H,d] and the Ulysses chunked
receive layout [P,B,S/P,H,d]) and the Ulysses pack kernel.

Every kernel that touches a raster tensor addresses it through raster_row(); the
results must be BITWISE identical to the head-major op on the same data (same
kernels, same arithmetic, only the addresses differ), for max and mean pooling,
the tcgen05 (bf16) and SIMT (fp32) paths."""
import pytest
import torch

from gpu_helpers import Problem, to_dev

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def vsa():
    import paper_2505_13389_b200 as v

    v.lib()
    return v


def to_chunked(x, P):
    """[B,H,S,d] -> [P,B,S/P,H,d] (P = 1 gives [1,B,S,H,d] == [B,S,H,d])."""
    B, H, S, d = x.shape
    return x.reshape(B, H, P, S // P, d).permute(2, 0, 3, 1, 4).contiguous()


def from_chunked(y, B, H, S, d):
    P = y.shape[0]
    return y.reshape(P, B, S // P, H, d).permute(1, 3, 0, 2, 4).reshape(B, H, S, d)


CASES = [
    (dict(grid=(9, 14, 22), B=2, H=3, d=128, top_k=6), torch.bfloat16, 1, 0),
    (dict(grid=(9, 14, 22), B=2, H=3, d=128, top_k=6), torch.bfloat16, 3, 0),
    (dict(grid=(8, 12, 12), B=1, H=4, d=64, top_k=5), torch.bfloat16, 4, 1),
    (dict(grid=(8, 12, 12), B=2, H=2, d=64, top_k=5), torch.float32, 2, 0),
]


@pytest.mark.parametrize("cfg,dtype,P,pool", CASES, ids=["bshd", "chunk3", "chunk4-max", "f32-chunk2"])
def test_seq_major_io_bitwise(vsa, cfg, dtype, P, pool):
    p = Problem(**cfg, seed=101)
    L = vsa.TileLayout(*p.grid, pad=True)
    S = L.seq_len
    ins = [to_dev(x, dtype) for x in (p.q, p.k, p.v, p.gc, p.gf, p.dout)]
    ref_op = vsa.VsaOp(L, p.B, p.H, p.d, p.top_k, dtype=dtype, pool=pool)
    ref = [ref_op.forward(*ins[:5]).clone()] + [t.clone() for t in ref_op.backward(ins[5])]
    op = vsa.VsaOp(L, p.B, p.H, p.d, p.top_k, dtype=dtype, pool=pool, io="bshd", seq_chunks=P)
    xin = [to_chunked(t, P) for t in ins]
    if P == 1:
        xin = [t.view(p.B, S, p.H, p.d) for t in xin]
    got = [op.forward(*xin[:5]).clone()] + [t.clone() for t in op.backward(xin[5])]
    assert torch.equal(op.sel, ref_op.sel)
    names = ["out", "dq", "dk", "dv", "dgc", "dgf"]
    for g, r, n in zip(got, ref, names):
        g = g.view(P, p.B, S // P, p.H, p.d)
        assert torch.equal(from_chunked(g, p.B, p.H, S, p.d), r), n


def test_seq_major_rejects_bad_shapes(vsa):
    L = vsa.TileLayout(8, 8, 8)
    with pytest.raises(ValueError):
        vsa.VsaOp(L, 1, 2, 64, 2, io="bshd", seq_chunks=3)  # 512 % 3 != 0
    with pytest.raises(ValueError):
        vsa.VsaOp(L, 1, 2, 64, 2, io="bshd", raster=False)
    op = vsa.VsaOp(L, 1, 2, 64, 2, io="bshd")
    x = torch.zeros(1, 2, 512, 64, dtype=torch.bfloat16, device="cuda")  # head-major shape
    with pytest.raises(ValueError):
        op.forward(x, x, x, x, x)


@pytest.mark.parametrize("n0,n1,blk", [(7, 3, 128), (1, 8, 640), (300, 8, 640), (5, 1, 16)])
def test_transpose_blocks_kernel(vsa, n0, n1, blk):
    from paper_2505_13389_b200.ulysses import transpose_blocks_cuda

    src = torch.randn(n0, n1, blk, device="cuda").to(torch.bfloat16)
    dst = torch.empty(n1, n0, blk, device="cuda", dtype=torch.bfloat16)
    transpose_blocks_cuda(src, dst, n0, n1, blk)
    assert torch.equal(dst, src.transpose(0, 1))


def test_ulysses_single_rank_matches_op(vsa):
    """P = 1 (no process group): UlyssesVsa on [B,S,H,d] == VsaOp head-major, bitwise."""
    p = Problem(grid=(8, 12, 12), B=1, H=4, d=128, top_k=5, seed=111)
    L = vsa.TileLayout(*p.grid, pad=True)
    dt = torch.bfloat16
    ins = [to_dev(x, dt) for x in (p.q, p.k, p.v, p.gc, p.gf, p.dout)]
    ref_op = vsa.VsaOp(L, p.B, p.H, p.d, p.top_k, dtype=dt)
    ref = [ref_op.forward(*ins[:5]).clone()] + [t.clone() for t in ref_op.backward(ins[5])]
    u = vsa.UlyssesVsa(L, p.B, p.H, p.d, p.top_k, dtype=dt)
    sh = [t.permute(0, 2, 1, 3).contiguous() for t in ins]
    got = [u.forward(*sh[:5])] + list(u.backward(sh[5]))
    for g, r in zip(got, ref):
        assert torch.equal(g.permute(0, 2, 1, 3), r)
