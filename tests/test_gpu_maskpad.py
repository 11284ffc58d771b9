# SPDX-License-Identifier: Apache-2.0
"""Mask-pad mode (FastVideo-style padding): padded keys are
excluded from attention, cube means / maxima run over the real tokens, the mean unpool
divides by the real count. There is no reference semantics to pin it to (the reference
rejects non-divisible grids), so it is checked, as the survey prescribes, against the
oracle's masked dense attention (dense_forward / dense_backward with a DenseMask,
dense.hpp:94-209) on the zero-padded tile-ordered problem:

* pooled cubes: bit-exact with the sequential fp32 sum over real tokens / real count;
* the fine stage (fed the operator's own block map): out and dq / dk / dv equal masked
  dense attention with mask = selected blocks AND real keys (Gc = 0, Gf = 1 isolates it);
* the tcgen05 (bf16) and SIMT (fp32) kernels, with and without the dS workspace."""
import numpy as np
import pytest
import torch

import oracle as orc
from gpu_helpers import Problem, assert_close, host, rounded, to_dev

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def vsa():
    import paper_2505_13389_b200 as v

    v.lib()
    return v


def real_tokens(p):
    """bool [Lp]: tile position -> real (non-padded) token."""
    real = np.ones((1, 1, p.S, 1), np.float32)
    return p.pad_tile(real)[0, 0, :, 0] > 0.5


def pooled_mean_real(xt, real, cube=64):
    """Sequential fp32 sum over the real tokens of each cube (tile order) / real count."""
    B, H, Lp, d = xt.shape
    nc = Lp // cube
    out = np.zeros((B, H, nc, d), np.float32)
    for c in range(nc):
        acc = np.zeros((B, H, d), np.float32)
        n = 0
        for o in range(cube):
            if real[c * cube + o]:
                acc = (acc + xt[:, :, c * cube + o]).astype(np.float32)
                n += 1
        out[:, :, c] = acc / np.float32(n)
    return out


CASES = [((9, 14, 14), 64, 5, torch.bfloat16), ((9, 14, 14), 128, 16, torch.bfloat16),
         ((9, 14, 14), 64, 5, torch.float32), ((5, 10, 11), 128, 8, torch.bfloat16)]


@pytest.mark.parametrize("grid,d,k,dtype", CASES, ids=["bf16-d64", "bf16-d128-k16", "f32-d64", "bf16-d128-ragged"])
@pytest.mark.parametrize("ws", [True, False], ids=["ds-ws", "recompute"])
def test_maskpad_vs_masked_dense(vsa, grid, d, k, dtype, ws):
    p = Problem(grid=grid, B=1, H=2, d=d, top_k=k, seed=91)
    L = vsa.TileLayout(*grid, pad="mask")
    assert L.mask_pad and L.seq_padded > L.seq_len
    op = vsa.VsaOp(L, p.B, p.H, d, k, dtype=dtype, adaptation=True, bwd_workspace=ws)
    gc = np.zeros_like(p.gc)  # Gc = 0, Gf = 1: out is the fine stage alone
    out = op.forward(*(to_dev(x, dtype) for x in (p.q, p.k, p.v)), to_dev(gc, dtype))
    grads = op.backward(to_dev(p.dout, dtype))
    torch.cuda.synchronize()
    real = real_tokens(p)
    q, kk, v, do = (p.pad_tile(rounded(x, dtype)) for x in (p.q, p.k, p.v, p.dout))
    # pooled cubes over real tokens, bit-exact
    for got, x in ((op.qc, q), (op.kc, kk), (op.vc, v)):
        np.testing.assert_array_equal(got.cpu().numpy(), pooled_mean_real(x, real))
    # fine stage == masked dense attention (selected blocks AND real keys)
    sel = op.sel.cpu().numpy()
    OL = p.olayout
    allowed = np.stack([orc.selection_to_mask(OL, sel, 0)[h] & real[None, :] for h in range(p.H)]).astype(np.uint8)
    dense_o, _, dense_lse = orc.dense_forward(q, kk, v, allowed)
    dq, dk, dv = orc.dense_backward(q, kk, v, allowed, do, dense_lse)
    assert_close(host(out), p.untile_crop(dense_o), dtype, "maskpad out")
    for g, r, n in zip(grads[:3], (dq, dk, dv), ("dq", "dk", "dv")):
        assert_close(host(g), p.untile_crop(r), dtype, f"maskpad {n}")


def test_maskpad_max_pool_and_unpool(vsa):
    """Max pooling over real tokens only, and the coarse backward's unpool (mean by real
    count / first argmax among real tokens) on tile-ordered tensors."""
    p = Problem(grid=(9, 14, 14), B=1, H=1, d=64, top_k=4, seed=92)
    L = vsa.TileLayout(*p.grid, pad="mask")
    real = real_tokens(p)
    q = p.pad_tile(p.q.astype(np.float32)) - 5.0  # all values negative: the zero pads would win a plain max
    q[:, :, ~real] = 0.0
    qt = to_dev(q, torch.float32)
    mx = vsa.pool_cubes(L, qt, vsa.POOL_MAX).cpu().numpy()
    ref = np.stack([q[:, :, c * 64:(c + 1) * 64][:, :, real[c * 64:(c + 1) * 64]].max(axis=2)
                    for c in range(L.num_cubes)], axis=2)
    np.testing.assert_array_equal(mx, ref)
    mean = vsa.pool_cubes(L, qt, vsa.POOL_MEAN).cpu().numpy()
    np.testing.assert_array_equal(mean, pooled_mean_real(q, real))
