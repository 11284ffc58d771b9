# SPDX-License-Identifier: Apache-2.0
"""The complete reference entry points vsa_forward / vsa_backward (vsa.hpp:89-189),
hidden states and gate parameters included, composed from the GPU pieces (tcgen05
gate GEMM -> VsaOp on tile-ordered tensors -> gate-projection backward) against the
oracle's vsa_forward / vsa_backward on the same bf16-rounded inputs."""
import numpy as np
import pytest
import torch

import oracle as orc
from gpu_helpers import assert_close, host, rounded

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def vsa():
    import paper_2505_13389_b200 as v

    v.lib()
    return v


@pytest.mark.parametrize("act", [0, 1], ids=["identity", "sigmoid"])
def test_vsa_forward_backward_with_hidden(vsa, act):
    grid, B, H, d, md, k = (8, 12, 12), 1, 2, 128, 256, 4
    L = vsa.TileLayout(*grid)
    OL = orc.TileLayout(*grid, 4, 4, 4)
    rng = orc.Rng(81)
    S = L.seq_len
    bf = lambda a: rounded(a, torch.bfloat16)
    hidden = bf(orc.randn(rng, B, 1, S, md, np.float32))
    q, kk, v = (bf(orc.randn(rng, B, H, S, d, np.float32)) for _ in range(3))
    w = bf(orc.randn_matrix(rng, md, 2 * H * d, np.float32, 1.0 / np.sqrt(md)))
    bias = orc.randn_matrix(rng, 1, 2 * H * d, np.float32, 0.1).reshape(-1)
    dout = bf(orc.randn(rng, B, H, S, d, np.float32))
    # oracle (tile-ordered tensors, the reference contract)
    op_params = orc.VsaParams(w, bias, k, activation=act)
    fwd = orc.vsa_forward(OL, hidden, q, kk, v, op_params)
    grads = orc.vsa_backward(OL, fwd, hidden, q, kk, v, op_params, dout)
    # GPU
    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda().bfloat16()
    params = vsa.VsaParams(dev(w), torch.from_numpy(bias).cuda(), k, activation=act)
    h = dev(hidden)
    gc, gf = vsa.gates_from_hidden(h, params, H, d)
    op = vsa.VsaOp(L, B, H, d, k, raster=False)
    out = op.forward(dev(q), dev(kk), dev(v), gc, gf)
    np.testing.assert_array_equal(op.sel.cpu().numpy(), fwd.coarse.sel)
    assert_close(host(out), fwd.out, torch.bfloat16, "out")
    dq, dk, dv, dgc, dgf = op.backward(dev(dout))
    dhidden, dw, db = vsa.gate_backward(h, params, gc, gf, dgc, dgf)
    for got, ref, n in ((dq, grads.dq, "dq"), (dk, grads.dk, "dk"), (dv, grads.dv, "dv"),
                        (dhidden, grads.dhidden, "dhidden")):
        assert_close(host(got), np.asarray(ref).reshape(tuple(got.shape)), torch.bfloat16, n)
    # dWg / dbias reduce bf16 gate gradients over all S tokens: the error scales with the
    # reduction, so they are checked relative to the tensor's scale (norm and max)
    for got, ref, n in ((dw, grads.dgate_weight, "dWg"), (db, grads.dgate_bias, "dbias")):
        g, r = host(got).astype(np.float64), np.asarray(ref, np.float64).reshape(tuple(got.shape))
        assert np.linalg.norm(g - r) / np.linalg.norm(r) < 1e-2, n
        assert np.abs(g - r).max() < 1e-2 * np.abs(r).max(), n


@pytest.mark.parametrize("act,bias", [(0, False), (1, True)], ids=["identity", "sigmoid-bias"])
def test_public_vsa_forward_backward(vsa, act, bias):
    """The reference signatures vsa_forward(layout, hidden, q, k, v, params, sel_override)
    and vsa_backward(layout, fwd, hidden, q, k, v, params, dout) (vsa.hpp:89-93, 129-133),
    through the native operator context (vsa_forward / vsa_backward of the C ABI) vs the
    oracle (oracle.py vsa_forward / vsa_backward)."""
    grid, B, H, d, md, k = (8, 12, 12), 2, 2, 64, 256, 5
    L = vsa.TileLayout(*grid)
    OL = orc.TileLayout(*grid, 4, 4, 4)
    rng = orc.Rng(73)
    S = L.seq_len
    bf = lambda a: rounded(a, torch.bfloat16)
    hidden = bf(orc.randn(rng, B, 1, S, md, np.float32))
    q, kk, v = (bf(orc.randn(rng, B, H, S, d, np.float32)) for _ in range(3))
    w = bf(orc.randn_matrix(rng, md, 2 * H * d, np.float32, 1.0 / np.sqrt(md)))
    b = orc.randn_matrix(rng, 1, 2 * H * d, np.float32, 0.1).reshape(-1) if bias else None
    dout = bf(orc.randn(rng, B, H, S, d, np.float32))
    oparams = orc.VsaParams(w, b, k, activation=act)
    fwd = orc.vsa_forward(OL, hidden, q, kk, v, oparams)
    grads = orc.vsa_backward(OL, fwd, hidden, q, kk, v, oparams, dout)
    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda().bfloat16()
    params = vsa.VsaParams(dev(w), None if b is None else torch.from_numpy(b).cuda(), k, activation=act)
    h, qd, kd, vd = dev(hidden), dev(q), dev(kk), dev(v)
    out = vsa.vsa_forward(L, h, qd, kd, vd, params)
    np.testing.assert_array_equal(out.fine_sel.cpu().numpy(), fwd.fine_sel)
    assert_close(host(out.out), fwd.out, torch.bfloat16, "out")
    assert_close(host(out.gate_coarse), fwd.gate_coarse, torch.bfloat16, "gate_coarse")
    assert_close(host(out.fine.out), fwd.fine_out, torch.bfloat16, "fine.out")
    np.testing.assert_allclose(host(out.fine.row_lse).reshape(-1), np.asarray(fwd.fine_row_lse).reshape(-1),
                               atol=2e-2, rtol=1e-2)
    g = vsa.vsa_backward(L, out, h, qd, kd, vd, params, dev(dout))
    for got, ref, n in ((g.dq, grads.dq, "dq"), (g.dk, grads.dk, "dk"), (g.dv, grads.dv, "dv"),
                        (g.dhidden, grads.dhidden, "dhidden")):
        assert_close(host(got), np.asarray(ref).reshape(tuple(got.shape)), torch.bfloat16, n)
    refs = [(g.dgate_weight, grads.dgate_weight, "dWg")] + ([(g.dgate_bias, grads.dgate_bias, "dbias")] if bias else [])
    for got, ref, n in refs:
        gg, r = host(got).astype(np.float64), np.asarray(ref, np.float64).reshape(tuple(got.shape))
        assert np.linalg.norm(gg - r) / np.linalg.norm(r) < 1e-2, n


def test_public_vsa_adaptation_init_is_dense(vsa):
    """VsaParams::adaptation_init (Wg = 0, Gf = 1, k = nc) reproduces dense attention, and
    the fine half of dWg is exactly zero (test_vsa.cpp:32-52)."""
    grid, B, H, d, md = (8, 12, 12), 1, 2, 128, 256
    L = vsa.TileLayout(*grid)
    OL = orc.TileLayout(*grid, 4, 4, 4)
    rng = orc.Rng(74)
    S = L.seq_len
    bf = lambda a: rounded(a, torch.bfloat16)
    hidden = bf(orc.randn(rng, B, 1, S, md, np.float32))
    q, kk, v, dout = (bf(orc.randn(rng, B, H, S, d, np.float32)) for _ in range(4))
    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda().bfloat16()
    params = vsa.VsaParams.adaptation_init(md, H, d, L.num_cubes)
    h, qd, kd, vd = dev(hidden), dev(q), dev(kk), dev(v)
    out = vsa.vsa_forward(L, h, qd, kd, vd, params)
    dense = orc.dense_forward(q, kk, v)[0]
    assert_close(host(out.out), dense, torch.bfloat16, "adaptation out == dense")
    g = vsa.vsa_backward(L, out, h, qd, kd, vd, params, dev(dout))
    dW = host(g.dgate_weight)
    assert (dW[:, H * d:] == 0).all(), "fine half of dWg must be exactly 0"
    with pytest.raises(ValueError):
        vsa.vsa_backward(L, None, h, qd, kd, vd, params, dev(dout))
