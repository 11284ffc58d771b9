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
