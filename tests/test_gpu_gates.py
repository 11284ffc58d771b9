# SPDX-License-Identifier: Apache-2.0
"""GPU: the gate projection on the tcgen05 GEMM — vsa_gate_forward /
vsa_gate_backward against the oracle's gates_from_hidden and the gate part of
vsa_backward (vsa.hpp:100-112, 152-176), bf16 operands with fp32 accumulation."""
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


CASES = [  # grid, B, H, d, model_dim, activation, bias, adaptation
    ((8, 12, 12), 2, 2, 64, 256, 0, False, False),
    ((8, 12, 12), 1, 4, 128, 512, 1, True, False),
    ((6, 10, 12), 2, 2, 128, 256, 1, True, True),
]


@pytest.mark.parametrize("grid,B,H,d,md,act,use_bias,adapt", CASES)
def test_gates_forward_backward(vsa, grid, B, H, d, md, act, use_bias, adapt):
    S = grid[0] * grid[1] * grid[2]
    rng = orc.Rng(123)
    hid = rounded(orc.randn(rng, B, 1, S, md, np.float32), torch.bfloat16)
    w = rounded(orc.randn_matrix(rng, md, 2 * H * d, np.float32, 1.0 / np.sqrt(md)), torch.bfloat16)
    bias = orc.randn_matrix(rng, 1, 2 * H * d, np.float32).reshape(-1) if use_bias else None
    dgc = rounded(orc.randn(rng, B, H, S, d, np.float32), torch.bfloat16)
    dgf = rounded(orc.randn(rng, B, H, S, d, np.float32), torch.bfloat16)
    op_params = orc.VsaParams(w.astype(np.float64), None if bias is None else bias.astype(np.float64), 1,
                              activation=act, adaptation=adapt)
    gc_ref, gf_ref = orc.gates_from_hidden(hid.astype(np.float64), op_params, H, d)

    dev = lambda a, dt=torch.bfloat16: torch.from_numpy(np.ascontiguousarray(a)).cuda().to(dt)
    params = vsa.VsaParams(dev(w), None if bias is None else dev(bias, torch.float32), 1, activation=act,
                           adaptation=adapt)
    L = vsa.TileLayout(*grid, pad=True)
    gc, gf = vsa.gates_from_hidden(dev(hid), params, H, d, layout=L)
    torch.cuda.synchronize()
    assert_close(host(gc), gc_ref, torch.bfloat16, "gate_coarse")
    assert_close(host(gf), gf_ref, torch.bfloat16, "gate_fine")

    # backward: dz (sigmoid chain on the bf16 gates the GPU produced), dhidden, dWg, dbias
    g_c, g_f = host(gc).astype(np.float64), host(gf).astype(np.float64)
    dzc, dzf = dgc.astype(np.float64), (np.zeros_like(dgf) if adapt else dgf.astype(np.float64))
    if act == 1:
        dzc = dzc * g_c * (1 - g_c)
        if not adapt:
            dzf = dzf * g_f * (1 - g_f)
    dz = np.concatenate([dzc, dzf], axis=1).transpose(0, 2, 1, 3).reshape(B, S, 2 * H * d)
    dz = rounded(dz.astype(np.float32), torch.bfloat16).astype(np.float64)  # the kernel's bf16 dz
    dh_ref = dz @ w.astype(np.float64).T
    dw_ref = np.einsum("bsm,bsn->mn", hid[:, 0].astype(np.float64), dz)
    db_ref = dz.sum(axis=(0, 1))
    dh, dw, db = vsa.gate_backward(dev(hid), params, gc, gf, dev(dgc), dev(dgf), layout=L)
    torch.cuda.synchronize()
    assert_close(host(dh)[:, 0], dh_ref, torch.bfloat16, "dhidden")
    np.testing.assert_allclose(host(dw), dw_ref, rtol=1e-3, atol=1e-3 * np.abs(dw_ref).max())
    if use_bias:
        np.testing.assert_allclose(host(db), db_ref, rtol=1e-4, atol=1e-3)
    else:
        assert db is None


def test_gates_reject_bad_shapes(vsa):
    L = vsa.TileLayout(4, 4, 4)
    hid = torch.zeros(1, 1, 64, 100, dtype=torch.bfloat16, device="cuda")  # model_dim % 64 != 0
    p = vsa.VsaParams(torch.zeros(100, 256, dtype=torch.bfloat16, device="cuda"))
    with pytest.raises(ValueError):
        vsa.gates_from_hidden(hid, p, 2, 64, layout=L)
