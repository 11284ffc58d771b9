# SPDX-License-Identifier: Apache-2.0
"""The TMA forms of the two HBM passes (K1+K2 tile / pool: one 5-D box per cube; K6a backward
prologue: slab boxes + bulk / box stores) against the thread-load kernels they replace
(VSA_HBM_TMA=0): every forward / backward output bitwise identical, on the operator, at
head dims 64 and 128, a padded odd grid, a grid that divides, and the adaptation mode."""
import os

import pytest
import torch

pytestmark = pytest.mark.gpu

CASES = [((9, 14, 22), 2, 2, 64, 6, False), ((16, 16, 16), 1, 2, 128, 8, False), ((5, 7, 9), 1, 3, 128, 3, False),
         ((8, 8, 8), 1, 2, 64, 2, True)]


def run(vsa, grid, B, H, d, k, adaptation):
    L = vsa.TileLayout(*grid, pad=True)
    op = vsa.VsaOp(L, B, H, d, k, adaptation=adaptation)
    g = torch.Generator(device="cuda").manual_seed(5)
    x = [torch.randn((B, H, L.seq_len, d), generator=g, device="cuda").bfloat16() for _ in range(6)]
    out = op.forward(*x[:5]).clone()
    grads = [t.clone() for t in op.backward(x[5])]
    torch.cuda.synchronize()
    return [out] + grads


@pytest.mark.parametrize("case", CASES, ids=["padded-d64", "d128", "odd-d128", "adapt-d64"])
def test_hbm_tma_bitwise_vs_thread_kernels(case):
    import paper_2505_13389_b200 as vsa

    vsa.lib()
    old = os.environ.pop("VSA_HBM_TMA", None)
    try:
        a = run(vsa, *case)
        os.environ["VSA_HBM_TMA"] = "0"
        b = run(vsa, *case)
    finally:
        os.environ.pop("VSA_HBM_TMA", None)
        if old is not None:
            os.environ["VSA_HBM_TMA"] = old
    for name, x, y in zip(("out", "dq", "dk", "dv", "dgc", "dgf"), a, b):
        assert torch.equal(x.view(torch.int16), y.view(torch.int16)), name
