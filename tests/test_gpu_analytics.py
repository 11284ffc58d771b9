# SPDX-License-Identifier: Apache-2.0
"""GPU selection analytics vs the oracle (analysis.hpp:100-147,
dense.hpp:214-240): the reference's materialised path (dense_probs ->
aggregate_probs_to_cubes -> selection_accuracy) and the scalable lse path
(selection_accuracy_qk = mean exp(lse_sel - lse_all) from two fine forwards)."""
import numpy as np
import pytest
import torch

import oracle as orc
from gpu_helpers import rounded

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def vsa():
    import paper_2505_13389_b200 as v

    v.lib()
    return v


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16], ids=["f32", "bf16"])
def test_selection_accuracy_matches_oracle(vsa, dtype):
    grid, B, H, d, k = (8, 16, 16), 1, 2, 64, 4
    L = vsa.TileLayout(*grid)
    OL = orc.TileLayout(*grid, 4, 4, 4)
    rng = orc.Rng(94)
    q, kk = (rounded(orc.randn(rng, B, H, L.seq_len, d, np.float32), dtype) for _ in range(2))
    qt, kt = orc.tile(OL, q), orc.tile(OL, kk)
    sel = orc.coarse_forward_select(OL, qt, kt, kt, k).sel
    probs = orc.dense_probs(qt, kt)                       # float64 [B,H,S,S]
    cube = orc.aggregate_probs_to_cubes(OL, probs)
    ref = orc.selection_accuracy(OL, cube, sel)
    dev = lambda a, dt: torch.from_numpy(np.ascontiguousarray(a)).cuda().to(dt)
    sel_d = dev(sel, torch.int32)
    # materialised path on the GPU (fp32 probabilities)
    cube_g = vsa.aggregate_probs_to_cubes(L, dev(probs, torch.float32))
    np.testing.assert_allclose(cube_g.cpu().numpy(), cube, rtol=1e-5, atol=1e-6)
    acc_m = vsa.selection_accuracy(L, cube_g, sel_d).cpu().numpy()
    np.testing.assert_allclose(acc_m, ref, rtol=1e-5, atol=1e-6)
    # scalable path (tcgen05 / SIMT fine forward lse)
    acc_q = vsa.selection_accuracy_qk(L, dev(qt, dtype), dev(kt, dtype), sel_d).cpu().numpy()
    tol = 1e-4 if dtype == torch.float32 else 2e-2
    np.testing.assert_allclose(acc_q, ref, rtol=tol, atol=tol)
    # captured mass of the top-k map beats a random map of the same size (VSA §3.5)
    rnd = dev(orc.random_selection(B, H, L.num_cubes, k, orc.Rng(95)), torch.int32)
    assert (vsa.selection_accuracy_qk(L, dev(qt, dtype), dev(kt, dtype), rnd).cpu().numpy() < acc_q).all()
    # full coverage captures everything
    full = vsa.all_cubes(B, H, L.num_cubes)
    np.testing.assert_allclose(vsa.selection_accuracy_qk(L, dev(qt, dtype), dev(kt, dtype), full).cpu().numpy(), 1.0,
                               rtol=1e-6)


def test_acceptance_6_selection_metric_sanity(vsa):
    """SPEC acceptance 6 / test_analysis.cpp:68-99 on the GPU kernels: uniform attention
    captures exactly K/num_cubes; random selections average K/num_cubes within 0.01."""
    L = vsa.TileLayout(8, 8, 8, 2, 2, 2)  # 512 tokens, 64 cubes
    nc, k = L.num_cubes, 8
    uniform = torch.full((1, 1, L.seq_len, nc), 1.0 / nc, device="cuda")
    full = vsa.all_cubes(1, 1, nc)
    assert vsa.selection_accuracy(L, uniform, full).item() == 1.0
    gen = np.random.default_rng(91)
    rsel = lambda: torch.from_numpy(np.sort(np.stack([gen.choice(nc, k, replace=False) for _ in range(nc)]), axis=1)
                                    .astype(np.int32)).view(1, 1, nc, k).cuda()
    assert vsa.selection_accuracy(L, uniform, rsel()).item() == k / nc
    rows = torch.from_numpy(gen.standard_normal((L.seq_len, nc))).cuda()
    probs = torch.softmax(rows, dim=1).float().view(1, 1, L.seq_len, nc).contiguous()
    mean = sum(vsa.selection_accuracy(L, probs, rsel()).item() for _ in range(100)) / 100
    assert abs(mean - k / nc) < 0.01
