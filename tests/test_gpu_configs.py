# SPDX-License-Identifier: Apache-2.0
"""Oracle parity at every BASELINE.json config, on head subsets the CPU oracle
finishes in seconds (the oracle is ~2 s per Wan2.1-1.3B head, fwd + bwd, on the
box's cores). Each case runs the full bf16 operator (K1..K6, raster in / raster out)
and compares with the oracle on the same bf16-rounded inputs (zero-padded problem,
SURVEY.md §7.2 H4):

* the coarse block map bit-exact (the coarse stage is the canonical fp32 order on
  the pooled bf16 values — the "coarse stage runs in fp32" arm of north_star);
* out, dq, dk, dv, dgc, dgf within 2e-2 abs + 1e-2 rel per element and 1e-2
  relative in norm (north_star's bf16 tolerance);
* the fine stage's row_lse / row_max (FineSaved, fine.hpp:13-14) against the oracle's.

Configs: Wan2.1-1.3B (2 heads of the 21x30x52 layer, k=78 of 624), DiT (2 (b,h)
units of 16x32x32, d=64, k=32 of 256), Wan2.1-14B (1 head of 21x45x80, k=144 of
1440), the paper sweep (16^3 and 32^3, d=64 and d=128, 50% and 95% sparsity), plus
the fp32 coarse map at nc=624 / 1440 and the bf16 SIMT path."""
import numpy as np
import pytest
import torch

import oracle as orc
from gpu_helpers import Problem, assert_close, host, rounded, to_dev

pytestmark = pytest.mark.gpu
BF = torch.bfloat16


@pytest.fixture(scope="module")
def vsa():
    import paper_2505_13389_b200 as v

    v.lib()
    orc.set_num_threads(max(1, orc.max_threads()))
    return v


def sweep_k(nc, sparsity):
    return max(1, int(round(nc * (1.0 - sparsity))))


CASES = {
    # BASELINE configs[1]: Wan2.1-1.3B 480p layer, 2 of its 12 heads
    "wan13": dict(grid=(21, 30, 52), B=1, H=2, d=128, top_k=78),
    # configs[4]: DiT pretraining batch, 2 (b, h) units (batch 2 x 1 head)
    "dit": dict(grid=(16, 32, 32), B=2, H=1, d=64, top_k=32),
    # configs[3]: Wan2.1-14B 720p layer, 1 of its 40 heads (nc = 1440, 90%)
    "wan14": dict(grid=(21, 45, 80), B=1, H=1, d=128, top_k=144),
    # configs[2]: the paper kernel sweep
    "sweep16_d64_s50": dict(grid=(16, 16, 16), B=1, H=1, d=64, top_k=sweep_k(64, 0.5)),
    "sweep16_d64_s95": dict(grid=(16, 16, 16), B=1, H=1, d=64, top_k=sweep_k(64, 0.95)),
    "sweep16_d128_s50": dict(grid=(16, 16, 16), B=1, H=1, d=128, top_k=sweep_k(64, 0.5)),
    "sweep16_d128_s95": dict(grid=(16, 16, 16), B=1, H=1, d=128, top_k=sweep_k(64, 0.95)),
    "sweep32_d64_s50": dict(grid=(32, 32, 32), B=1, H=1, d=64, top_k=sweep_k(512, 0.5)),
    "sweep32_d64_s95": dict(grid=(32, 32, 32), B=1, H=1, d=64, top_k=sweep_k(512, 0.95)),
    "sweep32_d128_s50": dict(grid=(32, 32, 32), B=1, H=1, d=128, top_k=sweep_k(512, 0.5)),
    "sweep32_d128_s95": dict(grid=(32, 32, 32), B=1, H=1, d=128, top_k=sweep_k(512, 0.95)),
}


@pytest.mark.parametrize("name", list(CASES))
def test_config_operator_vs_oracle(vsa, name):
    cfg = CASES[name]
    p = Problem(**cfg, seed=2024)
    L = vsa.TileLayout(*p.grid, pad=True)
    op = vsa.VsaOp(L, p.B, p.H, p.d, p.top_k, dtype=BF)
    out = op.forward(*(to_dev(x, BF) for x in (p.q, p.k, p.v, p.gc, p.gf)))
    grads = op.backward(to_dev(p.dout, BF))
    torch.cuda.synchronize()
    ref = p.oracle(BF)
    np.testing.assert_array_equal(op.sel.cpu().numpy(), ref["sel"], err_msg=f"{name}: block map")
    assert_close(host(out), ref["out"], BF, f"{name} out")
    for g, n in zip(grads, ("dq", "dk", "dv", "dgc", "dgf")):
        assert_close(host(g), ref[n], BF, f"{name} {n}")
    # FineSaved row_lse of the operator's fine stage (tile order, padded rows included)
    lse = op.lse.cpu().numpy().reshape(ref["lse"].shape)
    np.testing.assert_allclose(lse, ref["lse"], atol=2e-2, rtol=1e-2, err_msg=f"{name}: row_lse")


@pytest.mark.parametrize("name", ["wan13", "dit", "sweep16_d128_s95"])
def test_config_fine_row_max_vs_oracle(vsa, name):
    """fine_forward's FineSaved (row_max, row_lse; fine.hpp:13-14, 93-96) on the oracle's
    block map, tile-ordered inputs (the reference contract)."""
    cfg = dict(CASES[name])
    cfg["H"] = 1
    cfg["B"] = 1
    p = Problem(**cfg, seed=7)
    L = vsa.TileLayout(*p.grid, pad=True)
    q, k, v = (p.pad_tile(rounded(x, BF)) for x in (p.q, p.k, p.v))
    art = orc.coarse_forward_select(p.olayout, q, k, v, p.top_k)
    fo, fmax, flse = orc.fine_forward(p.olayout, q, k, v, art.sel)
    res = vsa.fine_forward(L, to_dev(q, BF), to_dev(k, BF), to_dev(v, BF), to_dev(art.sel, torch.int32))
    assert_close(host(res.out), fo, BF, f"{name} fine out")
    # row_max is the exact running max of the scaled scores (tau = 0 when requested)
    np.testing.assert_allclose(res.row_max.cpu().numpy().reshape(fmax.shape), fmax, atol=2e-2, rtol=1e-2,
                               err_msg=f"{name}: row_max")
    np.testing.assert_allclose(res.row_lse.cpu().numpy().reshape(flse.shape), flse, atol=2e-2, rtol=1e-2,
                               err_msg=f"{name}: row_lse")


@pytest.mark.parametrize("grid,H", [((21, 30, 52), 2), ((21, 45, 80), 1)], ids=["nc624", "nc1440"])
def test_config_coarse_map_fp32_bitexact(vsa, grid, H):
    """The fp32 coarse stage (tile_pool + coarse_forward_select) at the Wan2.1 sizes:
    pooled cubes, probabilities Ac, Oc and the top-k map bit-exact with the oracle."""
    d, k = 128, (78 if grid[1] == 30 else 144)
    p = Problem(grid=grid, B=1, H=H, d=d, top_k=k, seed=31)
    L = vsa.TileLayout(*grid, pad=True)
    q, kk, v = (p.pad_tile(np.ascontiguousarray(x, np.float32)) for x in (p.q, p.k, p.v))
    art = vsa.coarse_forward_select(L, *(to_dev(x, torch.float32) for x in (q, kk, v)), k)
    ref = orc.coarse_forward_select(p.olayout, q, kk, v, k, token_oc=False)
    np.testing.assert_array_equal(art.sel.cpu().numpy(), ref.sel)
    np.testing.assert_array_equal(art.ac.cpu().numpy(), ref.ac)
    np.testing.assert_array_equal(art.qc.cpu().numpy(), ref.qc)


def test_bf16_simt_path_vs_oracle(vsa):
    """The SIMT kernels in bf16 (VSA_FINE_FORCE_SIMT, the debug / cross-check path) vs the
    oracle on a padded grid with both head dims the tcgen05 path covers."""
    for d in (64, 128):
        p = Problem(grid=(9, 14, 14), B=1, H=2, d=d, top_k=5, seed=61)
        L = vsa.TileLayout(*p.grid, pad=True)
        op = vsa.VsaOp(L, p.B, p.H, p.d, p.top_k, dtype=BF, force_simt=True)
        out = op.forward(*(to_dev(x, BF) for x in (p.q, p.k, p.v, p.gc, p.gf)))
        grads = op.backward(to_dev(p.dout, BF))
        ref = p.oracle(BF)
        np.testing.assert_array_equal(op.sel.cpu().numpy(), ref["sel"])
        assert_close(host(out), ref["out"], BF, f"simt d{d} out")
        for g, n in zip(grads, ("dq", "dk", "dv", "dgc", "dgf")):
            assert_close(host(g), ref[n], BF, f"simt d{d} {n}")


def test_bf16_unsupported_shape_is_explicit(vsa):
    """bf16 outside the tcgen05 shapes (cube != 64 or d not in {64, 128}) is an explicit
    error unless the SIMT kernels are requested (no silent dispatch)."""
    L = vsa.TileLayout(8, 8, 8, 2, 2, 2)
    with pytest.raises(ValueError, match="SIMT"):
        vsa.VsaOp(L, 1, 1, 64, 2, dtype=BF)
    x = torch.zeros((1, 1, L.seq_padded, 96), dtype=BF, device="cuda")
    sel = vsa.all_cubes(1, 1, L.num_cubes)
    with pytest.raises(ValueError, match="SIMT"):
        vsa.fine_forward(L, x, x, x, sel)
    res = vsa.fine_forward(L, x, x, x, sel, force_simt=True)
    assert torch.isfinite(res.out.float()).all()
