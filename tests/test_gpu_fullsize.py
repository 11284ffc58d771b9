# SPDX-License-Identifier: Apache-2.0
"""Full-size properties at BASELINE.json configs[1] (the Wan2.1-1.3B 480p grid,
21x30x52 tokens, zero-padded to 624 cubes, d = 128, top-k 78), where the CPU oracle
is too slow: the tcgen05 operator against the oracle-validated SIMT CUDA path on the
same bf16 inputs (2 heads), run-to-run bitwise determinism, block-map validity and
transposed-map consistency, and linearity of the backward in dO."""
import numpy as np
import pytest
import torch

from gpu_helpers import assert_close, host

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def vsa():
    import paper_2505_13389_b200 as v

    v.lib()
    return v


@pytest.fixture(scope="module")
def problem(vsa):
    L = vsa.TileLayout(21, 30, 52, pad=True)
    B, H, d, k = 1, 2, 128, 78
    g = torch.Generator(device="cuda").manual_seed(2024)
    x = [torch.randn((B, H, L.seq_len, d), generator=g, device="cuda").bfloat16() for _ in range(7)]
    return L, B, H, d, k, x


def run(vsa, L, B, H, d, k, x, dout, **kw):
    op = vsa.VsaOp(L, B, H, d, k, **kw)
    o = op.forward(*x[:5]).clone()
    g = [t.clone() for t in op.backward(dout)]
    return op, o, g


def test_fullsize_tcgen05_matches_simt(vsa, problem):
    L, B, H, d, k, x = problem
    op, o, g = run(vsa, L, B, H, d, k, x, x[5])
    _, o_s, g_s = run(vsa, L, B, H, d, k, x, x[5], force_simt=True)
    assert L.num_cubes == 624 and L.seq_len == 32760
    assert_close(host(o), host(o_s), torch.bfloat16, "out")
    for a, b, n in zip(g, g_s, ("dq", "dk", "dv", "dgc", "dgf")):
        assert_close(host(a), host(b), torch.bfloat16, n)


def test_fullsize_deterministic_and_maps_valid(vsa, problem):
    L, B, H, d, k, x = problem
    op1, o1, g1 = run(vsa, L, B, H, d, k, x, x[5])
    op2, o2, g2 = run(vsa, L, B, H, d, k, x, x[5])
    assert torch.equal(o1, o2) and all(torch.equal(a, b) for a, b in zip(g1, g2))
    sel = op1.sel.cpu().numpy().reshape(B * H * L.num_cubes, k)
    assert (np.diff(sel, axis=1) > 0).all() and sel.min() >= 0 and sel.max() < L.num_cubes
    offs, idx = op1.selT_offs.cpu().numpy(), op1.selT_idx.cpu().numpy()
    for u in range(B * H):  # CSR transpose: same (q, kc) pairs, ascending q per key cube
        assert offs[u, 0] == 0 and offs[u, -1] == L.num_cubes * k
        counts = np.bincount(sel[u * L.num_cubes:(u + 1) * L.num_cubes].ravel(), minlength=L.num_cubes)
        assert (np.diff(offs[u]) == counts).all()
        for kc in (0, 1, 311, 623):
            lst = idx[u, offs[u, kc]:offs[u, kc + 1]]
            assert (np.diff(lst) > 0).all()
            assert set(lst) == set(np.nonzero((sel[u * L.num_cubes:(u + 1) * L.num_cubes] == kc).any(1))[0])


def test_fullsize_backward_linear_in_dout(vsa, problem):
    L, B, H, d, k, x = problem
    op = vsa.VsaOp(L, B, H, d, k)
    op.forward(*x[:5])
    ga = [t.float() for t in op.backward(x[5])]
    gb = [t.float() for t in op.backward(x[6])]
    gab = [t.float() for t in op.backward((x[5].float() + x[6].float()).bfloat16())]
    for a, b, ab, n in zip(ga, gb, gab, ("dq", "dk", "dv", "dgc", "dgf")):
        # bf16 rounding of dO1 + dO2 and of each result bounds the deviation
        assert_close(host(ab), host(a + b), torch.bfloat16, n)


def test_coarse_large_bitexact(vsa):
    """The coarse stage at a size with many GEMM tiles per launch (6 heads, nc = 576
    with edge tiles): probabilities, block map and Oc bit-exact with the oracle,
    coarse gradients equal to the oracle's."""
    import oracle as orc

    L = vsa.TileLayout(16, 48, 48)
    OL = orc.TileLayout(16, 48, 48, 4, 4, 4)
    B, H, d, k = 1, 6, 128, 72
    rng = orc.Rng(36)
    q, kk, v, doc = (orc.randn(rng, B, H, L.seq_len, d, np.float32) for _ in range(4))
    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    art = vsa.coarse_forward_select(L, dev(q), dev(kk), dev(v), k)
    ref = orc.coarse_forward_select(OL, q, kk, v, k)
    assert L.num_cubes == 576
    np.testing.assert_array_equal(art.ac.cpu().numpy(), ref.ac)
    np.testing.assert_array_equal(art.sel.cpu().numpy(), ref.sel)
    np.testing.assert_array_equal(art.oc_cube.cpu().numpy(), ref.oc_cube)
    got = vsa.coarse_backward(art, L, dev(doc), dev(q), dev(kk), dev(v))
    exp = orc.coarse_backward(ref, OL, doc, q, kk, v)
    for g, e, n in zip(got, exp, ("dq", "dk", "dv")):
        np.testing.assert_allclose(g.cpu().numpy(), e, rtol=1e-5, atol=1e-6, err_msg=n)
