# SPDX-License-Identifier: Apache-2.0
"""Oracle pinning: the reference operator tests (proj/tests/test_vsa.cpp) and the
end-to-end gradcheck suite (proj/include/vsa/verify.hpp:147-215)."""
import numpy as np
import pytest


def make_problem(orc, B, H, D, md, seed, dt=np.float64):
    L = orc.TileLayout(4, 4, 4, 2, 2, 2)
    rng = orc.Rng(seed)
    hidden = orc.randn(rng, B, 1, L.seq_len, md, dt)
    q, k, v = (orc.randn(rng, B, H, L.seq_len, D, dt) for _ in range(3))
    return L, hidden, q, k, v


def test_adaptation_equals_dense(orc):
    L, hid, q, k, v = make_problem(orc, 2, 2, 8, 12, 71, np.float32)
    p = orc.VsaParams.adaptation_init(12, 2, 8, L.num_cubes, np.float32)
    out = orc.vsa_forward(L, hid, q, k, v, p)
    do, _, lse = orc.dense_forward(q, k, v)
    assert np.abs(out.out - do).max() < 1e-5
    dout = orc.randn(orc.Rng(72), 2, 2, L.seq_len, 8, np.float32)
    g = orc.vsa_backward(L, out, hid, q, k, v, p, dout)
    dg = orc.dense_backward(q, k, v, None, dout, lse)
    for a, b in zip((g.dq, g.dk, g.dv), dg):
        assert np.abs(a - b).max() < 1e-5
    assert np.abs(g.dgate_weight[:, :16]).max() > 0
    assert (g.dgate_weight[:, 16:] == 0).all()


def test_unit_coarse_gate_reduces_to_coarse(orc):
    L, hid, q, k, v = make_problem(orc, 1, 2, 8, 10, 73)
    bias = np.zeros(32)
    bias[:16] = 1.0
    p = orc.VsaParams(np.zeros((10, 32)), bias, 3)
    out = orc.vsa_forward(L, hid, q, k, v, p)
    assert (out.out == out.coarse.oc).all()


def test_single_cube_layout(orc):
    L = orc.TileLayout(2, 2, 2, 2, 2, 2)
    rng = orc.Rng(74)
    hid = orc.randn(rng, 1, 1, L.seq_len, 6)
    q, k, v = (orc.randn(rng, 1, 1, L.seq_len, 4) for _ in range(3))
    p = orc.VsaParams.random_init(6, 1, 4, 1, rng)
    out = orc.vsa_forward(L, hid, q, k, v, p)
    do, _, _ = orc.dense_forward(q, k, v)
    vmean = v[0, 0].mean(axis=0)
    exp = out.gate_coarse[0, 0] * vmean + out.gate_fine[0, 0] * do[0, 0]
    assert np.abs(out.out[0, 0] - exp).max() < 1e-12


def test_zero_upstream_zero_grads(orc):
    L, hid, q, k, v = make_problem(orc, 1, 2, 4, 8, 75)
    rng = orc.Rng(76)
    p = orc.VsaParams.random_init(8, 2, 4, 3, rng)
    p.gate_bias = orc.randn_matrix(rng, 1, 16)[0]
    out = orc.vsa_forward(L, hid, q, k, v, p)
    g = orc.vsa_backward(L, out, hid, q, k, v, p, np.zeros_like(q))
    for x in (g.dq, g.dk, g.dv, g.dhidden, g.dgate_weight, g.dgate_bias):
        assert (x == 0).all()


def test_missing_artifacts_rejected(orc):
    L, hid, q, k, v = make_problem(orc, 1, 1, 4, 6, 77)
    p = orc.VsaParams.random_init(6, 1, 4, 2, orc.Rng(78))
    with pytest.raises(ValueError):
        orc.vsa_backward(L, None, hid, q, k, v, p, np.zeros_like(q))


def test_batch_permutation_invariance(orc):
    L, hid, q, k, v = make_problem(orc, 3, 2, 4, 8, 79)
    p = orc.VsaParams.random_init(8, 2, 4, 2, orc.Rng(80))
    out = orc.vsa_forward(L, hid, q, k, v, p)
    order = [2, 0, 1]
    out2 = orc.vsa_forward(L, hid[order], q[order], k[order], v[order], p)
    np.testing.assert_array_equal(out2.out, out.out[order])


def test_sigmoid_gate_gradcheck(orc):
    L = orc.TileLayout(2, 4, 4, 2, 2, 2)
    rng = orc.Rng(81)
    D, md, H = 4, 7, 2
    hid = orc.randn(rng, 1, 1, L.seq_len, md)
    q, k, v = (orc.randn(rng, 1, H, L.seq_len, D) for _ in range(3))
    p = orc.VsaParams.random_init(md, H, D, L.num_cubes, rng)
    p.activation = orc.SIGMOID
    p.gate_bias = orc.randn_matrix(rng, 1, 2 * H * D, stddev=0.2)[0]
    loss = lambda: 0.5 * float((orc.vsa_forward(L, hid, q, k, v, p).out ** 2).sum())
    out = orc.vsa_forward(L, hid, q, k, v, p)
    g = orc.vsa_backward(L, out, hid, q, k, v, p, out.out.copy())
    worst = max(orc.max_rel_err(gi, orc.fd_gradient(x, 1e-5, loss))
                for x, gi in ((hid, g.dhidden), (p.gate_weight, g.dgate_weight), (p.gate_bias, g.dgate_bias)))
    assert worst < 1e-6


def run_gradcheck_suite(orc, cases=4, step=1e-5, tol=1e-5, seed=7):
    """run_gradcheck_suite (verify.hpp:147-215)."""
    rng = orc.Rng(seed)
    shapes = [(4, 4, 4, 2, 2, 2, 1, 2, 8, 16, 3), (2, 4, 4, 2, 2, 2, 2, 1, 4, 9, 2),
              (4, 4, 2, 2, 1, 2, 1, 2, 4, 12, 5), (2, 2, 2, 2, 2, 2, 2, 2, 8, 16, 1)]
    lines = []
    for c in range(cases):
        t, h, w, ct, ch, cw, B, H, D, md, tk = shapes[c % 4]
        L = orc.TileLayout(t, h, w, ct, ch, cw)
        top_k = min(tk, L.num_cubes)
        for _ in range(16):
            q, k, v = (orc.randn(rng, B, H, L.seq_len, D) for _ in range(3))
            hid = orc.randn(rng, B, 1, L.seq_len, md)
            p = orc.VsaParams.random_init(md, H, D, top_k, rng)
            p.gate_bias = orc.randn_matrix(rng, 1, 2 * H * D, stddev=0.3)[0]
            if top_k == L.num_cubes:
                break
            art = orc.coarse_forward_select(L, q, k, v, top_k)
            srt = -np.sort(-art.ac, axis=-1)
            if (srt[..., top_k - 1] - srt[..., top_k]).min() > 1e-3:
                break
        loss = lambda: 0.5 * float((orc.vsa_forward(L, hid, q, k, v, p).out ** 2).sum())
        out = orc.vsa_forward(L, hid, q, k, v, p)
        g = orc.vsa_backward(L, out, hid, q, k, v, p, out.out.copy())
        for name, x, gi in (("Q", q, g.dq), ("K", k, g.dk), ("V", v, g.dv), ("hidden", hid, g.dhidden),
                            ("Wg", p.gate_weight, g.dgate_weight), ("gate_bias", p.gate_bias, g.dgate_bias)):
            lines.append((f"case {c}: d{name}", orc.max_rel_err(gi, orc.fd_gradient(x, step, loss))))
    return lines, tol


def test_gradcheck_suite(orc):
    lines, tol = run_gradcheck_suite(orc, cases=2)
    for name, err in lines:
        assert err < tol, (name, err)


def test_mean_pool_conservation(orc):
    L, hid, q, k, v = make_problem(orc, 1, 1, 4, 6, 82)
    rng = orc.Rng(83)
    p = orc.VsaParams.random_init(6, 1, 4, 2, rng)
    out = orc.vsa_forward(L, hid, q, k, v, p)
    dout = orc.randn(rng, 1, 1, L.seq_len, 4)
    doc = dout * out.gate_coarse
    _, _, dv = orc.coarse_backward(out.coarse, L, doc, q, k, v)
    b = L.cube_size
    dcube = doc[0, 0].reshape(L.num_cubes, b, 4).sum(axis=1)
    dvc = out.coarse.ac[0, 0].T @ dcube
    tok = dv[0, 0].reshape(L.num_cubes, b, 4).sum(axis=1)
    assert np.abs(tok - dvc).max() < 1e-12
