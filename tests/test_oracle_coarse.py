# SPDX-License-Identifier: Apache-2.0
"""Oracle pinning: the reference coarse-stage tests (proj/tests/test_coarse.cpp)."""
import numpy as np
import pytest


def test_pool_constant(orc):
    L = orc.TileLayout(4, 4, 4, 2, 2, 2)
    x = np.full((1, 2, L.seq_len, 3), 2.5)
    for mode in (orc.KMEAN, orc.KMAX):
        p = orc.pool_cubes(L, x, mode)
        assert p.shape[2] == L.num_cubes and (p == 2.5).all()


def test_pool_one_to_b(orc):
    L = orc.TileLayout(2, 2, 2, 2, 2, 2)
    x = np.arange(1, 9, dtype=np.float64).reshape(1, 1, 8, 1)
    assert orc.pool_cubes(L, x, orc.KMEAN)[0, 0, 0, 0] == pytest.approx(4.5)
    assert orc.pool_cubes(L, x, orc.KMAX)[0, 0, 0, 0] == 8.0


def test_pool_loop_oracle(orc):
    L = orc.TileLayout(4, 4, 4, 2, 2, 2)
    rng = orc.Rng(31)
    x = orc.randn(rng, 1, 1, 64, 4)
    mean, mx = orc.pool_cubes(L, x, orc.KMEAN), orc.pool_cubes(L, x, orc.KMAX)
    cube = x[0, 0].reshape(L.num_cubes, L.cube_size, 4)
    np.testing.assert_allclose(mean[0, 0], cube.sum(axis=1) / 8.0, rtol=1e-12)
    np.testing.assert_array_equal(mx[0, 0], cube.max(axis=1))


def test_k_equals_nc_selects_all(orc):
    L = orc.TileLayout(4, 4, 4, 2, 2, 2)
    rng = orc.Rng(32)
    q, k, v = (orc.randn(rng, 1, 2, 64, 8, np.float32) for _ in range(3))
    art = orc.coarse_forward_select(L, q, k, v, L.num_cubes)
    np.testing.assert_array_equal(art.sel, orc.all_cubes(1, 2, L.num_cubes))


def test_aligned_key_cube_wins(orc):
    L = orc.TileLayout(4, 2, 2, 2, 2, 2)
    D = 4
    q, k, v = (np.zeros((1, 1, L.seq_len, D)) for _ in range(3))
    for i in range(L.seq_len):
        q[0, 0, i, 0] = 1.0
        if i // L.cube_size == 1:
            k[0, 0, i, 0] = 10.0
        else:
            k[0, 0, i, 1] = 1.0
    art = orc.coarse_forward_select(L, q, k, v, 1)
    assert (art.sel[0, 0, :, 0] == 1).all()
    qc, kc = orc.pool_cubes(L, q), orc.pool_cubes(L, k)
    scores = qc[0, 0] @ kc[0, 0].T / np.sqrt(D)
    assert (scores.argmax(axis=1) == 1).all()


def test_topk_scores_equal_probs(orc):
    rng = orc.Rng(33)
    n, k = 24, 7
    for _ in range(50):
        s = orc.randn_matrix(rng, 1, n)[0]
        p = np.exp(s - s.max())
        p /= p.sum()
        np.testing.assert_array_equal(orc.topk_row(s, k), orc.topk_row(p, k))


def test_topk_affine_and_ties(orc):
    rng = orc.Rng(34)
    n, k = 16, 5
    for _ in range(50):
        s = orc.randn_matrix(rng, 1, n)[0]
        slope = rng.uniform_real(0.1, 5.0)
        shift = rng.uniform_real(-3.0, 3.0)
        np.testing.assert_array_equal(orc.topk_row(s, k), orc.topk_row(s * slope + shift, k))
    tied = np.array([1.0, 5.0, 5.0, 0.0, 5.0, 2.0])
    np.testing.assert_array_equal(orc.topk_row(tied, 3), [1, 2, 4])


def test_coarse_invariants(orc):
    L = orc.TileLayout(4, 4, 2, 2, 2, 2)
    rng = orc.Rng(35)
    q, k, v = (orc.randn(rng, 2, 2, L.seq_len, 6) for _ in range(3))
    art = orc.coarse_forward_select(L, q, k, v, 2)
    orc.validate(art.sel)
    np.testing.assert_allclose(art.ac.sum(axis=-1), 1.0, rtol=1e-6)
    oc = art.oc.reshape(2, 2, L.num_cubes, L.cube_size, 6)
    assert (oc == oc[:, :, :, :1]).all()
    with pytest.raises(ValueError):
        orc.coarse_forward_select(L, q, k, v, 0)
    with pytest.raises(ValueError):
        orc.coarse_forward_select(L, q, k, v, L.num_cubes + 1)


def test_coarse_backward_cases(orc):
    rng = orc.Rng(36)
    L = orc.TileLayout(4, 2, 2, 2, 2, 2)
    q, k, v = (orc.randn(rng, 1, 1, L.seq_len, 4) for _ in range(3))
    art = orc.coarse_forward_select(L, q, k, v, 1)
    g = orc.coarse_backward(art, L, np.zeros_like(q), q, k, v)
    assert all(not x.any() for x in g)

    L1 = orc.TileLayout(2, 2, 2, 2, 2, 2)
    q, k, v = (orc.randn(rng, 1, 1, 8, 4) for _ in range(3))
    art = orc.coarse_forward_select(L1, q, k, v, 1)
    dout = orc.randn(rng, 1, 1, 8, 4)
    dq, dk, dv = orc.coarse_backward(art, L1, dout, q, k, v)
    exp = dout[0, 0].sum(axis=0) / 8.0
    assert np.abs(dv[0, 0] - exp).max() < 1e-14
    assert np.abs(dq).max() < 1e-14 and np.abs(dk).max() < 1e-14

    L2 = orc.TileLayout(4, 4, 2, 2, 2, 2)
    q, k, v = (orc.randn(rng, 1, 1, L2.seq_len, 4) for _ in range(3))
    art = orc.coarse_forward_select(L2, q, k, v, 2)
    dout = orc.randn(rng, 1, 1, L2.seq_len, 4)
    dq, dk, dv = orc.coarse_backward(art, L2, dout, q, k, v)
    doc = dout[0, 0].reshape(L2.num_cubes, L2.cube_size, 4).sum(axis=1)
    dvc = art.ac[0, 0].T @ doc
    tok = dv[0, 0].reshape(L2.num_cubes, L2.cube_size, 4).sum(axis=1)
    assert np.abs(tok - dvc).max() < 1e-12


def coarse_gradcheck(orc, mode, seed):
    L = orc.TileLayout(4, 4, 4, 2, 2, 2)
    rng = orc.Rng(seed)
    q, k, v = (orc.randn(rng, 1, 2, L.seq_len, 4) for _ in range(3))
    loss = lambda: 0.5 * float((orc.coarse_forward_select(L, q, k, v, 2, mode).oc ** 2).sum())
    art = orc.coarse_forward_select(L, q, k, v, 2, mode)
    g = orc.coarse_backward(art, L, art.oc.copy(), q, k, v)
    return max(orc.max_rel_err(gi, orc.fd_gradient(x, 1e-5, loss)) for x, gi in zip((q, k, v), g))


def test_coarse_gradcheck(orc):
    assert coarse_gradcheck(orc, orc.KMEAN, 41) < 1e-6
    assert coarse_gradcheck(orc, orc.KMAX, 42) < 1e-6
