# SPDX-License-Identifier: Apache-2.0
"""Oracle pinning: the reference dense-attention tests (proj/tests/test_dense.cpp)."""
import numpy as np
import pytest


def test_seq1_output_is_v(orc):
    rng = orc.Rng(1)
    q, k, v = (orc.randn(rng, 2, 2, 1, 8) for _ in range(3))
    out, _, _ = orc.dense_forward(q, k, v)
    np.testing.assert_array_equal(out, v)


def test_identical_keys_mean_of_v(orc):
    rng = orc.Rng(2)
    q = orc.randn(rng, 1, 1, 16, 4)
    v = orc.randn(rng, 1, 1, 16, 4)
    one = orc.randn_matrix(rng, 1, 4)
    k = np.broadcast_to(one, (1, 1, 16, 4)).copy()
    out, _, _ = orc.dense_forward(q, k, v)
    assert np.abs(out[0, 0] - v[0, 0].mean(axis=0)).max() < 1e-12


def test_single_allowed_key_copies_row(orc):
    rng = orc.Rng(3)
    q, k, v = (orc.randn(rng, 1, 1, 12, 6, np.float32) for _ in range(3))
    mask = np.zeros((12, 12), np.uint8)
    allowed = []
    for i in range(12):
        a = rng.uniform_int(0, 11)
        allowed.append(a)
        mask[i, a] = 1
    out, _, _ = orc.dense_forward(q, k, v, mask)
    for i in range(12):
        np.testing.assert_array_equal(out[0, 0, i], v[0, 0, allowed[i]])


def test_rejects_empty_row_and_nan(orc):
    rng = orc.Rng(4)
    q, k, v = (orc.randn(rng, 1, 1, 4, 2) for _ in range(3))
    mask = np.ones((4, 4), np.uint8)
    mask[2] = 0
    with pytest.raises(ValueError):
        orc.dense_forward(q, k, v, mask)
    bad = q.copy()
    bad[0, 0, 1, 1] = np.nan
    with pytest.raises(ValueError):
        orc.dense_forward(bad, k, v)


def test_all_true_mask_bitwise(orc):
    rng = orc.Rng(5)
    q, k, v = (orc.randn(rng, 2, 2, 33, 8, np.float32) for _ in range(3))
    w, _, lw = orc.dense_forward(q, k, v, np.ones((33, 33), np.uint8))
    wo, _, lwo = orc.dense_forward(q, k, v)
    np.testing.assert_array_equal(w, wo)
    np.testing.assert_array_equal(lw, lwo)


def test_permutation_equivariance(orc):
    rng = orc.Rng(7)
    q, k, v = (orc.randn(rng, 1, 1, 24, 8) for _ in range(3))
    perm = np.arange(24, dtype=np.int64)
    rng.shuffle(perm)
    base, _, _ = orc.dense_forward(q, k, v)
    pm, _, _ = orc.dense_forward(q[:, :, perm], k[:, :, perm], v[:, :, perm])
    assert np.abs(pm[0, 0] - base[0, 0, perm]).max() < 1e-12


def test_backward_edge_cases(orc):
    rng = orc.Rng(8)
    q, k, v = (orc.randn(rng, 1, 1, 6, 4) for _ in range(3))
    _, _, lse = orc.dense_forward(q, k, v)
    dq, dk, dv = orc.dense_backward(q, k, v, None, np.zeros_like(q), lse)
    assert not dq.any() and not dk.any() and not dv.any()
    q1, k1, v1, do1 = (orc.randn(rng, 1, 1, 1, 4) for _ in range(4))
    _, _, lse1 = orc.dense_forward(q1, k1, v1)
    dq, dk, dv = orc.dense_backward(q1, k1, v1, None, do1, lse1)
    np.testing.assert_array_equal(dv, do1)
    assert np.abs(dq).max() < 1e-15 and np.abs(dk).max() < 1e-15


def dense_gradcheck(orc, B, H, S, D, masked, seed):
    """test_dense.cpp:140-175."""
    rng = orc.Rng(seed)
    q, k, v = (orc.randn(rng, B, H, S, D) for _ in range(3))
    mask = np.ones((S, S), np.uint8)
    if masked:
        for i in range(S):
            anyv = False
            for j in range(S):
                mask[i, j] = rng.bernoulli(0.35)
                anyv |= bool(mask[i, j])
            if not anyv:
                mask[i, i] = 1
    loss = lambda: 0.5 * float((orc.dense_forward(q, k, v, mask)[0] ** 2).sum())
    out, _, lse = orc.dense_forward(q, k, v, mask)
    dq, dk, dv = orc.dense_backward(q, k, v, mask, out, lse)
    worst = 0.0
    for data, g in ((q, dq), (k, dk), (v, dv)):
        worst = max(worst, orc.max_rel_err(g, orc.fd_gradient(data, 1e-5, loss)))
    return worst


def test_gradcheck(orc):
    assert dense_gradcheck(orc, 1, 1, 8, 4, False, 21) < 1e-6
    assert dense_gradcheck(orc, 1, 2, 12, 4, True, 22) < 1e-5


@pytest.mark.slow
def test_gradcheck_large(orc):
    assert dense_gradcheck(orc, 2, 2, 64, 16, False, 23) < 1e-5
