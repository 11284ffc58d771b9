# SPDX-License-Identifier: Apache-2.0
"""Oracle pinning: the reference fine-stage tests (proj/tests/test_fine.cpp) and
the randomized oracle suite (proj/include/vsa/verify.hpp:43-134)."""
import numpy as np
import pytest


def test_full_selection_is_dense(orc):
    L = orc.TileLayout(4, 8, 4, 2, 2, 2)
    rng = orc.Rng(51)
    for dt, tol in ((np.float32, 1e-5), (np.float64, 1e-10)):
        q, k, v = (orc.randn(rng, 2, 2, L.seq_len, 16, dt) for _ in range(3))
        fo, _, _ = orc.fine_forward(L, q, k, v, orc.all_cubes(2, 2, L.num_cubes))
        do, _, _ = orc.dense_forward(q, k, v)
        assert np.abs(fo - do).max() < tol


def test_random_selection_is_masked_dense(orc):
    L = orc.TileLayout(4, 4, 8, 2, 2, 2)
    rng = orc.Rng(52)
    for _ in range(10):
        q, k, v = (orc.randn(rng, 2, 2, L.seq_len, 8) for _ in range(3))
        kk = rng.uniform_int(1, L.num_cubes)
        sel = orc.random_selection(2, 2, L.num_cubes, kk, rng)
        fo, _, _ = orc.fine_forward(L, q, k, v, sel)
        for b in range(2):
            mask = orc.selection_to_mask(L, sel, b)
            do, _, _ = orc.dense_forward(q[b:b + 1], k[b:b + 1], v[b:b + 1], mask)
            assert np.abs(do[0] - fo[b]).max() < 1e-10


def test_self_only_selection(orc):
    L = orc.TileLayout(4, 4, 4, 2, 2, 2)
    rng = orc.Rng(53)
    q, k, v = (orc.randn(rng, 1, 1, L.seq_len, 8) for _ in range(3))
    sel = np.arange(L.num_cubes, dtype=np.int32).reshape(1, 1, -1, 1)
    fo, _, _ = orc.fine_forward(L, q, k, v, sel)
    b = L.cube_size
    for c in range(L.num_cubes):
        s = slice(c * b, (c + 1) * b)
        do, _, _ = orc.dense_forward(q[:, :, s], k[:, :, s], v[:, :, s])
        assert np.abs(do[0, 0] - fo[0, 0, s]).max() < 1e-12


def test_invalid_selections(orc):
    L = orc.TileLayout(4, 4, 4, 2, 2, 2)
    rng = orc.Rng(54)
    q, k, v = (orc.randn(rng, 1, 1, L.seq_len, 4) for _ in range(3))
    nc = L.num_cubes
    for bad in (np.tile(np.array([3, 1], np.int32), (1, 1, nc, 1)), np.tile(np.array([1, 1], np.int32), (1, 1, nc, 1)),
                np.full((1, 1, nc, 1), nc, np.int32)):
        with pytest.raises(ValueError):
            orc.fine_forward(L, q, k, v, bad)


def test_backward_full_is_dense(orc):
    L = orc.TileLayout(4, 4, 4, 2, 2, 2)
    rng = orc.Rng(55)
    for B, dt, tol in ((2, np.float64, 1e-10), (1, np.float32, 1e-5)):
        q, k, v, dout = (orc.randn(rng, B, 2, L.seq_len, 8, dt) for _ in range(4))
        sel = orc.all_cubes(B, 2, L.num_cubes)
        _, _, flse = orc.fine_forward(L, q, k, v, sel)
        fg = orc.fine_backward(L, q, k, v, sel, dout, flse)
        _, _, dlse = orc.dense_forward(q, k, v)
        dg = orc.dense_backward(q, k, v, None, dout, dlse)
        for a, b in zip(fg, dg):
            assert np.abs(a - b).max() < tol


def test_unselected_key_cubes_zero_grad(orc):
    L = orc.TileLayout(4, 4, 4, 2, 2, 2)
    rng = orc.Rng(56)
    q, k, v, dout = (orc.randn(rng, 1, 1, L.seq_len, 8) for _ in range(4))
    sel = np.tile(np.array([0, 1], np.int32), (1, 1, L.num_cubes, 1))
    _, _, lse = orc.fine_forward(L, q, k, v, sel)
    _, dk, dv = orc.fine_backward(L, q, k, v, sel, dout, lse)
    assert (dk[0, 0, 2 * L.cube_size:] == 0).all() and (dv[0, 0, 2 * L.cube_size:] == 0).all()


def test_sparse_gradcheck(orc):
    L = orc.TileLayout(4, 4, 4, 2, 2, 2)
    rng = orc.Rng(57)
    q, k, v = (orc.randn(rng, 1, 2, L.seq_len, 4) for _ in range(3))
    sel = orc.random_selection(1, 2, L.num_cubes, 3, rng)
    loss = lambda: 0.5 * float((orc.fine_forward(L, q, k, v, sel)[0] ** 2).sum())
    out, _, lse = orc.fine_forward(L, q, k, v, sel)
    g = orc.fine_backward(L, q, k, v, sel, out.copy(), lse)
    worst = max(orc.max_rel_err(gi, orc.fd_gradient(x, 1e-5, loss)) for x, gi in zip((q, k, v), g))
    assert worst < 1e-6


def test_tile_visit_order_invariance(orc):
    L = orc.TileLayout(4, 4, 4, 2, 2, 2)
    rng = orc.Rng(58)
    b, nc, D = L.cube_size, L.num_cubes, 8
    perm = np.arange(nc, dtype=np.int64)
    rng.shuffle(perm)
    inv = np.empty(nc, np.int64)
    inv[perm] = np.arange(nc)
    for dt, tol in ((np.float64, 1e-12), (np.float32, 1e-5)):
        drng = orc.Rng(59)
        q, k, v = (orc.randn(drng, 1, 1, L.seq_len, D, dt) for _ in range(3))
        sel = orc.random_selection(1, 1, nc, 3, drng)
        idx = (perm[:, None] * b + np.arange(b)[None]).reshape(-1)
        qp, kp, vp = q[:, :, idx], k[:, :, idx], v[:, :, idx]
        selp = np.sort(inv[sel[0, 0][perm]], axis=1).astype(np.int32)[None, None]
        base, _, _ = orc.fine_forward(L, q, k, v, sel)
        sh, _, _ = orc.fine_forward(L, qp, kp, vp, selp)
        assert np.abs(sh[0, 0] - base[0, 0, idx]).max() < tol


def test_mac_count_density(orc):
    """test_fine.cpp:251-270 — executed work equals selection density: the fine
    stage touches B*H*nc*k tiles of 2*b*b*d MACs, dense 2*L*L*d per (b,h)."""
    L = orc.TileLayout(4, 4, 8, 2, 2, 2)
    B, H, D, k = 2, 2, 8, 2
    fine_macs = B * H * L.num_cubes * k * 2 * L.cube_size ** 2 * D
    dense_macs = B * H * 2 * L.seq_len ** 2 * D
    assert fine_macs * 8 == dense_macs


def random_layout(orc, rng, max_seq):
    """verify.hpp:43-54."""
    def pick(xs):
        return xs[rng.uniform_size(0, len(xs) - 1)]
    while True:
        ct, ch, cw = pick([1, 2, 4]), pick([1, 2, 4]), pick([1, 2, 4])
        nt, nh, nw = pick([1, 2, 3, 4]), pick([1, 2, 3, 4]), pick([1, 2, 4, 8])
        L = orc.TileLayout(ct * nt, ch * nh, cw * nw, ct, ch, cw)
        if L.seq_len <= max_seq and L.num_cubes >= 2:
            return L


def run_oracle_suite(orc, cases=100, seed=2024, double=False, inject_fault=False, max_seq=1024):
    """run_oracle_suite (verify.hpp:99-134): worst (full, sparse) errors."""
    rng = orc.Rng(seed)
    dt = np.float64 if double else np.float32
    worst = [0.0, 0.0]
    for c in range(cases):
        L = random_layout(orc, rng, max_seq)
        B = rng.uniform_int(1, 2)
        H = rng.uniform_int(1, 4)
        D = [8, 16, 32][rng.uniform_int32(0, 2)]
        kk = rng.uniform_int(1, L.num_cubes)
        full = c % 2 == 0
        q, k, v = (orc.randn(rng, B, H, L.seq_len, D, dt) for _ in range(3))
        sel = orc.all_cubes(B, H, L.num_cubes) if full else orc.random_selection(B, H, L.num_cubes, kk, rng)
        fo, _, _ = orc.fine_forward(L, q, k, v, sel)
        if inject_fault and c == 1 and not full:
            sel = sel.copy()
            sel[0, 0, 0, 0] = (sel[0, 0, 0, 0] + 1) % L.num_cubes
            sel[0, 0, 0].sort()
        for b in range(B):
            mask = None if full else orc.selection_to_mask(L, sel, b)
            do, _, _ = orc.dense_forward(q[b:b + 1], k[b:b + 1], v[b:b + 1], mask)
            worst[0 if full else 1] = max(worst[0 if full else 1], float(np.abs(do[0] - fo[b]).max()))
    return worst


def test_oracle_suite_f32(orc):
    full, sparse = run_oracle_suite(orc, cases=40)
    assert full < 1e-5 and sparse < 1e-5


def test_oracle_suite_fault_injection_fails(orc):
    full, sparse = run_oracle_suite(orc, cases=4, double=True, inject_fault=True)
    assert sparse >= 1e-10  # the corrupted selection must be caught


@pytest.mark.slow
def test_oracle_suite_full(orc):
    for double, tol in ((False, 1e-5), (True, 1e-10)):
        full, sparse = run_oracle_suite(orc, cases=100, double=double)
        assert full < tol and sparse < tol
