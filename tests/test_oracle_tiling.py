# SPDX-License-Identifier: Apache-2.0
"""Oracle pinning: the reference tiling tests (proj/tests/test_tiling.cpp), same seeds."""
import numpy as np
import pytest


def enumerate_tile_order(t, h, w, ct, ch, cw):
    """Independent oracle (test_tiling.cpp:15-26): enumerate cubes, then tokens."""
    out = np.empty(t * h * w, np.int64)
    pos = 0
    for bt in range(0, t, ct):
        for bh in range(0, h, ch):
            for bw in range(0, w, cw):
                for it in range(bt, bt + ct):
                    for ih in range(bh, bh + ch):
                        for iw in range(bw, bw + cw):
                            out[(it * h + ih) * w + iw] = pos
                            pos += 1
    return out


def random_small_layout(orc, rng):
    """test_tiling.cpp:28-36."""
    def pick(xs):
        return xs[rng.uniform_size(0, len(xs) - 1)]
    ct, ch, cw = pick([1, 2, 3]), pick([1, 2, 3]), pick([1, 2, 4])
    nt, nh, nw = pick([1, 2, 3]), pick([1, 2, 4]), pick([1, 2, 3])
    return orc.TileLayout(ct * nt, ch * nh, cw * nw, ct, ch, cw)


def test_flatten_index_444_222(orc):
    L = orc.TileLayout(4, 4, 4, 2, 2, 2)
    assert (L.cube_size, L.seq_len, L.num_cubes) == (8, 64, 8)
    assert orc.flatten_index(L, 0, 0, 0) == 0
    assert orc.flatten_index(L, 1, 1, 1) == 7
    assert orc.flatten_index(L, 2, 0, 0) == 32
    ref = enumerate_tile_order(4, 4, 4, 2, 2, 2)
    for t in range(4):
        for h in range(4):
            for w in range(4):
                assert orc.flatten_index(L, t, h, w) == ref[(t * 4 + h) * 4 + w]


def test_flatten_index_varied_layouts(orc):
    for args in [(6, 4, 4, 3, 2, 2), (2, 6, 8, 1, 3, 4), (4, 4, 4, 4, 4, 4), (1, 1, 8, 1, 1, 2), (5, 2, 2, 5, 1, 2)]:
        L = orc.TileLayout(*args)
        np.testing.assert_array_equal(L.tile_of_raster(), enumerate_tile_order(*args))


def test_bijection(orc):
    rng = orc.Rng(11)
    for _ in range(20):
        L = random_small_layout(orc, rng)
        t2r = L.tile_of_raster()
        assert t2r.min() >= 0 and t2r.max() < L.seq_len
        assert len(set(t2r.tolist())) == L.seq_len


def test_contiguous_cube_spans(orc):
    rng = orc.Rng(12)
    for _ in range(10):
        L = random_small_layout(orc, rng)
        t2r = L.tile_of_raster()
        spans = [set() for _ in range(L.num_cubes)]
        for n in t2r:
            spans[n // L.cube_size].add(int(n))
        for c, s in enumerate(spans):
            assert len(s) == L.cube_size
            assert min(s) == c * L.cube_size and max(s) == (c + 1) * L.cube_size - 1


def test_tile_untile_identity(orc):
    rng = orc.Rng(13)
    for _ in range(50):
        L = random_small_layout(orc, rng)
        x = orc.randn(rng, 2, 2, L.seq_len, 3)
        np.testing.assert_array_equal(orc.untile(L, orc.tile(L, x)), x)


def test_tile_constant(orc):
    L = orc.TileLayout(4, 4, 4, 2, 2, 2)
    x = np.full((1, 1, L.seq_len, 2), 3.25, np.float32)
    np.testing.assert_array_equal(orc.tile(L, x), x)


def test_tile_moves_111_to_7(orc):
    L = orc.TileLayout(4, 4, 4, 2, 2, 2)
    x = np.arange(L.seq_len, dtype=np.float64).reshape(1, 1, -1, 1)
    assert orc.tile(L, x)[0, 0, 7, 0] == orc.raster_index(L, 1, 1, 1)


def test_contract_violations(orc):
    with pytest.raises(ValueError):
        orc.TileLayout(5, 4, 4, 2, 2, 2)
    with pytest.raises(ValueError):
        orc.TileLayout(4, 4, 4, 0, 2, 2)
    L = orc.TileLayout(4, 4, 4, 2, 2, 2)
    with pytest.raises(ValueError):
        orc.flatten_index(L, 4, 0, 0)
    with pytest.raises(ValueError):
        orc.flatten_index(L, 0, -1, 0)
    wrong = np.zeros((1, 1, L.seq_len + 1, 2))
    with pytest.raises(ValueError):
        orc.tile(L, wrong)
    with pytest.raises(ValueError):
        orc.untile(L, wrong)
