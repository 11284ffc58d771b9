# SPDX-License-Identifier: Apache-2.0
"""Oracle selection analytics pinned by the reference's
test_analysis.cpp:69-114 (full coverage, uniform attention, random-selection mean,
aggregation preserves row mass)."""
import numpy as np


def test_selection_accuracy_full_uniform_random(orc):
    L = orc.TileLayout(8, 8, 8, 2, 2, 2)  # 512 tokens, 64 cubes (test_analysis.cpp:70)
    k = 8
    rng = orc.Rng(91)
    uniform = np.full((1, 1, L.seq_len, L.num_cubes), 1.0 / L.num_cubes)
    assert orc.selection_accuracy(L, uniform, orc.all_cubes(1, 1, L.num_cubes))[0, 0] == 1.0
    sel = orc.random_selection(1, 1, L.num_cubes, k, rng)
    assert abs(orc.selection_accuracy(L, uniform, sel)[0, 0] - k / L.num_cubes) < 1e-12
    probs = np.empty((1, 1, L.seq_len, L.num_cubes))
    for i in range(L.seq_len):
        row = orc.randn_matrix(rng, 1, L.num_cubes, np.float64)[0]
        row = np.exp(row - row.max())
        probs[0, 0, i] = row / row.sum()
    mean = np.mean([orc.selection_accuracy(L, probs, orc.random_selection(1, 1, L.num_cubes, k, rng))[0, 0]
                    for _ in range(100)])
    assert abs(mean - k / L.num_cubes) < 0.01


def test_aggregate_preserves_row_mass(orc):
    L = orc.TileLayout(4, 4, 4, 2, 2, 2)
    rng = orc.Rng(92)
    probs = np.empty((1, 1, L.seq_len, L.seq_len))
    for i in range(L.seq_len):
        row = orc.randn_matrix(rng, 1, L.seq_len, np.float64)[0]
        row = np.exp(row - row.max())
        probs[0, 0, i] = row / row.sum()
    cube = orc.aggregate_probs_to_cubes(L, probs)
    assert cube.shape[-1] == L.num_cubes
    np.testing.assert_allclose(cube.sum(axis=-1), 1.0, rtol=0, atol=1e-12)


def test_dense_probs_row_stochastic(orc):
    rng = orc.Rng(93)
    q, k = (orc.randn(rng, 1, 2, 64, 16, np.float64) for _ in range(2))
    p = orc.dense_probs(q, k)
    np.testing.assert_allclose(p.sum(-1), 1.0, atol=1e-12)
    assert (p >= 0).all()
