# SPDX-License-Identifier: Apache-2.0
"""Host-side pieces of the toy trainer, no GPU: the sparsity
schedule (test_analysis.cpp:9-41) and the cube-level fixed-pattern selections
(test_analysis.cpp:165-184)."""
import numpy as np
import pytest

from paper_2505_13389_b200 import TileLayout
from paper_2505_13389_b200.toy import (COMPRESS_KV, SPATIAL, SPATIAL_TEMPORAL, STRIDED_WINDOW, TEMPORAL,
                                       PatternSpec, SparsitySchedule, fixed_pattern_selection)


def test_schedule_step_decay_shape():
    s = SparsitySchedule()  # 256 -> 32, warmup 50, -10 every 50
    assert [s.k_at(x) for x in (0, 49, 50, 100, 149, 1000000)] == [256, 256, 256, 246, 246, 32]
    flat = SparsitySchedule(64, 64)
    assert all(flat.k_at(x) == 64 for x in (0, 10, 500))


def test_schedule_monotone_reaches_target():
    s = SparsitySchedule(200, 17, 30, 20, 7)
    ks = [s.k_at(x) for x in range(2000)]
    assert all(b <= a for a, b in zip(ks, ks[1:])) and min(ks) == 17 and all(k >= 17 for k in ks)
    with pytest.raises(ValueError):
        s.k_at(-1)
    with pytest.raises(ValueError):
        SparsitySchedule(4, 8).k_at(0)


def test_pattern_selections_match_phase_definitions():
    L = TileLayout(4, 8, 8, 2, 2, 2)  # cubes 2 x 4 x 4
    sp = fixed_pattern_selection(L, PatternSpec(SPATIAL_TEMPORAL, SPATIAL, 8, 2))
    assert sp.shape == (L.num_cubes, L.cubes_h * L.cubes_w)
    te = fixed_pattern_selection(L, PatternSpec(SPATIAL_TEMPORAL, TEMPORAL, 8, 2))
    assert te.shape == (L.num_cubes, L.cubes_t)
    co = fixed_pattern_selection(L, PatternSpec(COMPRESS_KV, SPATIAL, 8, 2))
    assert co.shape == (L.num_cubes, L.num_cubes)
    for sel in (sp, te, co):  # BlockSelection::validate: ascending, unique, in range
        assert (np.diff(sel, axis=1) > 0).all() and sel.min() >= 0 and sel.max() < L.num_cubes
    hw = L.cubes_h * L.cubes_w
    for qc in range(L.num_cubes):
        assert set(sp[qc]) == {c for c in range(L.num_cubes) if c // hw == qc // hw}
        assert set(te[qc]) == {c for c in range(L.num_cubes) if c % hw == qc % hw}
    with pytest.raises(ValueError):  # cube-misaligned window
        fixed_pattern_selection(L, PatternSpec(STRIDED_WINDOW, SPATIAL, 8, 3))


def test_strided_window_covering_grid_is_full():
    L = TileLayout(4, 4, 4, 2, 2, 2)
    full = fixed_pattern_selection(L, PatternSpec(STRIDED_WINDOW, SPATIAL, 8, 4))
    assert full.shape == (L.num_cubes, L.num_cubes)
    w2 = fixed_pattern_selection(L, PatternSpec(STRIDED_WINDOW, SPATIAL, 8, 2))
    assert w2.shape == (L.num_cubes, L.cubes_h * L.cubes_w)  # window_t = cube_t: one cube layer per window


def test_flop_accounting_exact_8x():
    """test_analysis.cpp:43-66 / SPEC acceptance 4."""
    from paper_2505_13389_b200.analysis import FULL, VSA, FlopsConfig, compute_flops, sparsity_density

    cfg = FlopsConfig(n_params=1e6, n_tokens=1e3, seq_len=16384, n_heads=12, head_dim=64, n_layers=12,
                      block_size=64, density=sparsity_density(32, 64, 16384))
    assert cfg.density == 0.125
    full, sparse = compute_flops(cfg, FULL), compute_flops(cfg, VSA)
    assert full.model_flops == 6e9 and sparse.model_flops == 6e9
    assert full.attention_flops / sparse.attention_flops == 8.0
    assert sparse.attention_flops / full.attention_flops == cfg.density
    assert sparse.coarse_flops == full.attention_flops / (64.0 * 64.0)
    assert sparse.total == sparse.model_flops + sparse.attention_flops + sparse.coarse_flops
    js = sparse.to_json()
    assert '"model_flops"' in js and '"density": 0.125' in js
    with pytest.raises(ValueError):
        compute_flops(FlopsConfig(), VSA)
