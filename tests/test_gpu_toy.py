# SPDX-License-Identifier: Apache-2.0
"""GPU-driven toy trainer — the reference's test_toy.cpp cases on
the B200 operator: generated targets follow the closed form, zero learning rate keeps
the loss constant, dense-equivalent mode has recall 1 and a decreasing smoothed loss,
seeded runs are bitwise reproducible, the schedule anneals k, and the learned
selection finds the planted cubes better than a fixed random one."""
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def vsa():
    import paper_2505_13389_b200 as v

    v.lib()
    return v


def small_task(vsa, seed=5):
    from paper_2505_13389_b200.toy import PlantedTask

    # test_toy.cpp:11-18: TileLayout(4,4,4, 2,2,2), 2 planted cubes, 2 heads, head_dim 4
    return PlantedTask(vsa.TileLayout(4, 4, 4, 2, 2, 2), planted_count=2, heads=2, head_dim=4, seed=seed)


def test_generated_targets_closed_form(vsa):
    from paper_2505_13389_b200.toy import generate_batch

    for noise in (0.0, 0.5):
        task = small_task(vsa)
        task.noise_scale = noise
        b = generate_batch(task, 3, 17, dtype=torch.float64)
        cube = task.layout.cube_size
        for i in range(3):
            assert len(b.planted[i]) == task.planted_count
            for h in range(task.heads):
                vv = b.v[i, h]
                mean = sum(vv[c * cube:(c + 1) * cube].sum(0) for c in b.planted[i]) / (len(b.planted[i]) * cube)
                assert (b.target[i, h] - vv - mean).abs().max() < 1e-12


def test_zero_lr_constant_loss(vsa):
    from paper_2505_13389_b200.toy import OptimizerSettings, ToyTrainConfig, train_toy

    rep = train_toy(small_task(vsa), ToyTrainConfig(batch_size=2, steps=5, top_k=4,
                                                    optimizer=OptimizerSettings(lr=0.0)))
    assert len(rep.steps) == 5
    assert all(s.loss == rep.steps[0].loss for s in rep.steps)


def test_dense_equivalent_recall_one_and_learning(vsa):
    from paper_2505_13389_b200.toy import ToyTrainConfig, train_toy

    task = small_task(vsa)
    rep = train_toy(task, ToyTrainConfig(batch_size=2, steps=240, top_k=task.layout.num_cubes))
    assert not rep.diverged
    assert all(s.recall == 1.0 for s in rep.steps)
    mean = lambda a, b: sum(s.loss for s in rep.steps[a:b]) / (b - a)
    assert mean(len(rep.steps) - 40, len(rep.steps)) < mean(0, 40)


def test_seeded_runs_bitwise_reproducible(vsa):
    from paper_2505_13389_b200.toy import ToyTrainConfig, train_toy

    cfg = ToyTrainConfig(batch_size=2, steps=20, top_k=4)
    a, b = train_toy(small_task(vsa), cfg), train_toy(small_task(vsa), cfg)
    assert [(s.loss, s.recall) for s in a.steps] == [(s.loss, s.recall) for s in b.steps]
    assert a.snapshot_id == b.snapshot_id


def test_schedule_anneals_k(vsa):
    from paper_2505_13389_b200.toy import SparsitySchedule, ToyTrainConfig, train_toy

    task = small_task(vsa)
    nc = task.layout.num_cubes
    rep = train_toy(task, ToyTrainConfig(batch_size=2, steps=60, schedule=SparsitySchedule(nc, 2, 10, 10, 2)))
    assert rep.steps[0].k == nc and rep.steps[-1].k == 2
    assert all(b.k <= a.k for a, b in zip(rep.steps, rep.steps[1:]))


def test_learned_selection_beats_fixed_random(vsa):
    from paper_2505_13389_b200.toy import OptimizerSettings, ToyTrainConfig, train_toy

    task = small_task(vsa)
    cfg = ToyTrainConfig(batch_size=2, steps=300, top_k=2, optimizer=OptimizerSettings(lr=3e-3))
    learned = train_toy(task, cfg)
    cfg.policy = "fixed_random"
    fixed = train_toy(task, cfg)
    assert not learned.diverged and not fixed.diverged
    assert learned.final_recall() > fixed.final_recall()
    assert learned.final_loss() < fixed.final_loss()


def test_acceptance_7_default_task(vsa):
    """SPEC acceptance 7: the default planted-cube task (vsa_cli.cpp:515-523
    train-toy defaults) reaches recall >= 0.8 and final MSE <= 1.10x the dense control's
    within 5000 steps, and the learned selection beats the fixed-random control."""
    from paper_2505_13389_b200.toy import PlantedTask, ToyTrainConfig, train_toy

    task = PlantedTask(vsa.TileLayout(8, 8, 8, 2, 2, 2), planted_count=4, heads=2, head_dim=8, seed=0)
    run = lambda k, policy: train_toy(task, ToyTrainConfig(batch_size=4, steps=5000, top_k=k, policy=policy, seed=1))
    learned, dense, fixed = run(8, "learned"), run(task.layout.num_cubes, "learned"), run(8, "fixed_random")
    assert not (learned.diverged or dense.diverged or fixed.diverged)
    assert learned.final_recall() >= 0.8
    assert learned.final_loss() <= 1.10 * dense.final_loss()
    assert learned.final_recall() > fixed.final_recall()


def test_fixed_pattern_control_runs(vsa):
    from paper_2505_13389_b200.toy import PatternSpec, ToyTrainConfig, train_toy

    task = small_task(vsa)
    rep = train_toy(task, ToyTrainConfig(batch_size=2, steps=6, top_k=2, policy="fixed_pattern",
                                         pattern=PatternSpec()))  # spatial-temporal, alternating phases
    assert len(rep.steps) == 6 and not rep.diverged
    assert all(0.0 <= s.recall <= 1.0 for s in rep.steps)
