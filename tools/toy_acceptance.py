# SPDX-License-Identifier: Apache-2.0
"""SPEC acceptance 7 on the GPU op: the default planted-cube task (the reference CLI's
train-toy defaults, vsa_cli.cpp:515-523) trained for 5000 steps with the learned
selection, the dense control (k = num_cubes) and the fixed-random control."""
import json
import sys
import time

sys.path.insert(0, ".")
import paper_2505_13389_b200 as vsa  # noqa: E402
from paper_2505_13389_b200.toy import PlantedTask, ToyTrainConfig, train_toy  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 5000
task = PlantedTask(vsa.TileLayout(8, 8, 8, 2, 2, 2), planted_count=4, heads=2, head_dim=8, seed=0)
res = {}
for name, k, policy in (("learned", 8, "learned"), ("dense", task.layout.num_cubes, "learned"),
                        ("fixed_random", 8, "fixed_random")):
    t0 = time.time()
    rep = train_toy(task, ToyTrainConfig(batch_size=4, steps=steps, top_k=k, policy=policy, seed=1))
    res[name] = {"final_loss": rep.final_loss(), "final_recall": rep.final_recall(), "diverged": rep.diverged,
                 "seconds": round(time.time() - t0, 1), "snapshot": rep.snapshot_id}
    print(name, res[name], flush=True)
ok = (res["learned"]["final_recall"] >= 0.8 and res["learned"]["final_loss"] <= 1.10 * res["dense"]["final_loss"]
      and res["learned"]["final_recall"] > res["fixed_random"]["final_recall"])
print(json.dumps({"steps": steps, "acceptance_7": ok, **res}))
