# SPDX-License-Identifier: Apache-2.0
"""bench.py under torchrun with several ranks on the one GPU of the sandbox (gloo for the
barrier / max-over-ranks / lse-delta all-reduce; NCCL needs one GPU per rank): the whole
unit partition (2 ranks over 2 heads) and the head sub-split (3 ranks over 2 heads) run to
completion and rank 0 prints one contract line with strong scaling."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world", [2, 3])
def test_bench_torchrun_ranks(world):
    env = dict(os.environ, VSA_BENCH_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), os.path.join(ROOT, "bench.py"),
           "--gpus", str(world), "--config", "tiny", "--steps", "3", "--warmup", "3", "--no-dense", "--no-cpu"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT, env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == world and d["scaling"] == "strong" and d["value"] > 0
    assert ("cube split" in d["config"]["parallelism"]) == (world == 3)
