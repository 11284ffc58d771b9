# SPDX-License-Identifier: Apache-2.0
"""A/B helper: median per-stage device time over N steps of the Wan2.1-1.3B layer."""
import statistics
import sys

import torch

sys.path.insert(0, ".")
import paper_2505_13389_b200 as vsa  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 20
L = vsa.TileLayout(21, 30, 52, pad=True)
op = vsa.VsaOp(L, 1, 12, 128, 78)
g = torch.Generator(device="cuda").manual_seed(1)
x = [torch.randn((1, 12, L.seq_len, 128), generator=g, device="cuda").bfloat16() for _ in range(6)]
for _ in range(3):
    op.forward(*x[:5])
    op.backward(x[5])
torch.cuda.synchronize()
acc = {}
for _ in range(n):
    op.trace = []
    op.forward(*x[:5])
    op.backward(x[5])
    torch.cuda.synchronize()
    tr = op.trace
    for (_, a), (name, b) in zip(tr[:-1], tr[1:]):
        acc.setdefault(name, []).append(a.elapsed_time(b))
    acc.setdefault("step", []).append(tr[0][1].elapsed_time(tr[-1][1]))
print({k: round(statistics.median(v), 4) for k, v in acc.items()})
