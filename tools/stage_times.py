# SPDX-License-Identifier: Apache-2.0
"""A/B helper: mean per-stage device time over N back-to-back steps of the Wan2.1-1.3B layer
(native stage events, no host gaps)."""
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
op.timing(True)
for _ in range(n):
    op.forward(*x[:5])
    op.backward(x[5])
print({k: round(v, 4) if isinstance(v, float) else v for k, v in op.stage_ms().items()})
