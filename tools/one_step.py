# SPDX-License-Identifier: Apache-2.0
"""One VSA fwd+bwd step on the Wan2.1-1.3B layer or the DiT batch (argv[1]: wan13 | dit; for ncu captures): 2 warm-up
steps, then one step between cudaProfilerStart/Stop markers."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2505_13389_b200 as vsa  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "wan13"
grid, B, H, d, k = {"wan13": ((21, 30, 52), 1, 12, 128, 78), "dit": ((16, 32, 32), 8, 16, 64, 32)}[cfg]
L = vsa.TileLayout(*grid, pad=True)
op = vsa.VsaOp(L, B, H, d, k)
g = torch.Generator(device="cuda").manual_seed(1)
x = [torch.randn((B, H, L.seq_len, d), generator=g, device="cuda").bfloat16() for _ in range(6)]
for _ in range(2):
    op.forward(*x[:5])
    op.backward(x[5])
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
op.forward(*x[:5])
op.backward(x[5])
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("step done")
