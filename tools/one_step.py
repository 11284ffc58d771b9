# SPDX-License-Identifier: Apache-2.0
"""One VSA fwd+bwd step on the Wan2.1-1.3B layer (for ncu captures): 2 warm-up
steps, then one step between cudaProfilerStart/Stop markers."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2505_13389_b200 as vsa  # noqa: E402

L = vsa.TileLayout(21, 30, 52, pad=True)
op = vsa.VsaOp(L, 1, 12, 128, 78)
g = torch.Generator(device="cuda").manual_seed(1)
x = [torch.randn((1, 12, L.seq_len, 128), generator=g, device="cuda").bfloat16() for _ in range(6)]
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
