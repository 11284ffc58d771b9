# SPDX-License-Identifier: Apache-2.0
"""A/B: fine backward with the dS workspace (dK/dV stores dS, dQ = GEMM over it) vs
without (dK/dV without stores, dQ recomputes S and dP), Wan2.1-1.3B layer."""
import statistics
import sys

import torch

sys.path.insert(0, ".")
import paper_2505_13389_b200 as vsa  # noqa: E402

L = vsa.TileLayout(21, 30, 52, pad=True)
g = torch.Generator(device="cuda").manual_seed(1)
x = [torch.randn((1, 12, L.seq_len, 128), generator=g, device="cuda").bfloat16() for _ in range(6)]
for ws in (True, False, True, False):
    op = vsa.VsaOp(L, 1, 12, 128, 78, bwd_workspace=ws)
    for _ in range(3):
        op.forward(*x[:5])
        op.backward(x[5])
    ts = []
    for _ in range(20):
        op.forward(*x[:5])
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        op.backward(x[5])
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    print("workspace" if ws else "recompute", round(statistics.median(ts), 4), "ms backward")
