# SPDX-License-Identifier: Apache-2.0
"""Debug: fine-forward stage time with and without the backward in the loop (32^3, H=16)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2505_13389_b200 as vsa  # noqa: E402

for d, k in ((64, 128), (128, 64)):
    L = vsa.TileLayout(32, 32, 32)
    xs = [torch.randn((1, 16, L.seq_len, d), device="cuda").bfloat16() for _ in range(6)]
    op = vsa.VsaOp(L, 1, 16, d, k)
    res = {}
    for mode in ("fwd", "fwdbwd", "fwd", "sleep", "fwd"):
        if mode == "sleep":
            import time
            time.sleep(3.0)
            continue
        for _ in range(3):
            op.forward(*xs[:5])
            if mode == "fwdbwd":
                op.backward(xs[5])
        torch.cuda.synchronize()
        op.timing(True)
        for _ in range(10):
            op.forward(*xs[:5])
            if mode == "fwdbwd":
                op.backward(xs[5])
        st = op.stage_ms()
        op.timing(False)
        torch.cuda.synchronize()
        print(d, k, mode, round(st["fine_fwd"], 4), round(st.get("fine_bwd", 0), 4), flush=True)
