# SPDX-License-Identifier: Apache-2.0
"""Time VsaHostPipeline (the e2e leg of bench.py) over (chunks, slots) on the
Wan2.1-1.3B layer: pinned host inputs in, the six results out, every step."""
import itertools
import json
import sys

import torch

sys.path.insert(0, ".")
import paper_2505_13389_b200 as vsa  # noqa: E402

B, H, d, K = 1, 12, 128, 78
L = vsa.TileLayout(21, 30, 52, pad=True)
S = L.seq_len
hin = [torch.randn((B, H, S, d), dtype=torch.bfloat16).pin_memory() for _ in range(6)]
hout = [torch.empty((B, H, S, d), dtype=torch.bfloat16, pin_memory=True) for _ in range(6)]
res = []
for chunks, slots in itertools.product((12, 6, 4), (2, 3, 4)):
    pipe = vsa.VsaHostPipeline(L, B, H, d, K, chunks=chunks, slots=slots)
    pipe.run(hin, hout)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(5):
        pipe.run(hin, hout)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 5
    res.append({"chunks": chunks, "slots": slots, "ms": round(ms, 3)})
    print(json.dumps(res[-1]), flush=True)
    del pipe
    torch.cuda.empty_cache()
