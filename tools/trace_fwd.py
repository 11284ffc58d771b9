# SPDX-License-Identifier: Apache-2.0
"""Debug: pipeline event trace of one persistent fine-forward CTA (Wan2.1-1.3B shape)."""
import ctypes as C
import sys

import torch

sys.path.insert(0, ".")
import paper_2505_13389_b200 as vsa  # noqa: E402

L = vsa.TileLayout(21, 30, 52, pad=True)
op = vsa.VsaOp(L, 1, 12, 128, 78)
g = torch.Generator(device="cuda").manual_seed(1)
x = [torch.randn((1, 12, L.seq_len, 128), generator=g, device="cuda").bfloat16() for _ in range(5)]
for _ in range(2):
    op.forward(*x)
torch.cuda.synchronize()
cap = 16 * 256
buf = torch.zeros(cap, dtype=torch.int64, device="cuda")
vsa.lib().vsa_debug_trace(C.c_void_p(buf.data_ptr()), cap, 5, 0)
op.forward(*x)
torch.cuda.synchronize()
vsa.lib().vsa_debug_trace(None, 0, 0, 0)
b = buf.cpu().tolist()
ev = {(i // 256, i % 256): b[i] for i in range(cap) if b[i] != 0}
t0 = min(ev.values())
cols = [("ldK", 1, lambda p: 2 * p), ("Kin", 2, lambda p: 2 * p), ("ldV", 1, lambda p: 2 * p + 1),
        ("Vin", 2, lambda p: 2 * p + 1),  ("gotS", 7, None), ("Prdy", 8, None),
        ("O0", 5, None), ("ldS", 9, None), ("vote", 10, None), ("Sfree", 11, None),
        ("Psts", 14, None), ("fence", 15, None)]
print("  gp" + "".join(f"{n:>8s}" for n, _, _ in cols))
for p in range(0, 120):
    row = [ev.get((code, f(p) if f else p)) for _, code, f in cols]
    if all(r is None for r in row):
        break
    if 8 <= p < 24:
        print(f"{p:4d}" + "".join(f"{(r - t0) if r else -1:8d}" for r in row))
