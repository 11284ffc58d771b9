# SPDX-License-Identifier: Apache-2.0
"""Debug: pipeline event trace of one persistent fine-forward CTA. Needs the library built
with -DVSA_TRACE (tools/build_variant.sh trace fine_fwd_sm100.cu -DVSA_TRACE, then
VSA_LIB_PATH=.../libvsa_trace.so). usage: trace_fwd.py [wan13|dit]"""
import ctypes as C
import sys

import torch

sys.path.insert(0, ".")
import paper_2505_13389_b200 as vsa  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "wan13"
grid, B, H, d, k = {"wan13": ((21, 30, 52), 1, 12, 128, 78), "dit": ((16, 32, 32), 8, 16, 64, 32)}[cfg]
L = vsa.TileLayout(*grid, pad=True)
op = vsa.VsaOp(L, B, H, d, k)
g = torch.Generator(device="cuda").manual_seed(1)
x = [torch.randn((B, H, L.seq_len, d), generator=g, device="cuda").bfloat16() for _ in range(5)]
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
