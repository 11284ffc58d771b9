# SPDX-License-Identifier: Apache-2.0
"""Debug: per-pair event trace of one dK/dV CTA (current kernel's probes). Needs a
-DVSA_TRACE build (tools/build_variant.sh trace fine_bwd_sm100.cu -DVSA_TRACE, then
VSA_LIB_PATH=.../libvsa_trace.so). usage: trace_dkdv.py [wan13|dit]
Columns (cycles from the first event): producer issued the Q / dO granule of the pair,
the watcher saw it land, the compute warps got S (and dP), finished P / dS, and the
issuer passed the P / dS rendezvous of the merged d = 64 product."""
import ctypes as C
import sys

import torch

sys.path.insert(0, ".")
import paper_2505_13389_b200 as vsa  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "dit"
grid, B, H, d, k = {"wan13": ((21, 30, 52), 1, 12, 128, 78), "dit": ((16, 32, 32), 8, 16, 64, 32)}[cfg]
L = vsa.TileLayout(*grid, pad=True)
op = vsa.VsaOp(L, B, H, d, k)
g = torch.Generator(device="cuda").manual_seed(1)
x = [torch.randn((B, H, L.seq_len, d), generator=g, device="cuda").bfloat16() for _ in range(6)]
for _ in range(2):
    op.forward(*x[:5])
    op.backward(x[5])
torch.cuda.synchronize()
cap = 28 * 256
buf = torch.zeros(cap, dtype=torch.int64, device="cuda")
vsa.lib().vsa_debug_trace(C.c_void_p(buf.data_ptr()), cap, 40, 0)
op.forward(*x[:5])
op.backward(x[5])
torch.cuda.synchronize()
vsa.lib().vsa_debug_trace(None, 0, 0, 0)
b = buf.cpu().tolist()
ev = {(i // 256, i % 256): b[i] for i in range(cap) if b[i] != 0}
t0 = min(ev.values())
cols = [("ldQ", 2, 0), ("ldO", 2, 1), ("inQ", 3, 0), ("inO", 3, 1), ("gotS", 5, None), ("done", 7, None), ("iG", 4, None)]
print("  p " + "".join(f"{n:>8s}" for n, _, _ in cols))
for p in range(20, 60):
    row = [ev.get((code, 2 * p + k if k is not None else p)) for _, code, k in cols]
    print(f"{p:3d} " + "".join(f"{(r - t0) if r else -1:8d}" for r in row))
