# SPDX-License-Identifier: Apache-2.0
"""Debug: pipeline event trace of one dK/dV CTA on the Wan2.1-1.3B shape.

Uses vsa_debug_trace (fixed-slot clock64 stores, no atomics) and prints the events
of the traced CTA in time order, relative to the first event."""
import ctypes as C
import sys

import torch

sys.path.insert(0, ".")
import paper_2505_13389_b200 as vsa  # noqa: E402

NAMES = {1: "prod_wait_empty", 2: "prod_issue", 3: "mma_SdP", 4: "mma_dVdK", 5: "cmp_wait_S", 6: "cmp_got_S",
         7: "cmp_done", 8: "cmp_tmem_ld_done", 9: "cmp_math_done", 10: "cmp_pd_empty_ok", 11: "cmp_bulk_read_ok",
         12: "cmp_bar_ok"}

L = vsa.TileLayout(21, 30, 52, pad=True)
op = vsa.VsaOp(L, 1, 12, 128, 78)
g = torch.Generator(device="cuda").manual_seed(1)
x = [torch.randn((1, 12, L.seq_len, 128), generator=g, device="cuda").bfloat16() for _ in range(6)]
for _ in range(2):
    op.forward(*x[:5])
    op.backward(x[5])
torch.cuda.synchronize()
cap = 16 * 256
buf = torch.zeros(cap, dtype=torch.int64, device="cuda")
for cta in (300, 301):
    buf.zero_()
    vsa.lib().vsa_debug_trace(C.c_void_p(buf.data_ptr()), cap, cta, 0)
    op.forward(*x[:5])
    op.backward(x[5])
    torch.cuda.synchronize()
    vsa.lib().vsa_debug_trace(None, 0, 0, 0)
    b = buf.cpu().tolist()
    ev = sorted((b[i], i // 256, i % 256) for i in range(cap) if b[i] != 0)
    t0 = ev[0][0]
    print(f"=== dkdv cta {cta}: {len(ev)} events")
    for c, code, idx in ev:
        print(f"{c - t0:8d} {NAMES.get(code, code):18s} {idx}")
