# SPDX-License-Identifier: Apache-2.0
"""Debug: pipeline event trace of one dK/dV CTA on the Wan2.1-1.3B shape. Needs the
library built with trace probes: make -C paper_2505_13389_b200/csrc -B EXTRA=-DVSA_TRACE

Uses vsa_debug_trace (fixed-slot clock64 stores, no atomics) and prints the events
of the traced CTA in time order, relative to the first event."""
import ctypes as C
import sys

import torch

sys.path.insert(0, ".")
import paper_2505_13389_b200 as vsa  # noqa: E402

NAMES = {2: "prod_issue(item)", 3: "mma_S", 13: "mma_dP", 4: "mma_dV", 12: "mma_dK", 5: "cmp_got_S",
         6: "cmp_P_ready", 8: "cmp_P_buf_free", 9: "cmp_got_dP", 10: "cmp_dS_ready", 11: "cmp_dS_buf_free",
         7: "cmp_done"}

L = vsa.TileLayout(21, 30, 52, pad=True)
op = vsa.VsaOp(L, 1, 12, 128, 78)
g = torch.Generator(device="cuda").manual_seed(1)
x = [torch.randn((1, 12, L.seq_len, 128), generator=g, device="cuda").bfloat16() for _ in range(6)]
for _ in range(2):
    op.forward(*x[:5])
    op.backward(x[5])
torch.cuda.synchronize()
cap = 28 * 256
buf = torch.zeros(cap, dtype=torch.int64, device="cuda")
for cta in (300, 301):
    buf.zero_()
    vsa.lib().vsa_debug_trace(C.c_void_p(buf.data_ptr()), cap, cta, 0)
    op.forward(*x[:5])
    op.backward(x[5])
    torch.cuda.synchronize()
    vsa.lib().vsa_debug_trace(None, 0, 0, 0)
    b = buf.cpu().tolist()
    ev = {(i // 256, i % 256): b[i] for i in range(cap) if b[i] != 0}
    t0 = ev.get((24, 0), min(ev.values()))
    cols = [("S.w", 12, None), ("S.go", 13, None), ("S.end", 14, None), ("dV.w", 17, None), ("dV.go", 18, None),
            ("dV.end", 19, None), ("dP.w", 20, None), ("dP.go", 21, None), ("dP.end", 22, None), ("dK.w", 25, None),
            ("dK.go", 26, None), ("dK.end", 27, None), ("Prdy", 6, None), ("done", 7, None)]
    print("  p " + "".join(f"{n:>8s}" for n, _, _ in cols))
    names = {0: "entry", 4: "after TMEM alloc", 1: "epilogue start", 2: "epilogue rows written", 3: "exit"}
    print("  CTA:", {names[i]: ev[(24, i)] - t0 for i in names if (24, i) in ev}, "npairs ~", max([p for (c, p) in ev if c == 1] or [-1]) + 1)
    for p in range(2, 10):
        a, b, c = ev.get((14, p)), ev.get((3, p)), ev.get((16, p))
        if None not in (a, b, c):
            print(f"S({p}): issue {b - a} cycles, complete {c - a} cycles after issue start")
    for p in range(64):
        row = [ev.get((code, f(p) if f else p)) for _, code, f in cols]
        if all(r is None for r in row):
            break
        print(f"{p:3d} " + "".join(f"{(r - t0) if r else -1:8d}" for r in row))
