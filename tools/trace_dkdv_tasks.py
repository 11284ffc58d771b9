# SPDX-License-Identifier: Apache-2.0
"""Debug: per-task timeline of one persistent dK/dV CTA (library built with -DVSA_TRACE):
issue start of each task, issue end (acc_full commit), epilogue done; pairs per task."""
import ctypes as C
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
cap = 28 * 256
buf = torch.zeros(cap, dtype=torch.int64, device="cuda")
cta = int(sys.argv[1]) if len(sys.argv) > 1 else 7
vsa.lib().vsa_debug_trace(C.c_void_p(buf.data_ptr()), cap, cta, 0)
op.forward(*x[:5])
op.backward(x[5])
torch.cuda.synchronize()
vsa.lib().vsa_debug_trace(None, 0, 0, 0)
b = buf.cpu().tolist()
ev = {(i // 256, i % 256): b[i] for i in range(cap) if b[i] != 0}
t0 = ev[(24, 0)]
print("exit", ev.get((24, 3), 0) - t0)
prev = None
tot_pairs = 0
for j in range(64):
    s, e, d = ev.get((12, j)), ev.get((13, j)), ev.get((14, j))
    if s is None and e is None and d is None:
        continue
    f = lambda v: (v - t0) if v else -1
    print(f"task {j:3d}: issue start {f(s):8d}  issue end {f(e):8d}  epi done {f(d):8d}  span {((e - s) if s and e else -1):7d}")
