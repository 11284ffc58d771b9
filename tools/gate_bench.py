# SPDX-License-Identifier: Apache-2.0
"""Gate projection on the tcgen05 GEMM at the Wan2.1-1.3B layer shape:
hidden [1, 1, 32760, 1536] bf16, Wg [1536, 3072], sigmoid + bias; fwd and bwd TFLOP/s."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2505_13389_b200 as vsa  # noqa: E402

L = vsa.TileLayout(21, 30, 52, pad=True)
B, H, d, md = 1, 12, 128, 1536
S = L.seq_len
hid = torch.randn(B, 1, S, md, device="cuda").bfloat16()
w = (torch.randn(md, 2 * H * d, device="cuda") / md ** 0.5).bfloat16()
bias = torch.randn(2 * H * d, device="cuda")
p = vsa.VsaParams(w, bias, 78, activation=1)
dgc = torch.randn(B, H, S, d, device="cuda").bfloat16()
dgf = torch.randn(B, H, S, d, device="cuda").bfloat16()
fl = 2 * B * S * md * 2 * H * d


def timeit(f, n=20):
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n):
        f()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n


gc, gf = vsa.gates_from_hidden(hid, p, H, d, layout=L)
tf = timeit(lambda: vsa.gates_from_hidden(hid, p, H, d, layout=L))
tb = timeit(lambda: vsa.gate_backward(hid, p, gc, gf, dgc, dgf, layout=L))
tt = timeit(lambda: hid[:, 0] @ w)
print({"gate_fwd_ms": round(tf, 4), "gate_fwd_tflops": round(fl / tf / 1e9, 1), "gate_bwd_ms": round(tb, 4),
       "gate_bwd_tflops": round(2 * fl / tb / 1e9, 1), "torch_matmul_fwd_ms": round(tt, 4),
       "torch_matmul_tflops": round(fl / tt / 1e9, 1)})
