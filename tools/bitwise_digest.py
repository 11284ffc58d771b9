# SPDX-License-Identifier: Apache-2.0
"""A/B helper: digest of every forward / backward output of VsaOp on seeded inputs, for
checking that a kernel variant (VSA_LIB_PATH) is bitwise identical to the default library.
usage: bitwise_digest.py  (prints one line per config: out / dq / dk / dv / dgc / dgf digests)"""
import hashlib
import sys

import torch

sys.path.insert(0, ".")
import paper_2505_13389_b200 as vsa  # noqa: E402


def digest(t):
    return hashlib.sha1(t.contiguous().view(torch.uint8).cpu().numpy().tobytes()).hexdigest()[:10]


for name, grid, B, H, d, k, pad, adapt in (("wan13-2h", (21, 30, 52), 1, 2, 128, 78, True, False),
                                           ("dit-2u", (16, 32, 32), 1, 2, 64, 32, True, False),
                                           ("odd-pad", (5, 7, 9), 1, 3, 64, 3, True, False),
                                           ("adapt", (8, 8, 8), 1, 2, 128, 2, False, True)):
    L = vsa.TileLayout(*grid, pad=pad)
    op = vsa.VsaOp(L, B, H, d, k, adaptation=adapt)
    g = torch.Generator(device="cuda").manual_seed(7)
    x = [torch.randn((B, H, L.seq_len, d), generator=g, device="cuda").bfloat16() for _ in range(6)]
    out = op.forward(*x[:5])
    grads = op.backward(x[5])
    torch.cuda.synchronize()
    print(name, digest(out), *[digest(t) for t in grads])
