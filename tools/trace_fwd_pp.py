# SPDX-License-Identifier: Apache-2.0
"""Debug: pipeline event trace of one persistent CTA of the d = 64 ping-pong forward
(fine_fwd_pp_sm100.cu). Needs the library built with -DVSA_TRACE:
    tools/build_variant.sh trace fine_fwd_pp_sm100.cu -DVSA_TRACE
    VSA_LIB_PATH=paper_2505_13389_b200/_lib/variants/libvsa_trace.so python tools/trace_fwd_pp.py
Items are numbered in the issue stream's order (cube pair jj, key pair p, group g):
tix = (jj * np + p) * 2 + g. Columns (clock64 cycles from the first event):
  Siss  the issuer's S(tix) commit      gotS  the group saw s_full
  vote  max / lazy-rescale vote done    tok   MUFU token acquired
  Pdn   P^T stores done                 Parr  P-full arrival (fence done)
  Oiss  the issuer's O(tix) issue (after the P-full barrier)
  Sgran the issuer passed the slot barrier before S(tix)   Omma  O's MMAs and commits issued
and, per ring slot k (events 2k, 2k+1 of the S / O stream), the producer's issue (ld)
and the watcher's landing (in). usage: trace_fwd_pp.py [cta] [first] [count]"""
import ctypes as C
import sys

import torch

sys.path.insert(0, ".")
import paper_2505_13389_b200 as vsa  # noqa: E402

cta = int(sys.argv[1]) if len(sys.argv) > 1 else 5
first = int(sys.argv[2]) if len(sys.argv) > 2 else 64
count = int(sys.argv[3]) if len(sys.argv) > 3 else 32
grid, B, H, d, k = (16, 32, 32), 8, 16, 64, 32  # DiT
L = vsa.TileLayout(*grid, pad=True)
op = vsa.VsaOp(L, B, H, d, k)
g = torch.Generator(device="cuda").manual_seed(1)
x = [torch.randn((B, H, L.seq_len, d), generator=g, device="cuda").bfloat16() for _ in range(5)]
for _ in range(3):
    op.forward(*x)
torch.cuda.synchronize()
cap = 16 * 256
buf = torch.zeros(cap, dtype=torch.int64, device="cuda")
vsa.lib().vsa_debug_trace(C.c_void_p(buf.data_ptr()), cap, cta, 0)
op.forward(*x)
torch.cuda.synchronize()
vsa.lib().vsa_debug_trace(None, 0, 0, 0)
b = buf.cpu().tolist()
ev = {(i // 256, i % 256): b[i] for i in range(cap) if b[i] != 0}
if not ev:
    sys.exit("no events: is the library built with -DVSA_TRACE?")
t0 = min(ev.values())
cols = [("Sgran", 5), ("Siss", 3), ("gotS", 7), ("vote", 10), ("tok", 12), ("Pdn", 13), ("Parr", 8), ("Oiss", 4),
        ("Omma", 6)]
print(" tix g" + "".join(f"{n:>8s}" for n, _ in cols))
for t in range(first, min(first + count, 256)):
    row = [ev.get((c, t)) for _, c in cols]
    print(f"{t:4d} {t & 1}" + "".join(f"{(r - t0) if r else -1:8d}" for r in row))
print("\nslot  ld      in")
for s in range(first, min(first + count, 256)):
    a, c = ev.get((1, s)), ev.get((2, s))
    print(f"{s:4d}" + "".join(f"{(r - t0) if r else -1:8d}" for r in (a, c)))


def span(c0, c1, ts):
    v = [ev[(c1, t)] - ev[(c0, t)] for t in ts if (c0, t) in ev and (c1, t) in ev]
    return sum(v) / len(v) if v else float("nan")


ts = [t for t in range(first, min(first + count, 256))]
per = [(ev[(3, t + 2)] - ev[(3, t)]) / 2 for t in ts if (3, t) in ev and (3, t + 2) in ev]
print(f"\nitem period (S issue to S issue, per item): {sum(per) / max(len(per), 1):.0f} cycles")
for name, c0, c1 in [("gotS->vote (score / max)", 7, 10), ("vote->tok (token wait)", 10, 12),
                     ("tok->Pdn (exponentials)", 12, 13), ("Pdn->Parr (fence)", 13, 8),
                     ("Parr->Oiss", 8, 4), ("Siss->gotS", 3, 7)]:
    print(f"  {name:28s} {span(c0, c1, ts):7.0f}")
gw = [ev[(7, t + 2)] - ev[(8, t)] for t in ts if (8, t) in ev and (7, t + 2) in ev]
print(f"  {'Parr->next gotS (S wait)':28s} {sum(gw) / max(len(gw), 1):7.0f}")
print("issuer loop (per item):")
for name, c0, c1 in [("Sgran->Siss (S MMAs + commits)", 5, 3), ("Oiss->Omma (O MMAs + commits)", 4, 6),
                     ("Opre->Oiss (P-full barrier)", 15, 4)]:
    print(f"  {name:28s} {span(c0, c1, ts):7.0f}")
# cross-item gaps: S(t+2) issued -> O(t) pre-barrier; O(t) issued -> Sgran(t+3)
a1 = [ev[(15, t)] - ev[(3, t + 2)] for t in ts if (3, t + 2) in ev and (15, t) in ev]
a2 = [ev[(5, t + 3)] - ev[(6, t)] for t in ts if (6, t) in ev and (5, t + 3) in ev]
print(f"  {'Siss(t+2)->Opre(t)':28s} {sum(a1) / max(len(a1), 1):7.0f}")
print(f"  {'Omma(t)->Sgran(t+3)':28s} {sum(a2) / max(len(a2), 1):7.0f}")
