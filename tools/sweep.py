# SPDX-License-Identifier: Apache-2.0
"""The paper's kernel sweep (BASELINE.json configs[2]): H=16,
d in {64, 128}, cubic grids 16^3 and 32^3, sparsity in {50, 75, 87.5, 90, 95}% (k =
round(nc * (1 - s))), VSA vs the dense baseline (the same kernels with k = all cubes),
forward and backward timed separately.

    python tools/sweep.py [--out profiles/sweep_r2.json] [--reps 5]

Per point: fine forward and fine backward device times from the operator's native
stage events (fine_fwd = K4+K5, fine_bwd = K6b+K6c), the whole-operator forward
(K1..K5) and backward (K6a..K6d) times, effective TFLOP/s on the algorithmic FLOPs
(fine fwd 4*64^2*d, bwd 10*64^2*d per selected tile) and the speed-up over dense.
Inputs: torch.randn bf16, larger than L2 at 32^3. Each point: 3 warm-up steps, then the
best of three rounds of --reps steps, after a ~2 s warm-up of the GPU."""
import argparse
import json
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2505_13389_b200 as vsa  # noqa: E402


def measure(L, H, d, k, xs, reps):
    op = vsa.VsaOp(L, 1, H, d, k)
    outs = [torch.empty_like(xs[0]) for _ in range(6)]

    def step():
        op.forward(*xs[:5], out=outs[0], check_inputs=False)
        op.backward(xs[5], *outs[1:], check_inputs=False)

    for _ in range(3):
        step()
    torch.cuda.synchronize()
    best = None
    for _ in range(3):  # best of three rounds (short launches on a shared box are noisy)
        op.timing(True)
        e = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        e[0].record()
        for _ in range(reps):
            step()
        e[1].record()
        st = op.stage_ms()
        op.timing(False)
        torch.cuda.synchronize()
        step_ms = e[0].elapsed_time(e[1]) / reps
        if best is None or step_ms < best[0]:
            best = (step_ms, st)
    del op
    return best


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "sweep_r2.json"))
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--grids", default="16,32")
    ap.add_argument("--dims", default="64,128")
    args = ap.parse_args()
    H = 16
    rows = []
    t0 = time.time()
    # warm the GPU to its steady clocks before the first point (~2 s of dense work)
    Lw = vsa.TileLayout(32, 32, 32)
    xw = [torch.randn((1, H, Lw.seq_len, 128), device="cuda").bfloat16() for _ in range(6)]
    tw = time.time()
    while time.time() - tw < 2.0:
        measure(Lw, H, 128, Lw.num_cubes, xw, 1)
    del xw
    for n in (int(x) for x in args.grids.split(",")):
        L = vsa.TileLayout(n, n, n)
        nc = L.num_cubes
        for d in (int(x) for x in args.dims.split(",")):
            g = torch.Generator(device="cuda").manual_seed(n * 1000 + d)
            xs = [torch.randn((1, H, L.seq_len, d), generator=g, device="cuda").bfloat16() for _ in range(6)]
            dstep, dst = measure(L, H, d, nc, xs, max(2, args.reps // 2))
            for s in (0.5, 0.75, 0.875, 0.9, 0.95):
                k = max(1, int(round(nc * (1 - s))))
                step, st = measure(L, H, d, k, xs, args.reps)
                tiles = H * nc * k
                ff, fb = 4 * 64 * 64 * d * tiles, 10 * 64 * 64 * d * tiles
                fwd = st["tile_pool"] + st["coarse_fwd"] + st["fine_fwd"]
                bwd = st["prologue"] + st["coarse_bwd"] + st["fine_bwd"]
                dfwd = dst["tile_pool"] + dst["coarse_fwd"] + dst["fine_fwd"]
                dbwd = dst["prologue"] + dst["coarse_bwd"] + dst["fine_bwd"]
                row = dict(grid=n, tokens=L.seq_len, d=d, heads=H, nc=nc, k=k, sparsity=round(1 - k / nc, 4),
                           fine_fwd_ms=round(st["fine_fwd"], 4), fine_bwd_ms=round(st["fine_bwd"], 4),
                           fine_fwd_tflops=round(ff / st["fine_fwd"] / 1e9, 1),
                           fine_bwd_tflops=round(fb / st["fine_bwd"] / 1e9, 1),
                           op_fwd_ms=round(fwd, 4), op_bwd_ms=round(bwd, 4), step_ms=round(step, 4),
                           dense_fine_fwd_ms=round(dst["fine_fwd"], 4), dense_fine_bwd_ms=round(dst["fine_bwd"], 4),
                           dense_op_fwd_ms=round(dfwd, 4), dense_op_bwd_ms=round(dbwd, 4),
                           speedup_fwd=round(dfwd / fwd, 2), speedup_bwd=round(dbwd / bwd, 2),
                           speedup_step=round(dstep / step, 2), ideal_speedup=round(nc / k, 2))
                rows.append(row)
                print(json.dumps(row), flush=True)
            del xs
            torch.cuda.empty_cache()
    meta = {"what": "paper kernel sweep (BASELINE configs[2]): VSA vs same-kernel dense, fwd / bwd separately",
            "device": torch.cuda.get_device_name(), "reps": args.reps, "seconds": round(time.time() - t0, 1),
            "flop_convention": "fine fwd 4*64^2*d, bwd 10*64^2*d per selected tile; times from native stage events"}
    with open(args.out, "w") as f:
        json.dump({"meta": meta, "rows": rows}, f, indent=1)


if __name__ == "__main__":
    main()
