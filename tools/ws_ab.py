import sys, torch
sys.path.insert(0, ".")
import paper_2505_13389_b200 as vsa
cfgs = {"wan13": ((21, 30, 52), 1, 12, 128, 78), "dit": ((16, 32, 32), 8, 16, 64, 32)}
for cfg, (grid, B, H, d, k) in cfgs.items():
    L = vsa.TileLayout(*grid, pad=True)
    g = torch.Generator(device="cuda").manual_seed(1)
    x = [torch.randn((B, H, L.seq_len, d), generator=g, device="cuda").bfloat16() for _ in range(6)]
    for ws in (True, False):
        op = vsa.VsaOp(L, B, H, d, k, bwd_workspace=ws)
        op.timing(True)
        for _ in range(3):
            op.forward(*x[:5]); op.backward(x[5])
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(5):
            op.forward(*x[:5]); op.backward(x[5])
        b.record(); torch.cuda.synchronize()
        print(cfg, "ws" if ws else "recompute", round(a.elapsed_time(b) / 5, 3), op.stage_ms(), op.used_ds_workspace, flush=True)
        del op; torch.cuda.empty_cache()
