#!/usr/bin/env python
# SPDX-License-Identifier: Apache-2.0
"""bench.py — VSA attention forward+backward on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config wan13] [--impl ours|reference]

One step = one VSA forward + backward pass (tile+pool, coarse attention + Top-K
block map, block-sparse fine attention with gated combine + untile, backward
prologue, coarse backward, fine dQ / dK dV) over one synthetic batch of the
Wan2.1-1.3B 480p layer shape (BASELINE.json configs[1]): B=1, H=12, d=128,
grid (21,30,52) zero-padded to (24,32,52), cube (4,4,4), top-k 78 of 624 cubes
(87.5% sparsity), bf16 I/O with fp32 accumulation.

value  : effective TFLOP/s = algorithmic FLOPs (fine 14*64^2*d per selected tile
         + coarse 14*nc^2*d per (b,h)) / device time, summed
         over ranks (weak scaling: every rank runs its own batch element),
         inputs resident in HBM. ms_per_step is the max over ranks.
e2e    : the same metric through the public API (VsaOp) with pinned HOST
         buffers: H2D of q,k,v,gc,gf,dO and D2H of O,dQ,dK,dV,dGc,dGf every step.
roofline: the dominant kernel (per-stage CUDA events on the launch stream).
cpu_baseline: the CPU restatement (oracle/, "port") on one (b,h) head of the
         same workload, all host threads, N=1 rank 0 only.
Multi-GPU: torchrun, one process per GPU over NCCL (barrier + max-over-ranks
timing only; the path has no data exchange — batch x head partitioning).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # BASELINE.json configs[1] — the headline workload
    "wan13": dict(workload="Wan2.1-1.3B 480p layer", grid=(21, 30, 52), B=1, H=12, d=128, top_k=78),
    "tiny": dict(workload="tiny (configs[0] grid, d=64)", grid=(8, 16, 16), B=1, H=2, d=64, top_k=4),
    "sweep32": dict(workload="paper sweep 32^3 d128 87.5%", grid=(32, 32, 32), B=1, H=16, d=128, top_k=64),
    "dit": dict(workload="DiT pretraining batch", grid=(16, 32, 32), B=8, H=16, d=64, top_k=32),
    "wan14": dict(workload="Wan2.1-14B 720p layer (1 GPU, all heads)", grid=(21, 45, 80), B=1, H=40, d=128,
                  top_k=144),
    # BASELINE configs[3]: sequence-parallel over the GPUs with the Ulysses all-to-all
    "wan14sp": dict(workload="Wan2.1-14B 720p layer, Ulysses sequence-parallel", grid=(21, 45, 80), B=1, H=40,
                    d=128, top_k=144, sp=True),
}

STAGES = ["tile_pool", "coarse_fwd", "fine_fwd", "prologue", "coarse_bwd", "fine_bwd"]


def metric_name(cfg):
    """The one metric string both arms print (the driver pairs the lines on it)."""
    return f"VSA fwd+bwd effective TFLOPS (algorithmic FLOPs / device time), {cfg['workload']}"


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return dict(hbm=p["hbm_gbs"], bf16=p["bf16_tflops"], bf16_sust=p["bf16_tflops_sustained"], src="measured")
    except Exception:
        return dict(hbm=6650.0, bf16=1590.0, bf16_sust=1400.0, src="fallback (B200_PROFILING.md)")


def flops(cfg, nc, top_k, d, cube=64):
    B, H = cfg["B"], cfg["H"]
    tiles = B * H * nc * top_k
    fine_f = 4 * cube * cube * d * tiles
    fine_b = 10 * cube * cube * d * tiles
    coarse_f = 4 * nc * nc * d * B * H
    coarse_b = 10 * nc * nc * d * B * H
    return dict(tiles=tiles, fine_fwd=fine_f, fine_bwd=fine_b, coarse_fwd=coarse_f, coarse_bwd=coarse_b,
                total=fine_f + fine_b + coarse_f + coarse_b)


class ClockSampler:
    """SM clock + clock-event (throttle) reasons polled through NVML every ~2 ms
    during the timed region (nvidia-smi's 100 ms cadence is too coarse for a
    10 ms step); falls back to nvidia-smi if NVML is unavailable."""

    REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown"}

    def __init__(self, local_rank):
        vis = os.environ.get("CUDA_VISIBLE_DEVICES", "")
        ids = [x for x in vis.split(",") if x.strip()]
        self.idx = int(ids[local_rank]) if local_rank < len(ids) and ids[local_rank].strip().isdigit() else local_rank
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        self._nvml = None

    def _sample(self):
        nv, h = self._nvml, self._h
        self.samples.append(float(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)))
        r = int(self._get_r(h))
        for bit, name in self.REASONS.items():
            if r & bit:
                self.reasons.add(name)

    def _poll(self):
        while not self._stop.is_set():
            try:
                self._sample()
            except Exception:
                return
            time.sleep(0.002)

    def __enter__(self):
        try:
            import pynvml

            pynvml.nvmlInit()
            self._nvml = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(self.idx)
            self._get_r = (getattr(pynvml, "nvmlDeviceGetCurrentClocksEventReasons", None)
                           or pynvml.nvmlDeviceGetCurrentClocksThrottleReasons)
            self.max_mhz = float(pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM))
            self._t = threading.Thread(target=self._poll, daemon=True)
            self._t.start()
        except Exception:
            self._nvml = None
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.idx), "--query-gpu=clocks.sm,clocks.max.sm",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=10)
                a, b = out.stdout.strip().split(",")[:2]
                self.samples.append(float(a))
                self.max_mhz = float(b)
            except Exception:
                pass
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._nvml is not None:
            self._t.join(timeout=2)
            try:
                self._sample()  # at least one sample at the end of the timed region
            except Exception:
                pass

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unsampled"], "samples": 0}
        s = sorted(self.samples)
        return {"sm_mhz": s[len(s) // 2], "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(s), "source": "nvml" if self._nvml is not None else "nvidia-smi"}


def make_inputs(cfg, S, dtype, device, u0, u1):
    """q, k, v, gc, gf, dO of (b,h) units [u0, u1) as [1, u1-u0, S, d]; each unit drawn from
    its own seeded generator, so a unit's data does not depend on the partition."""
    import torch

    n, d = u1 - u0, cfg["d"]
    xs = [torch.empty((1, n, S, d), dtype=dtype, device=device) for _ in range(6)]
    g = torch.Generator(device=device)
    for j, u in enumerate(range(u0, u1)):
        g.manual_seed(1234 + u)
        for x in xs:
            x[0, j].copy_(torch.randn((S, d), generator=g, device=device, dtype=torch.float32))
    return xs


def run_ours(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    import paper_2505_13389_b200 as vsa

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    cfg = CONFIGS[args.config]
    dtype = torch.bfloat16
    L = vsa.TileLayout(*cfg["grid"], pad=True)
    nc, S, d, K = L.num_cubes, L.seq_len, cfg["d"], cfg["top_k"]
    fl = flops(cfg, nc, K, d)
    peaks = load_peaks()

    # batch x head partition of the ONE problem: this rank's contiguous unit
    # range, no data-path collective (strong scaling; paper_2505_13389_b200/partition.py)
    from paper_2505_13389_b200.partition import SubSplitVsa, partition_tasks, partition_units

    units = cfg["B"] * cfg["H"]
    # whole units per rank when they divide evenly; otherwise the (unit, cube) task sub-split
    # (heads shared between ranks, lse / delta exchanged with one all-reduce each)
    split = world > 1 and units % world != 0
    if split:
        part = SubSplitVsa(L, cfg["B"], cfg["H"], d, K, rank, world, coarse=args.coarse)
        op, u0, u1 = part.op, part.ua, part.ub
        parts = partition_tasks(units, nc, world)
    else:
        part = None
        parts = partition_units(units, world)
        u0, u1 = parts[rank]
        op = vsa.VsaOp(L, 1, u1 - u0, d, K, dtype=dtype, coarse=args.coarse) if u1 > u0 else None
    n = u1 - u0
    q, k, v, gc, gf, do = make_inputs(cfg, S, dtype, dev, u0, u1)
    outs = [torch.empty_like(q) for _ in range(6)]

    def step():
        if split:
            part.forward(q, k, v, gc, gf, out=outs[0], check_inputs=False)
            part.backward(do, *outs[1:], check_inputs=False)
            return
        if op is None:
            return
        op.forward(q, k, v, gc, gf, out=outs[0], check_inputs=False)
        op.backward(do, *outs[1:], check_inputs=False)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    for _ in range(args.warmup):
        step()
    barrier()
    lib = vsa.lib()
    n0 = lib.vsa_kernel_launches()
    st = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    # per-stage breakdown: CUDA events the native operator records between its stages on
    # the launch stream during the timed steps themselves (no host gaps, same clocks)
    if op is not None:
        op.timing(True)
    with ClockSampler(local_rank) as clk:
        e0.record(st)
        for _ in range(args.steps):
            step()
        e1.record(st)
        barrier()
    launches = lib.vsa_kernel_launches() - n0
    ms = max_over_ranks(e0.elapsed_time(e1) / args.steps)
    value = fl["total"] / (ms * 1e-3) / 1e12  # the whole problem over the slowest rank

    stage_ms = {s_: 0.0 for s_ in STAGES}
    if op is not None:
        stage_ms = op.stage_ms()
        op.timing(False)

    # the other coarse mode (fp32 canonical <-> bf16 tcgen05), same inputs: step and coarse times
    other_coarse = None
    if op is not None and world == 1 and L.num_cubes % 8 == 0 and not split:
        alt = "bf16" if args.coarse == "fp32" else "fp32"
        opa = vsa.VsaOp(L, 1, n, d, K, dtype=dtype, coarse=alt)

        def astep():
            opa.forward(q, k, v, gc, gf, out=outs[0], check_inputs=False)
            opa.backward(do, *outs[1:], check_inputs=False)

        for _ in range(2):
            astep()
        barrier()
        opa.timing(True)
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        na = max(3, min(args.steps, 10))
        a0.record(st)
        for _ in range(na):
            astep()
        a1.record(st)
        barrier()
        ast = opa.stage_ms()
        ams = a0.elapsed_time(a1) / na
        other_coarse = {"coarse": alt, "ms_per_step": round(ams, 4),
                        "value": round(fl["total"] / (ams * 1e-3) / 1e12, 2),
                        "stages_ms": {s_: round(ast[s_], 4) for s_ in STAGES}}
        del opa

    # dense baseline: the same kernels with top-k = all cubes
    dense = None
    if not args.no_dense and not split:
        opd = vsa.VsaOp(L, 1, n, d, nc, dtype=dtype) if n else None
        fld = flops(cfg, nc, nc, d)

        def dstep():
            if opd is None:
                return
            opd.forward(q, k, v, gc, gf, out=outs[0], check_inputs=False)
            opd.backward(do, *outs[1:], check_inputs=False)

        dstep()
        barrier()
        d0, d1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        nd = max(1, min(args.steps, 3))
        d0.record(st)
        for _ in range(nd):
            dstep()
        d1.record(st)
        barrier()
        dms = max_over_ranks(d0.elapsed_time(d1) / nd)
        dense = dict(ms_per_step=round(dms, 3), tflops=round(fld["total"] / (dms * 1e-3) / 1e12, 1),
                     speedup_vsa_vs_dense=round(dms / ms, 2))
        del opd

    # gate projection (the rest of vsa_forward/vsa_backward): tcgen05 GEMMs
    # z = hidden.Wg (+bias, sigmoid, split) and dhidden / dWg / dbias, model_dim = H*d
    gate = None
    if world == 1 and cfg["B"] * cfg["H"] * cfg["d"] % 256 == 0 and (cfg["H"] * cfg["d"]) % 256 == 0:
        md = cfg["H"] * cfg["d"]
        hid = torch.randn((cfg["B"], 1, S, md), device=dev).to(dtype)
        wg = (torch.randn((md, 2 * cfg["H"] * d), device=dev) / md ** 0.5).to(dtype)
        gp = vsa.VsaParams(wg, torch.zeros(2 * cfg["H"] * d, device=dev), K, activation=1)
        gcg, gfg = vsa.gates_from_hidden(hid, gp, cfg["H"], d, layout=L)
        qg, kg = q.view(gcg.shape), k.view(gcg.shape)  # stand-in upstream gate gradients
        g0, g1, g2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        for _ in range(2):
            vsa.gates_from_hidden(hid, gp, cfg["H"], d, layout=L)
            vsa.gate_backward(hid, gp, gcg, gfg, qg, kg, layout=L)
        g0.record(st)
        for _ in range(5):
            vsa.gates_from_hidden(hid, gp, cfg["H"], d, layout=L)
        g1.record(st)
        for _ in range(5):
            vsa.gate_backward(hid, gp, gcg, gfg, qg, kg, layout=L)
        g2.record(st)
        torch.cuda.synchronize()
        gfl = 2 * cfg["B"] * S * md * 2 * cfg["H"] * d
        tf, tb = g0.elapsed_time(g1) / 5, g1.elapsed_time(g2) / 5
        gate = {"model_dim": md, "fwd_ms": round(tf, 4), "fwd_tflops": round(gfl / tf / 1e9, 1),
                "bwd_ms": round(tb, 4), "bwd_tflops": round(2 * gfl / tb / 1e9, 1),
                "note": "not in value: the BASELINE metric is the attention op; gates are inputs there"}
        del hid, wg, gcg, gfg, qg, kg

    # e2e through the public API with pinned host buffers: VsaHostPipeline overlaps the
    # H2D of unit-group i+1 and the D2H of group i-1 with the kernels of group i
    hin = [t.cpu().pin_memory() for t in (q, k, v, gc, gf, do)]
    hout = [torch.empty(t.shape, dtype=t.dtype, pin_memory=True) for t in outs]
    if not split:
        del op  # free the resident-input operator's buffers before building the pipeline
        torch.cuda.empty_cache()
    pipe = (vsa.VsaHostPipeline(L, 1, n, d, K, chunks=min(args.e2e_chunks, n), dtype=dtype, slots=args.e2e_slots)
            if n and not split
            else None)
    if split:  # the sub-split op stays; its inputs come from host every step
        op = part.op
        q, k, v, gc, gf, do = (torch.empty_like(t) for t in (q, k, v, gc, gf, do))

    def e2e_step():
        if pipe is not None:
            pipe.run(hin, hout)
        elif split:
            for dst, src in zip((q, k, v, gc, gf, do), hin):
                dst.copy_(src, non_blocking=True)
            step()
            for dst, src in zip(hout, outs):
                dst.copy_(src, non_blocking=True)

    e2e_step()
    barrier()
    e2 = torch.cuda.Event(enable_timing=True)
    e3 = torch.cuda.Event(enable_timing=True)
    ne = max(1, min(args.steps, 5))
    e2.record(st)
    for _ in range(ne):
        e2e_step()
    e3.record(st)
    barrier()
    ems = max_over_ranks(e2.elapsed_time(e3) / ne)
    h2d = sum(t.numel() * t.element_size() for t in hin)
    d2h = sum(t.numel() * t.element_size() for t in hout)
    if world > 1:  # whole-job bytes: every rank copies its own units
        t = torch.tensor([h2d, d2h], dtype=torch.float64, device=dev)
        dist.all_reduce(t)
        h2d, d2h = int(t[0].item()), int(t[1].item())

    if rank != 0:
        return None

    # roofline of the dominant kernel (rank 0's share of the work: n units)
    n_eff = (part.t1 - part.t0) / nc if split else n  # units' worth of rank 0's tasks
    fl_r = flops(dict(B=1, H=max(n_eff, 1e-9)), nc, K, d)
    dom = max(("fine_fwd", "fine_bwd"), key=lambda s: stage_ms[s])
    ach = fl_r[dom] / (max(stage_ms[dom], 1e-9) * 1e-3) / 1e12
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tpath):
        try:
            with open(tpath) as f:
                tj = json.load(f)
            traffic = tj.get(args.config, {}).get(dom)
        except Exception:
            traffic = None
    # the binding resource of the fine kernels: the SM's shared-memory data pipe
    # (tensor-core operand reads + thread shared stores), from the committed ncu summary
    smem_pipe = None
    npath = os.path.join(ROOT, "profiles", "ncu_r2k_kernels.json")
    if os.path.exists(npath) and args.config == "wan13" and d == 128:
        try:
            with open(npath) as f:
                ks = json.load(f)["kernels"]
            smem_pipe = {k["kernel"].split("(")[0].split()[-1]: round(k["smem_tc_wavefronts_pct"] +
                                                                      k["smem_lsu_wavefronts_pct"], 1)
                         for k in ks if k.get("smem_tc_wavefronts_pct")}
        except Exception:
            smem_pipe = None
    # Second roofline of the fine kernels: the L2 -> SMEM stream of the streamed operand
    # tiles (selections are random, so a tile's K/V (forward) or Q/dO (dK/dV) and the K + dS
    # of dQ come from L2 once per selected tile), against the measured chip-wide L2 -> SMEM
    # TMA rate (profiles/tma_bench_r1.txt, 2-D 64 x 128 B boxes on all SMs).
    tiles_r = n_eff * nc * K
    l2_bytes = {"fine_fwd": tiles_r * 4 * 64 * d,                                    # K, V tiles
                "fine_bwd": tiles_r * (4 * 64 * d + 8192 + 2 * 64 * d + 8192)}      # Q, dO; dS out; K, dS in
    l2_peak = 12805.4
    l2_roof = {"bound": "l2", "unit": "GB/s", "peak": l2_peak,
               "peak_src": "measured L2->SMEM TMA rate, all SMs (profiles/tma_bench_r1.txt)",
               "kernels": {s: {"bytes": int(l2_bytes[s]),
                               "achieved": round(l2_bytes[s] / (max(stage_ms[s], 1e-9) * 1e-3) / 1e9, 1),
                               "frac": round(l2_bytes[s] / (max(stage_ms[s], 1e-9) * 1e-3) / 1e9 / l2_peak, 4)}
                           for s in ("fine_fwd", "fine_bwd")}}
    bytes_tp = n * 3 * (S * d * 2 + L.seq_padded * d * 2 + nc * d * 4)  # K1 runs on whole units
    # K6a: reads dO, Gc, Gf (raster) + the tiled fine output + Oc cubes; writes dOf (tiled),
    # dGc, dGf (raster), delta (fp32 per tiled row) and the dOc cube sums
    bytes_pro = n * (5 * S * d * 2 + 2 * L.seq_padded * d * 2 + L.seq_padded * 4 + 2 * nc * d * 4)
    hbm_bytes = {"tile_pool": bytes_tp, "prologue": bytes_pro}
    stages = {}
    for s in STAGES:
        e = {"ms": round(stage_ms[s], 4)}
        if s in ("fine_fwd", "fine_bwd", "coarse_fwd", "coarse_bwd") and stage_ms[s] > 0:
            e["tflops"] = round(fl_r[s] / (stage_ms[s] * 1e-3) / 1e12, 1)
        if s in hbm_bytes and stage_ms[s] > 0:  # HBM passes: algorithmic bytes / time vs the copy rate
            e["gbs"] = round(hbm_bytes[s] / (stage_ms[s] * 1e-3) / 1e9, 1)
            e["frac_of_copy"] = round(e["gbs"] / peaks["hbm"], 3)
        stages[s] = e
    line = {
        "metric": metric_name(cfg),
        "value": round(value, 2),
        "unit": "TFLOP/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(ms, 4),
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "bf16",
        "data": "synthetic (torch.randn, seeded per (b,h) unit)",
        "config": {
            "workload": cfg["workload"], "B": cfg["B"], "H": cfg["H"], "head_dim": d, "grid": list(cfg["grid"]),
            "grid_padded": list(L.padded), "cube": [4, 4, 4], "num_cubes": nc, "top_k": K,
            "sparsity": round(1 - K / nc, 4), "global_batch": cfg["B"], "seq_len": S,
            "parallelism": (f"bh{world}: batch x head partition of one problem, "
                            f"{min(b - a for a, b in parts)}-{max(b - a for a, b in parts)} of {units} (b,h) units "
                            f"per GPU, no collective") if not split else
                           (f"bh{world}+cube split: {min(b - a for a, b in parts)}-{max(b - a for a, b in parts)} of "
                            f"{units * nc} (unit, cube) tasks per GPU, lse / delta all-reduce of shared heads"),
            "l2": "inputs larger than L2 (6 x {:.0f} MB bf16 per step)".format(q.numel() * 2 / 1e6),
            "flops_per_step": fl["total"],
        },
        "frac_of_peak": round(value / world / peaks["bf16"], 4),
        "roofline": {"bound": "tensor", "kernel": dom, "achieved": round(ach, 1), "peak": peaks["bf16"],
                     "peak_kind": f"bf16_tflops burst ({peaks['src']}; the kernel is a ms-long launch timed "
                                  f"inside a sub-second loop)", "unit": "TFLOP/s",
                     "frac": round(ach / peaks["bf16"], 4), "frac_of_sustained": round(ach / peaks["bf16_sust"], 4),
                     "traffic": traffic,
                     "algorithmic_flops_per_launch": fl_r[dom],
                     "smem_pipe_busy_pct": smem_pipe,
                     "note": "N=64 SS UMMAs are capped at 2/3 of the tensor peak by the 128 B/cycle SMEM "
                             "operand port; smem_pipe_busy_pct = ncu TC + LSU shared wavefronts per kernel "
                             "(profiles/ncu_r2k_kernels.json, DESIGN.md section 4)"},
        "l2_roofline": l2_roof,
        "stages": stages,
        "dense_baseline": dense,
        "coarse_mode": args.coarse,
        "other_coarse_mode": other_coarse,
        "gate_projection": gate,
        "e2e": {"value": round(fl["total"] / (ems * 1e-3) / 1e12, 3), "unit": "TFLOP/s",
                "ms_per_step": round(ems, 3), "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
        "gpu_launches": int(launches),
        "clocks": clk.summary(),
    }
    if world == 1 and not args.no_cpu:
        line["cpu_baseline"] = cpu_baseline(cfg, 3, warmup=1)
    return line


def run_sp(args, rank, world, local_rank):
    """Ulysses sequence parallelism (BASELINE configs[3]): rank r holds the
    sequence shard [B, S/P, H, d] of q, k, v, gates and dO; the all-to-alls reshard to
    H/P heads x the whole sequence and back. Total work is fixed: strong scaling."""
    import torch

    import paper_2505_13389_b200 as vsa

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    cfg = CONFIGS[args.config]
    dtype = torch.bfloat16
    L = vsa.TileLayout(*cfg["grid"], pad=True)
    nc, S, d, K, B, H = L.num_cubes, L.seq_len, cfg["d"], cfg["top_k"], cfg["B"], cfg["H"]
    fl = flops(cfg, nc, K, d)
    peaks = load_peaks()
    u = vsa.UlyssesVsa(L, B, H, d, K, dtype=dtype)
    P, Sc = u.x.P, u.x.Sc
    g = torch.Generator(device=dev)
    g.manual_seed(4321 + rank)
    shards = [torch.randn((B, Sc, H, d), generator=g, device=dev, dtype=torch.float32).to(dtype) for _ in range(6)]

    def step(xs):
        out = u.forward(*xs[:5])
        return (out,) + tuple(u.backward(xs[5]))

    def barrier():
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        return float(t.item())

    for _ in range(args.warmup):
        step(shards)
    barrier()
    lib = vsa.lib()
    n0 = lib.vsa_kernel_launches()
    st = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local_rank) as clk:
        e0.record(st)
        for _ in range(args.steps):
            step(shards)
        e1.record(st)
        barrier()
    launches = lib.vsa_kernel_launches() - n0
    ms = max_over_ranks(e0.elapsed_time(e1) / args.steps)
    value = fl["total"] / (ms * 1e-3) / 1e12

    nrep = max(3, min(args.steps, 10))
    u.op.timing(True)
    for _ in range(nrep):
        step(shards)
    stage_ms = u.op.stage_ms()
    u.op.timing(False)

    # e2e: pinned host shards in, the six results out, every step
    hin = [t.cpu().pin_memory() for t in shards]
    hout = [torch.empty((B, Sc, H, d), dtype=dtype, pin_memory=True) for _ in range(6)]

    def e2e_step():
        xs = [h.to(dev, non_blocking=True) for h in hin]
        for o, r in zip(hout, step(xs)):
            o.copy_(r, non_blocking=True)

    e2e_step()
    barrier()
    e2, e3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ne = max(1, min(args.steps, 3))
    e2.record(st)
    for _ in range(ne):
        e2e_step()
    e3.record(st)
    barrier()
    ems = max_over_ranks(e2.elapsed_time(e3) / ne)
    if rank != 0:
        return None
    h2d = sum(t.numel() * t.element_size() for t in hin)
    dom = max(("fine_fwd", "fine_bwd"), key=lambda s: stage_ms[s])
    fl_rank = flops(dict(B=B, H=H // P), nc, K, d)  # per-rank share (each rank owns H/P heads)
    ach = fl_rank[dom] / (stage_ms[dom] * 1e-3) / 1e12
    stages = {s: {"ms": round(stage_ms[s], 4)} for s in STAGES}
    for s in ("fine_fwd", "fine_bwd", "coarse_fwd", "coarse_bwd"):
        if stage_ms[s] > 0:
            stages[s]["tflops"] = round(fl_rank[s] / (stage_ms[s] * 1e-3) / 1e12, 1)
    return {
        "metric": metric_name(cfg),
        "value": round(value, 2), "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(ms, 4), "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "bf16", "data": "synthetic (torch.randn, seeded per rank)",
        "config": {"workload": cfg["workload"], "B": B, "H": H, "head_dim": d, "grid": list(cfg["grid"]),
                   "grid_padded": list(L.padded), "cube": [4, 4, 4], "num_cubes": nc, "top_k": K,
                   "sparsity": round(1 - K / nc, 4), "global_batch": B, "seq_len": S,
                   "parallelism": f"sp{P} (Ulysses all-to-all over NCCL, {H // P} heads per GPU)",
                   "l2": "inputs larger than L2", "flops_per_step": fl["total"]},
        "frac_of_peak": round(value / world / peaks["bf16"], 4),
        "roofline": {"bound": "tensor", "kernel": dom, "achieved": round(ach, 1), "peak": peaks["bf16"],
                     "peak_kind": f"bf16_tflops burst ({peaks['src']})", "unit": "TFLOP/s",
                     "frac": round(ach / peaks["bf16"], 4), "traffic": None,
                     "algorithmic_flops_per_launch": fl_rank[dom]},
        "stages": stages,
        "e2e": {"value": round(fl["total"] / (ems * 1e-3) / 1e12, 3), "unit": "TFLOP/s", "ms_per_step": round(ems, 3),
                "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": h2d},
        "gpu_launches": int(launches),
        "clocks": clk.summary(),
    }


def _oracle_head(cfg, seed):
    """One (b,h) head of the workload for the CPU restatement: tile-ordered padded q, k, v,
    dO drawn like the reference (mt19937_64, vsa_cli.cpp:227-230)."""
    import numpy as np

    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as orc

    T, X, Y = cfg["grid"]
    Tp, Xp, Yp = orc.padded_extents(T, X, Y, 4, 4, 4)
    L = orc.TileLayout(Tp, Xp, Yp, 4, 4, 4)
    rng = orc.Rng(seed)
    q, k, v, do = (orc.randn(rng, 1, 1, L.seq_len, cfg["d"], np.float32) for _ in range(4))
    return orc, L, (q, k, v, do)


def _oracle_step(orc, L, x, K):
    """coarse_forward_select + fine_forward + fine_backward + coarse_backward of one head
    (the reference's vsa fwd + bwd attention work; vsa_cli.cpp:232-256 times the forward)."""
    q, k, v, do = x
    t0 = time.perf_counter()
    art = orc.coarse_forward_select(L, q, k, v, K)
    _, _, lse = orc.fine_forward(L, q, k, v, art.sel)
    orc.fine_backward(L, q, k, v, art.sel, do, lse)
    orc.coarse_backward(art, L, do, q, k, v)
    return time.perf_counter() - t0


def cpu_baseline(cfg, reps, warmup=1):
    """The oracle (CPU restatement of the reference) on ONE (b,h) head of the workload:
    coarse fwd + fine fwd + fine bwd + coarse bwd, all host threads; `warmup` untimed
    runs, then the median of `reps` (the reference bench protocol, vsa_cli.cpp:232-256)."""
    orc, L, x = _oracle_head(cfg, 0)
    for _ in range(warmup):
        _oracle_step(orc, L, x, cfg["top_k"])
    times = sorted(_oracle_step(orc, L, x, cfg["top_k"]) for _ in range(reps))
    t = times[len(times) // 2]
    fl = flops(dict(B=1, H=1), L.num_cubes, cfg["top_k"], cfg["d"])["total"]
    return {"value": round(fl / t / 1e12, 5), "unit": "TFLOP/s", "cores": orc.max_threads(), "kind": "port",
            "sample": f"one (b,h) head of {cfg['workload']} (1/{cfg['B'] * cfg['H']} of a step), "
                      f"coarse+fine fwd+bwd, median of {reps} after {warmup} warm-up: {t:.2f} s",
            "seconds": round(t, 3)}


def run_reference(args, rank, world):
    """--impl reference: the reference algorithm on the host cores (the oracle port; the
    Eigen reference cannot be compiled here), same metric, unit and config as our arm.
    Each step is a bounded sample of the workload: one (b,h) head's fwd + bwd (1/(B*H)
    of the layer); `steps` samples are timed after `warmup` untimed ones, and ms_per_step
    is the time of one such sample (what was actually timed)."""
    if rank != 0:
        return None
    cfg = CONFIGS[args.config]
    orc, L, x = _oracle_head(cfg, 0)
    orc.set_num_threads(os.cpu_count() or 1)
    K = cfg["top_k"]
    for _ in range(args.warmup):
        _oracle_step(orc, L, x, K)
    times = [_oracle_step(orc, L, x, K) for _ in range(args.steps)]
    t = sum(times) / len(times)
    fl = flops(dict(B=1, H=1), L.num_cubes, K, cfg["d"])["total"]
    value = fl / t / 1e12
    sample = (f"one (b,h) head of {cfg['workload']} per step (1/{cfg['B'] * cfg['H']} of the layer): coarse+fine "
              f"fwd+bwd, {args.steps} timed after {args.warmup} warm-up, mean {t:.3f} s")
    return {
        "metric": metric_name(cfg),
        "impl": "reference", "value": round(value, 5), "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(t * 1e3, 1), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic (mt19937_64 randn, the reference's draws)",
        "config": {"workload": cfg["workload"], "B": cfg["B"], "H": cfg["H"], "head_dim": cfg["d"],
                   "grid": list(cfg["grid"]), "top_k": K, "num_cubes": L.num_cubes,
                   "sample": "one (b,h) head per step; value = that head's algorithmic FLOPs / its time"},
        "cpu_baseline": {"value": round(value, 5), "unit": "TFLOP/s", "cores": orc.max_threads(), "kind": "port",
                         "sample": sample},
        "e2e": {"value": round(value, 5), "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="wan13", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-dense", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--e2e-chunks", type=int, default=6, help="host-pipeline unit groups for the e2e leg")
    ap.add_argument("--e2e-slots", type=int, default=3, help="host-pipeline device buffer slots for the e2e leg")
    ap.add_argument("--coarse", default="fp32", choices=["fp32", "bf16"],
                    help="coarse-stage mode of the headline op: fp32 (bit-exact block map) or bf16 (tcgen05)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    # test hook: VSA_BENCH_BACKEND=gloo runs several ranks on the visible GPUs (ranks share a
    # device when there are fewer GPUs than ranks); the product path is NCCL, one GPU per rank
    backend = os.environ.get("VSA_BENCH_BACKEND", "nccl")
    if backend != "nccl":
        import torch

        local_rank = local_rank % max(1, torch.cuda.device_count())
    if args.impl == "reference":
        line = run_reference(args, rank, world)
        if line is not None:
            print(json.dumps(line), flush=True)
        return
    if world > 1:
        import torch
        import torch.distributed as dist

        torch.cuda.set_device(local_rank)
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        else:
            dist.init_process_group(backend)
    try:
        line = (run_sp if CONFIGS[args.config].get("sp") else run_ours)(args, rank, world, local_rank)
        if line is not None:
            print(json.dumps(line), flush=True)
    finally:
        if world > 1:
            import torch.distributed as dist

            dist.destroy_process_group()


if __name__ == "__main__":
    main()
