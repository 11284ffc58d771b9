# SPDX-License-Identifier: Apache-2.0
"""GPU-driven toy trainer: the reference's planted-cube retrieval
task and single-layer VSA training loop (toy.hpp:17-346, analysis.cpp:8-14) on the
B200 operator.

Every step runs the VSA forward and backward through ``VsaOp`` (the C ABI, fp32
parity mode by default: the SIMT kernels accept the toy's tiny head_dim and cube
sizes); the model's own projections (Wq, Wk, Wv, the gate projection) and the
optimizer are small dense host-of-the-op algebra done with torch on the GPU, as the
reference does them with Eigen around its attention calls. Semantics follow
toy.hpp: pass-through gate initialisation (fine gate 1 via the constant channel),
MSE loss |O - target|^2 / n, planted-cube recall of the selection actually used,
Adam or SGD, the sparsity schedule, learned / fixed-random selection policies,
divergence abort, and an FNV-1a snapshot id of the trained weights. The data
generator reproduces generate_batch's construction with numpy's PCG64 stream (the
reference draws from libstdc++'s mt19937_64 + normal_distribution; the task
distribution is the same, the exact samples are not).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np
import torch

from .api import VsaOp, TileLayout, POOL_MEAN


@dataclass
class PlantedTask:
    """PlantedTask (toy.hpp:17-35)."""

    layout: TileLayout
    planted_count: int = 4
    heads: int = 2
    head_dim: int = 8
    signal_scale: float = 2.0
    noise_scale: float = 0.5
    seed: int = 0

    def model_dim(self) -> int:  # [key signature per head | value per head | constant 1]
        return 2 * self.heads * self.head_dim + 1

    def check(self):
        if not (1 <= self.planted_count <= self.layout.num_cubes):
            raise ValueError("PlantedTask: planted_count must be in [1, num_cubes]")
        if self.heads < 1 or self.head_dim < 1:
            raise ValueError("PlantedTask: bad head config")


@dataclass
class ToyBatch:
    hidden: torch.Tensor  # [B, 1, S, model_dim]
    q: torch.Tensor       # generator reference tensors [B, H, S, d]
    k: torch.Tensor
    v: torch.Tensor
    target: torch.Tensor  # [B, H, S, d]
    planted: List[List[int]]


def generate_batch(task: PlantedTask, batch_size: int, seed: int, device="cuda",
                   dtype=torch.float32) -> ToyBatch:
    """generate_batch (toy.hpp:47-103): planted cubes carry a shared key signature,
    values are noise, target = mean of planted-token values + the token's own value.
    Tokens are in tile order (cube = token // cube_size)."""
    task.check()
    if batch_size < 1:
        raise ValueError("generate_batch: batch_size must be >= 1")
    L = task.layout
    S, nc, H, d, cube = L.seq_len, L.num_cubes, task.heads, task.head_dim, L.cube_size
    sig = np.random.Generator(np.random.PCG64(task.seed)).standard_normal((H, d))
    rng = np.random.Generator(np.random.PCG64(seed))
    md = task.model_dim()
    hidden = np.zeros((batch_size, 1, S, md))
    q = np.empty((batch_size, H, S, d))
    k = np.empty_like(q)
    v = np.empty_like(q)
    target = np.empty_like(q)
    planted_all = []
    for b in range(batch_size):
        planted = sorted(rng.choice(nc, size=task.planted_count, replace=False).tolist())
        planted_all.append(planted)
        is_p = np.isin(np.arange(S) // cube, planted)
        for h in range(H):
            key = task.noise_scale * rng.standard_normal((S, d))
            key[is_p] += task.signal_scale * sig[h]
            val = rng.standard_normal((S, d))
            k[b, h], v[b, h] = key, val
            hidden[b, 0, :, h * d:(h + 1) * d] = key
            hidden[b, 0, :, (H + h) * d:(H + h + 1) * d] = val
            q[b, h] = sig[h] + 0.5 * key  # the shared signature plus a self-retrieval term
            pm = val[is_p].sum(axis=0) / (task.planted_count * cube)
            target[b, h] = val + pm
        hidden[b, 0, :, 2 * H * d] = 1.0
    t = lambda a: torch.from_numpy(a).to(device=device, dtype=dtype)
    return ToyBatch(t(hidden), t(q), t(k), t(v), t(target), planted_all)


@dataclass
class SparsitySchedule:
    """SparsitySchedule (analysis.hpp:14-27) and schedule_k (analysis.cpp:8-14)."""

    k_start: int = 256
    k_target: int = 32
    warmup_steps: int = 50
    interval_steps: int = 50
    decrement: int = 10

    def check(self):
        if not (self.k_start >= self.k_target >= 1):
            raise ValueError("SparsitySchedule: need k_start >= k_target >= 1")
        if self.decrement < 1 or self.interval_steps < 1 or self.warmup_steps < 0:
            raise ValueError("SparsitySchedule: decrement and interval must be >= 1")

    def k_at(self, step: int) -> int:
        self.check()
        if step < 0:
            raise ValueError("schedule_k: step must be >= 0")
        if step < self.warmup_steps:
            return self.k_start
        drops = (step - self.warmup_steps) // self.interval_steps
        return max(self.k_target, self.k_start - self.decrement * drops)


SPATIAL_TEMPORAL, STRIDED_WINDOW, COMPRESS_KV = 0, 1, 2
SPATIAL, TEMPORAL = 0, 1


@dataclass
class PatternSpec:
    """PatternSpec (analysis.hpp:78-86): the fixed-pattern baselines."""

    kind: int = SPATIAL_TEMPORAL
    phase: int = SPATIAL
    window_s: int = 8
    window_t: int = 2


def fixed_pattern_selection(layout: TileLayout, spec: PatternSpec) -> np.ndarray:
    """fixed_pattern_selection (analysis.cpp:99-157): the pattern's connectivity at cube
    granularity, [num_cubes, row_len] int32 ascending. Windows must be cube-aligned so
    every row selects the same number of cubes; raises ValueError otherwise."""
    L = layout
    if spec.kind == STRIDED_WINDOW:
        if spec.window_t < 1 or spec.window_s < 1:
            raise ValueError("fixed pattern: window sizes must be >= 1")
        if spec.phase == SPATIAL:
            if spec.window_t % L.cube_t or L.tokens_t % spec.window_t:
                raise ValueError("fixed pattern: temporal window must be cube-aligned")
        elif (spec.window_s % L.cube_h or spec.window_s % L.cube_w or L.tokens_h % spec.window_s
              or L.tokens_w % spec.window_s):
            raise ValueError("fixed pattern: spatial window must be cube-aligned")
    c = np.arange(L.num_cubes)
    ct, ch, cw = c // (L.cubes_h * L.cubes_w), (c // L.cubes_w) % L.cubes_h, c % L.cubes_w
    t, h, w = ct * L.cube_t, ch * L.cube_h, cw * L.cube_w  # cube representatives
    if spec.kind == SPATIAL_TEMPORAL:
        allow = (ct[:, None] == ct[None, :]) if spec.phase == SPATIAL else \
            (ch[:, None] == ch[None, :]) & (cw[:, None] == cw[None, :])
    elif spec.kind == STRIDED_WINDOW:
        if spec.phase == SPATIAL:
            allow = (t[:, None] // spec.window_t) == (t[None, :] // spec.window_t)
        else:
            ws = spec.window_s
            allow = ((h[:, None] // ws) == (h[None, :] // ws)) & ((w[:, None] // ws) == (w[None, :] // ws))
    elif spec.kind == COMPRESS_KV:
        allow = np.ones((L.num_cubes, L.num_cubes), dtype=bool)
    else:
        raise ValueError("fixed pattern: unknown kind")
    counts = allow.sum(axis=1)
    if (counts != counts[0]).any():
        raise ValueError("fixed pattern: window sizes give uneven selection rows")
    if counts[0] < 1:
        raise ValueError("fixed pattern: empty selection row")
    return np.nonzero(allow)[1].reshape(L.num_cubes, int(counts[0])).astype(np.int32)


@dataclass
class OptimizerSettings:
    kind: str = "adam"  # "adam" | "sgd"
    lr: float = 1e-3
    beta1: float = 0.9
    beta2: float = 0.95
    eps: float = 1e-8


@dataclass
class ToyTrainConfig:
    """ToyTrainConfig (toy.hpp:120-131); policy "learned" | "fixed_random" | "fixed_pattern"."""

    batch_size: int = 4
    steps: int = 5000
    top_k: int = 8
    pool: int = POOL_MEAN
    activation: int = 0
    schedule: Optional[SparsitySchedule] = None
    optimizer: OptimizerSettings = field(default_factory=OptimizerSettings)
    policy: str = "learned"
    pattern: PatternSpec = field(default_factory=PatternSpec)  # used by "fixed_pattern"
    seed: int = 1


@dataclass
class TrainStep:
    step: int
    loss: float
    recall: float
    k: int


@dataclass
class TrainReport:
    steps: List[TrainStep]
    model: dict
    snapshot_id: str = ""
    diverged: bool = False

    def _tail(self, name, window):
        if not self.steps:
            return float("nan")
        xs = [getattr(s, name) for s in self.steps[-window:]]
        return sum(xs) / len(xs)

    def final_loss(self, window=50):
        return self._tail("loss", window)

    def final_recall(self, window=50):
        return self._tail("recall", window)


def _fnv1a64(data: bytes, h: int = 0xCBF29CE484222325) -> int:
    for byte in data:
        h ^= byte
        h = (h * 0x100000001B3) & 0xFFFFFFFFFFFFFFFF
    return h


def planted_recall(sel: torch.Tensor, planted: List[List[int]]) -> float:
    """detail::planted_recall (toy.hpp:186-203): fraction of each sample's planted
    cubes present in the used selection, averaged over (sample, head, query cube)."""
    B, H, nc, K = sel.shape
    hit = torch.zeros((B, H, nc), dtype=torch.float64, device=sel.device)
    for b in range(B):
        p = torch.tensor(planted[b], dtype=sel.dtype, device=sel.device)
        hit[b] = (sel[b].unsqueeze(-1) == p).any(dim=2).sum(dim=-1).double() / len(planted[b])
    return float(hit.mean())


def train_toy(task: PlantedTask, cfg: ToyTrainConfig, device="cuda", dtype=torch.float32) -> TrainReport:
    """train_toy (toy.hpp:233-346) with every VSA forward/backward on the B200 operator."""
    task.check()
    if cfg.schedule is not None:
        cfg.schedule.check()
    L = task.layout
    H, d, md = task.heads, task.head_dim, task.model_dim()
    pc = H * d
    g = torch.Generator(device="cpu").manual_seed(cfg.seed)
    rnd = lambda *s: (torch.randn(*s, generator=g, dtype=torch.float64) / math.sqrt(md)).to(device, dtype)
    model = {"wq": rnd(md, pc), "wk": rnd(md, pc), "wv": rnd(md, pc),
             "gate_weight": torch.zeros(md, 2 * pc, device=device, dtype=dtype)}
    model["gate_weight"][md - 1, pc:] = 1.0  # pass-through: fine gate 1, coarse gate 0
    data = generate_batch(task, cfg.batch_size, cfg.seed + 0x9E3779B9, device, dtype)
    B, S = cfg.batch_size, L.seq_len
    fixed_sel = None
    if cfg.policy == "fixed_random":
        sg = np.random.Generator(np.random.PCG64(cfg.seed))
        fixed_sel = torch.from_numpy(np.stack([np.sort(sg.choice(L.num_cubes, cfg.top_k, replace=False))
                                               for _ in range(B * H * L.num_cubes)]).astype(np.int32)
                                     ).reshape(B, H, L.num_cubes, cfg.top_k).to(device)
    elif cfg.policy not in ("learned", "fixed_pattern"):
        raise ValueError("train_toy: policy must be 'learned', 'fixed_random' or 'fixed_pattern'")
    pattern_sel = {}
    if cfg.policy == "fixed_pattern":
        # spatial-temporal controls alternate phases across steps (toy.hpp:276-285)
        phases = (SPATIAL, TEMPORAL) if cfg.pattern.kind == SPATIAL_TEMPORAL else (cfg.pattern.phase,)
        for ph in phases:
            rows = fixed_pattern_selection(L, PatternSpec(cfg.pattern.kind, ph, cfg.pattern.window_s,
                                                          cfg.pattern.window_t))
            pattern_sel[ph] = torch.from_numpy(rows).to(device).expand(cfg.batch_size, H, *rows.shape).contiguous()
    adam = {n: (torch.zeros_like(w), torch.zeros_like(w)) for n, w in model.items()}
    ops = {}
    hid = data.hidden[:, 0]  # [B, S, md]
    n = B * H * S * d
    rep = TrainReport([], model)

    def heads(x):  # [B, S, H*d] -> [B, H, S, d]
        return x.view(B, S, H, d).permute(0, 2, 1, 3).contiguous()

    def packed(x):  # [B, H, S, d] -> [B, S, H*d]
        return x.permute(0, 2, 1, 3).reshape(B, S, pc)

    for step in range(cfg.steps):
        k_step = cfg.schedule.k_at(step) if cfg.schedule is not None else cfg.top_k
        k_step = min(max(k_step, 1), L.num_cubes)
        sel_override = fixed_sel
        if cfg.policy == "fixed_pattern":
            sel_override = pattern_sel[(SPATIAL, TEMPORAL)[step % 2]] if len(pattern_sel) == 2 \
                else next(iter(pattern_sel.values()))
        k_op = k_step if sel_override is None else sel_override.shape[-1]
        if k_op not in ops:
            ops[k_op] = VsaOp(L, B, H, d, k_op, dtype=dtype, pool=cfg.pool, raster=False, device=device)
        op = ops[k_op]
        q, k, v = (heads(hid @ model[w]) for w in ("wq", "wk", "wv"))
        z = hid @ model["gate_weight"]
        if cfg.activation == 1:
            z = torch.sigmoid(z)
        gc, gf = heads(z[..., :pc]), heads(z[..., pc:])
        out = op.forward(q, k, v, gc, gf, sel_override=sel_override)
        dout = out - data.target
        loss = float((dout.double() ** 2).sum()) / n
        recall = planted_recall(op.fine_sel, data.planted)
        rep.steps.append(TrainStep(step, loss, recall, k_step))
        if not math.isfinite(loss):
            rep.diverged = True
            break
        dq, dk, dv, dgc, dgf = op.backward((dout * (2.0 / n)).contiguous())
        dz = torch.cat([packed(dgc), packed(dgf)], dim=-1)
        if cfg.activation == 1:
            dz = dz * z * (1 - z)
        grads = {"wq": packed(dq), "wk": packed(dk), "wv": packed(dv), "gate_weight": dz}
        t = step + 1
        opt = cfg.optimizer
        for name, gr in grads.items():
            gw = torch.einsum("bsm,bsn->mn", hid, gr)
            w = model[name]
            if opt.kind == "sgd":
                w -= opt.lr * gw
                continue
            m, vv = adam[name]
            m.mul_(opt.beta1).add_(gw, alpha=1 - opt.beta1)
            vv.mul_(opt.beta2).addcmul_(gw, gw, value=1 - opt.beta2)
            bc1, bc2 = 1 - opt.beta1 ** t, 1 - opt.beta2 ** t
            w -= opt.lr * (m / bc1) / ((vv / bc2).sqrt() + opt.eps)
    h = 0xCBF29CE484222325
    for name in ("wq", "wk", "wv", "gate_weight"):
        # column-major bytes, as the reference hashes its Eigen matrices
        h = _fnv1a64(model[name].detach().t().contiguous().cpu().numpy().tobytes(), h)
    rep.snapshot_id = f"{h:016x}"
    return rep
