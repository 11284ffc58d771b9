# SPDX-License-Identifier: Apache-2.0
"""FLOP accounting of the reference's analysis module (analysis.hpp:29-75,
analysis.cpp:16-42): 6·N·D for the backbone plus 4·D·S·A·H·3.5·layers for attention,
scaled by the block density for VSA, plus the pooled coarse term. Host arithmetic only
(used to report model-level savings next to the kernel-level FLOP counts of bench.py).
The schedule and fixed-pattern helpers of the same module live in ``toy.py``."""
from __future__ import annotations

import json
from dataclasses import dataclass

FULL, VSA = 0, 1  # AttentionMode


def sparsity_density(k: int, block: int, seq_len: int) -> float:
    """Density K·B/L of a block-sparse selection (analysis.hpp:70-72)."""
    return float(k) * float(block) / float(seq_len)


@dataclass
class FlopsConfig:
    n_params: float = 0.0
    n_tokens: float = 0.0
    seq_len: float = 0.0
    n_heads: float = 0.0
    head_dim: float = 0.0
    n_layers: float = 0.0
    density: float = 1.0
    block_size: float = 64.0

    def check(self):
        if not all(x > 0 for x in (self.n_params, self.n_tokens, self.seq_len, self.n_heads, self.head_dim,
                                   self.n_layers, self.block_size)):
            raise ValueError("FlopsConfig: all quantities must be positive")
        if not (0 < self.density <= 1.0):
            raise ValueError("FlopsConfig: density must be in (0, 1]")


@dataclass
class FlopsReport:
    model_flops: float = 0.0
    attention_flops: float = 0.0
    coarse_flops: float = 0.0
    total: float = 0.0
    density: float = 1.0

    def to_json(self) -> str:  # keys in a stable order (analysis.cpp:36-43)
        return json.dumps({"model_flops": self.model_flops, "attention_flops": self.attention_flops,
                           "coarse_flops": self.coarse_flops, "total": self.total, "density": self.density})


def compute_flops(cfg: FlopsConfig, mode: int) -> FlopsReport:
    """compute_flops (analysis.cpp:16-34)."""
    cfg.check()
    r = FlopsReport(model_flops=6.0 * cfg.n_params * cfg.n_tokens)
    full = 4.0 * cfg.n_tokens * cfg.seq_len * cfg.n_heads * cfg.head_dim * 3.5 * cfg.n_layers
    if mode == FULL:
        r.attention_flops, r.coarse_flops, r.density = full, 0.0, 1.0
    else:
        r.attention_flops = full * cfg.density
        r.coarse_flops = full / (cfg.block_size * cfg.block_size)  # pooled: tokens and keys shrink by B
        r.density = cfg.density
    r.total = r.model_flops + r.attention_flops + r.coarse_flops
    return r
