# SPDX-License-Identifier: Apache-2.0
"""Shared helpers for the GPU parity tests: reference-seeded inputs, the
oracle composition of the full operator on a (padded) raster problem, and the
north_star tolerances."""
from __future__ import annotations

import numpy as np
import torch

import oracle as orc

# north_star: bf16 I/O with fp32 accumulation within 2e-2 max-abs / 1e-2 relative;
# fp32 mode within 1e-4.
BF16_ATOL, BF16_RTOL = 2e-2, 1e-2
F32_TOL = 1e-4


def to_dev(a: np.ndarray, dtype) -> torch.Tensor:
    return torch.from_numpy(np.ascontiguousarray(a)).to("cuda").to(dtype).contiguous()


def rounded(a: np.ndarray, dtype) -> np.ndarray:
    """The values the GPU actually sees, as float32 (bf16 RNE rounding)."""
    if dtype == torch.float32:
        return np.ascontiguousarray(a, dtype=np.float32)
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).to(torch.bfloat16).float().numpy()


def host(t: torch.Tensor) -> np.ndarray:
    return t.float().cpu().numpy()


def assert_close(got: np.ndarray, ref: np.ndarray, dtype, what: str):
    got = np.asarray(got, np.float64)
    ref = np.asarray(ref, np.float64)
    assert got.shape == ref.shape, (what, got.shape, ref.shape)
    assert np.isfinite(got).all(), f"{what}: non-finite output"
    err = np.abs(got - ref)
    if dtype == torch.float32:
        bad = err > F32_TOL * np.maximum(1.0, np.abs(ref))
        assert not bad.any(), f"{what}: fp32 max err {err.max():.3e}"
    else:
        bad = err > BF16_ATOL + BF16_RTOL * np.abs(ref)
        rel = np.linalg.norm(got - ref) / max(np.linalg.norm(ref), 1e-30)
        assert not bad.any() and rel < BF16_RTOL, f"{what}: bf16 max abs {err.max():.3e}, rel {rel:.3e}"


class Problem:
    """A raster-ordered VSA problem drawn like the reference fixtures:
    q, k, v, gc, gf, dO from one std::mt19937_64 in that order."""

    def __init__(self, grid, B, H, d, top_k, seed=0, cube=(4, 4, 4), gate_std=1.0):
        self.grid, self.B, self.H, self.d, self.top_k, self.cube = grid, B, H, d, top_k, cube
        T, X, Y = grid
        self.S = T * X * Y
        rng = orc.Rng(seed)
        self.q, self.k, self.v = (orc.randn(rng, B, H, self.S, d, np.float32) for _ in range(3))
        self.gc = orc.randn(rng, B, H, self.S, d, np.float32, gate_std)
        self.gf = orc.randn(rng, B, H, self.S, d, np.float32, gate_std)
        self.dout = orc.randn(rng, B, H, self.S, d, np.float32)
        self.padded = orc.padded_extents(*grid, *cube)
        self.olayout = orc.TileLayout(*self.padded, *cube)

    def pad_tile(self, x):
        return orc.tile(self.olayout, orc.pad_raster(x, self.grid, self.padded))

    def untile_crop(self, xt):
        return orc.crop_raster(orc.untile(self.olayout, xt), self.grid, self.padded)

    def oracle(self, dtype, sel_override=None, backward=True, heads=None, pool=None):
        """Reference semantics on the zero-padded problem."""
        hs = slice(None) if heads is None else heads
        r = lambda a: rounded(a[:, hs], dtype)
        q, k, v, gc, gf, do = (self.pad_tile(r(x)) for x in (self.q, self.k, self.v, self.gc, self.gf, self.dout))
        L = self.olayout
        art = orc.coarse_forward_select(L, q, k, v, self.top_k, *(() if pool is None else (pool,)))
        sel = art.sel if sel_override is None else np.ascontiguousarray(sel_override[:, hs])
        fo, _, lse = orc.fine_forward(L, q, k, v, sel)
        out = art.oc * gc + fo * gf
        res = dict(art=art, sel=sel, fo=fo, lse=lse, out=self.untile_crop(out))
        if backward:
            doc, dof = do * gc, do * gf
            cdq, cdk, cdv = orc.coarse_backward(art, L, doc, q, k, v)
            fdq, fdk, fdv = orc.fine_backward(L, q, k, v, sel, dof, lse)
            res.update(dq=self.untile_crop(cdq + fdq), dk=self.untile_crop(cdk + fdk),
                       dv=self.untile_crop(cdv + fdv), dgc=self.untile_crop(do * art.oc),
                       dgf=self.untile_crop(do * fo))
        return res
