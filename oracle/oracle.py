# SPDX-License-Identifier: Apache-2.0
"""TEST INFRASTRUCTURE ONLY — the CPU parity oracle.

ctypes front-end over ``oracle/_build/liboracle.so`` (the plain-loop C++
restatement in ``vsa_oracle.cpp``) plus numpy restatements of the operator-level
glue in ``/root/reference/proj/include/vsa/vsa.hpp`` (gate projection, combine,
joint backward). Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
CPU-baseline leg may import this module, and only as the checker.

Names follow the reference API (``proj/include/vsa/*.hpp``); precondition
failures raise ``ValueError`` where the reference throws ``std::invalid_argument``.
Tensors are numpy arrays ``[batch, heads, seq, dim]`` (AttnTensor, tensor.hpp:44-123).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "_build", "liboracle.so")

KMEAN, KMAX = 0, 1  # PoolMode (coarse.hpp:13)


def build() -> str:
    """Compile the restatement (make in oracle/)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _SO


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_SO):
            build()
        L = C.CDLL(_SO)
        L.orc_last_error.restype = C.c_char_p
        L.orc_canon_exp.restype = C.c_double
        L.orc_canon_exp.argtypes = [C.c_double]
        L.orc_rng_new.restype = C.c_void_p
        L.orc_rng_new.argtypes = [C.c_uint64]
        L.orc_rng_free.argtypes = [C.c_void_p]
        L.orc_rng_randn.argtypes = [C.c_void_p, C.c_int64, C.c_double, C.c_void_p]
        L.orc_rng_uniform_int.restype = C.c_int64
        L.orc_rng_uniform_int.argtypes = [C.c_void_p, C.c_int64, C.c_int64]
        L.orc_rng_uniform_size.restype = C.c_uint64
        L.orc_rng_uniform_size.argtypes = [C.c_void_p, C.c_uint64, C.c_uint64]
        L.orc_rng_uniform_int32.restype = C.c_int
        L.orc_rng_uniform_int32.argtypes = [C.c_void_p, C.c_int, C.c_int]
        L.orc_rng_uniform_real.restype = C.c_double
        L.orc_rng_uniform_real.argtypes = [C.c_void_p, C.c_double, C.c_double]
        L.orc_rng_bernoulli.restype = C.c_int
        L.orc_rng_bernoulli.argtypes = [C.c_void_p, C.c_double]
        L.orc_rng_shuffle.argtypes = [C.c_void_p, C.c_void_p, C.c_int64]
        L.orc_rng_random_selection.argtypes = [C.c_void_p] + [C.c_int64] * 4 + [C.c_void_p]
        L.orc_max_threads.restype = C.c_int
        _lib = L
    return _lib


def _p(a):
    return None if a is None else C.c_void_p(a.ctypes.data)


def _check(rc):
    if rc != 0:
        msg = lib().orc_last_error().decode()
        if rc == -1:
            raise ValueError(msg)
        raise RuntimeError(msg)


def _suf(dtype):
    if dtype == np.float32:
        return "f32"
    if dtype == np.float64:
        return "f64"
    raise TypeError(f"oracle supports float32/float64, got {dtype}")


def _c(a, dtype=None):
    a = np.ascontiguousarray(a if dtype is None else a.astype(dtype, copy=False))
    return a


def set_num_threads(n: int) -> None:
    lib().orc_set_num_threads(int(n))


def max_threads() -> int:
    return lib().orc_max_threads()


def canon_exp(x: float) -> float:
    return lib().orc_canon_exp(float(x))


# ----------------------------------------------------------------------------- RNG
class Rng:
    """std::mt19937_64 plus the libstdc++ distributions the reference tests use."""

    def __init__(self, seed: int):
        self._h = lib().orc_rng_new(C.c_uint64(seed))

    def __del__(self):
        try:
            lib().orc_rng_free(self._h)
        except Exception:
            pass

    def normal(self, n: int, stddev: float = 1.0) -> np.ndarray:
        out = np.empty(int(n), np.float64)
        lib().orc_rng_randn(self._h, int(n), float(stddev), _p(out))
        return out

    def uniform_int(self, a: int, b: int) -> int:  # uniform_int_distribution<Index>
        return int(lib().orc_rng_uniform_int(self._h, a, b))

    def uniform_size(self, a: int, b: int) -> int:  # uniform_int_distribution<size_t>
        return int(lib().orc_rng_uniform_size(self._h, a, b))

    def uniform_int32(self, a: int, b: int) -> int:  # uniform_int_distribution<int>
        return int(lib().orc_rng_uniform_int32(self._h, a, b))

    def uniform_real(self, a: float, b: float) -> float:
        return float(lib().orc_rng_uniform_real(self._h, a, b))

    def bernoulli(self, p: float) -> bool:
        return bool(lib().orc_rng_bernoulli(self._h, p))

    def shuffle(self, arr: np.ndarray) -> None:
        assert arr.dtype == np.int64 and arr.flags.c_contiguous
        lib().orc_rng_shuffle(self._h, _p(arr), arr.size)


def randn(rng: Rng, B, H, S, D, dtype=np.float64, stddev=1.0) -> np.ndarray:
    """AttnTensor<Scalar>::randn (tensor.hpp:62-68)."""
    return rng.normal(B * H * S * D, stddev).astype(dtype).reshape(B, H, S, D)


def randn_matrix(rng: Rng, rows, cols, dtype=np.float64, stddev=1.0) -> np.ndarray:
    """randn_matrix (tensor.hpp:126-133)."""
    return rng.normal(rows * cols, stddev).astype(dtype).reshape(rows, cols)


# ----------------------------------------------------------------------------- layout
@dataclass
class TileLayout:
    """vsa::TileLayout (layout.hpp:14-33, layout.cpp:6-31)."""

    tokens_t: int
    tokens_h: int
    tokens_w: int
    cube_t: int
    cube_h: int
    cube_w: int
    cubes_t: int = field(init=False)
    cubes_h: int = field(init=False)
    cubes_w: int = field(init=False)
    cube_size: int = field(init=False)
    seq_len: int = field(init=False)
    num_cubes: int = field(init=False)

    def __post_init__(self):
        out = (C.c_int64 * 6)()
        _check(lib().orc_layout(*[C.c_int64(v) for v in self.args()], out))
        self.cubes_t, self.cubes_h, self.cubes_w, self.cube_size, self.seq_len, self.num_cubes = list(out)

    def args(self):
        return (self.tokens_t, self.tokens_h, self.tokens_w, self.cube_t, self.cube_h, self.cube_w)

    def cargs(self):
        return [C.c_int64(v) for v in self.args()]

    def tile_of_raster(self) -> np.ndarray:
        out = np.empty(self.seq_len, np.int64)
        _check(lib().orc_tile_of_raster(*self.cargs(), _p(out)))
        return out


def raster_index(layout: TileLayout, t, h, w) -> int:
    if not (0 <= t < layout.tokens_t and 0 <= h < layout.tokens_h and 0 <= w < layout.tokens_w):
        raise ValueError("raster_index: coordinate out of range")
    return (t * layout.tokens_h + h) * layout.tokens_w + w


def flatten_index(layout: TileLayout, t, h, w) -> int:
    out = C.c_int64()
    _check(lib().orc_flatten_index(*layout.cargs(), C.c_int64(t), C.c_int64(h), C.c_int64(w), C.byref(out)))
    return out.value


def _tile(layout, x, inverse):
    x = _c(x)
    out = np.empty_like(x)
    B, H, S, D = x.shape
    _check(getattr(lib(), "orc_tile_" + _suf(x.dtype))(*layout.cargs(), _p(x), C.c_int64(B * H), C.c_int64(S),
                                                       C.c_int64(D), C.c_int(int(inverse)), _p(out)))
    return out


def tile(layout, x):
    """tile<S> (layout.hpp:43-55)."""
    return _tile(layout, x, False)


def untile(layout, x):
    """untile<S> (layout.hpp:58-70)."""
    return _tile(layout, x, True)


def padded_extents(t, h, w, ct, ch, cw):
    """Zero-pad extension: extents rounded up to cube multiples."""
    up = lambda a, c: (a + c - 1) // c * c
    return up(t, ct), up(h, ch), up(w, cw)


def pad_raster(x, grid, padded):
    """Zero-pad a raster-ordered [B,H,T*X*Y,D] tensor to the padded grid."""
    B, H, S, D = x.shape
    T, X, Y = grid
    Tp, Xp, Yp = padded
    out = np.zeros((B, H, Tp, Xp, Yp, D), x.dtype)
    out[:, :, :T, :X, :Y] = x.reshape(B, H, T, X, Y, D)
    return out.reshape(B, H, Tp * Xp * Yp, D)


def crop_raster(x, grid, padded):
    B, H, S, D = x.shape
    T, X, Y = grid
    Tp, Xp, Yp = padded
    return np.ascontiguousarray(x.reshape(B, H, Tp, Xp, Yp, D)[:, :, :T, :X, :Y].reshape(B, H, T * X * Y, D))


# ----------------------------------------------------------------------------- selection
def all_cubes(B, H, nc) -> np.ndarray:
    """BlockSelection::all_cubes (selection.cpp:13-22)."""
    return np.ascontiguousarray(np.broadcast_to(np.arange(nc, dtype=np.int32), (B, H, nc, nc)))


def random_selection(B, H, nc, k, rng: Rng) -> np.ndarray:
    """random_selection (selection.cpp:52-70)."""
    out = np.empty((B, H, nc, k), np.int32)
    _check(lib().orc_rng_random_selection(rng._h, B, H, nc, k, _p(out)))
    return out


def validate(sel: np.ndarray) -> None:
    """BlockSelection::validate (selection.cpp:24-37)."""
    sel = _c(sel, np.int32)
    if sel.size == 0:
        raise ValueError("BlockSelection: empty selection")
    B, H, nc, k = sel.shape
    _check(lib().orc_validate_selection(_p(sel), C.c_int64(B), C.c_int64(H), C.c_int64(nc), C.c_int64(k)))


def selection_to_mask(layout: TileLayout, sel: np.ndarray, b: int) -> np.ndarray:
    """selection_to_mask (selection.cpp:72-85): uint8 [H, L, L]."""
    B, H, nc, k = sel.shape
    if nc != layout.num_cubes:
        raise ValueError("selection_to_mask: selection does not match layout")
    cb = layout.cube_size
    m = np.zeros((H, layout.seq_len, layout.seq_len), np.uint8)
    for h in range(H):
        for qc in range(nc):
            for kc in sel[b, h, qc]:
                m[h, qc * cb:(qc + 1) * cb, kc * cb:(kc + 1) * cb] = 1
    return m


# ----------------------------------------------------------------------------- coarse
def topk_row(values: np.ndarray, k: int) -> np.ndarray:
    """topk_row (coarse.hpp:30-42)."""
    values = _c(values)
    out = np.empty(k, np.int32)
    _check(getattr(lib(), "orc_topk_row_" + _suf(values.dtype))(_p(values), C.c_int64(values.size), C.c_int64(k),
                                                               _p(out)))
    return out


def pool_cubes(layout, x, mode=KMEAN):
    """pool_cubes (coarse.hpp:47-65); mean = sequential sum / B (canonical order)."""
    x = _c(x)
    B, H, S, D = x.shape
    out = np.empty((B, H, layout.num_cubes, D), x.dtype)
    _check(getattr(lib(), "orc_pool_" + _suf(x.dtype))(*layout.cargs(), _p(x), C.c_int64(B * H), C.c_int64(S),
                                                       C.c_int64(D), C.c_int(mode), _p(out)))
    return out


@dataclass
class CoarseArtifacts:
    """CoarseArtifacts (coarse.hpp:18-25); oc_cube is the cube-level Oc."""

    qc: np.ndarray
    kc: np.ndarray
    vc: np.ndarray
    ac: np.ndarray
    oc: np.ndarray
    oc_cube: np.ndarray
    sel: np.ndarray
    pool: int = KMEAN


def coarse_forward_select(layout, q, k, v, top_k, mode=KMEAN, token_oc=True) -> CoarseArtifacts:
    """coarse_forward_select (coarse.hpp:71-117)."""
    q, k, v = _c(q), _c(k), _c(v)
    if q.size == 0:
        raise ValueError("attention: empty tensors")
    if not (q.shape == k.shape == v.shape):
        raise ValueError("attention: Q, K, V must share one shape")
    B, H, S, D = q.shape
    nc = layout.num_cubes
    dt = q.dtype
    qc, kc, vc = (np.empty((B, H, nc, D), dt) for _ in range(3))
    ac = np.empty((B, H, nc, nc), dt)
    oc_cube = np.empty((B, H, nc, D), dt)
    oc = np.empty((B, H, S, D), dt) if token_oc else None
    sel = np.empty((B, H, nc, max(int(top_k), 1)), np.int32)
    _check(getattr(lib(), "orc_coarse_forward_" + _suf(dt))(
        *layout.cargs(), _p(q), _p(k), _p(v), C.c_int64(B), C.c_int64(H), C.c_int64(S), C.c_int64(D),
        C.c_int64(top_k), C.c_int(mode), _p(qc), _p(kc), _p(vc), _p(ac), _p(oc_cube), _p(oc), _p(sel)))
    return CoarseArtifacts(qc, kc, vc, ac, oc, oc_cube, sel, mode)


def coarse_backward(art: CoarseArtifacts, layout, doc, q, k, v, cube_grads=False):
    """coarse_backward (coarse.hpp:124-184) -> (dq, dk, dv) token level."""
    q, k, v, doc = _c(q), _c(k), _c(v), _c(doc)
    if doc.shape != q.shape:
        raise ValueError("coarse_backward: dOc shape mismatch")
    if art.ac is None or art.ac.size == 0 or art.ac.shape[2] != layout.num_cubes:
        raise ValueError("coarse_backward: artifacts do not match layout")
    B, H, S, D = q.shape
    dq, dk, dv = (np.empty_like(q) for _ in range(3))
    nc = layout.num_cubes
    cg = [np.empty((B, H, nc, D), q.dtype) for _ in range(3)] if cube_grads else [None] * 3
    _check(getattr(lib(), "orc_coarse_backward_" + _suf(q.dtype))(
        *layout.cargs(), _p(q), _p(k), _p(v), _p(art.qc), _p(art.kc), _p(art.vc), _p(art.ac), C.c_int(art.pool),
        _p(doc), C.c_int64(B), C.c_int64(H), C.c_int64(S), C.c_int64(D), _p(dq), _p(dk), _p(dv), _p(cg[0]),
        _p(cg[1]), _p(cg[2])))
    return (dq, dk, dv, *cg) if cube_grads else (dq, dk, dv)


# ----------------------------------------------------------------------------- dense
def _mask_arg(mask, H, S):
    if mask is None:
        return None, 0
    m = _c(mask, np.uint8)
    if m.ndim == 2:
        m = m[None]
    if m.shape[1] != S or m.shape[2] != S:
        raise ValueError("attention: mask size does not match sequence length")
    if m.shape[0] not in (1, H):
        raise ValueError("attention: mask head count must be 1 or match heads")
    return np.ascontiguousarray(m), m.shape[0]


def dense_forward(q, k, v, mask=None):
    """dense_forward (dense.hpp:94-148) -> (out, row_max, row_lse); stats [B*H, S]."""
    q, k, v = _c(q), _c(k), _c(v)
    if q.size == 0:
        raise ValueError("attention: empty tensors")
    if not (q.shape == k.shape == v.shape):
        raise ValueError("attention: Q, K, V must share one shape")
    B, H, S, D = q.shape
    m, mh = _mask_arg(mask, H, S)
    out = np.empty_like(q)
    rmax = np.empty((B * H, S), q.dtype)
    lse = np.empty((B * H, S), q.dtype)
    _check(getattr(lib(), "orc_dense_forward_" + _suf(q.dtype))(
        _p(q), _p(k), _p(v), C.c_int64(B), C.c_int64(H), C.c_int64(S), C.c_int64(D), _p(m), C.c_int64(mh),
        _p(out), _p(rmax), _p(lse)))
    return out, rmax, lse


def dense_backward(q, k, v, mask, dout, row_lse):
    """dense_backward (dense.hpp:155-209) -> (dq, dk, dv)."""
    q, k, v, dout, row_lse = _c(q), _c(k), _c(v), _c(dout), _c(row_lse)
    B, H, S, D = q.shape
    if dout.shape != q.shape:
        raise ValueError("dense_backward: dO shape mismatch")
    if row_lse.shape != (B * H, S):
        raise ValueError("dense_backward: saved statistics do not match shapes")
    m, mh = _mask_arg(mask, H, S)
    dq, dk, dv = (np.empty_like(q) for _ in range(3))
    _check(getattr(lib(), "orc_dense_backward_" + _suf(q.dtype))(
        _p(q), _p(k), _p(v), C.c_int64(B), C.c_int64(H), C.c_int64(S), C.c_int64(D), _p(m), C.c_int64(mh),
        _p(dout), _p(row_lse), _p(dq), _p(dk), _p(dv)))
    return dq, dk, dv


# ----------------------------------------------------------------------------- fine
def _check_qkv(q, k, v):
    if q.size == 0:
        raise ValueError("attention: empty tensors")
    if not (q.shape == k.shape == v.shape):
        raise ValueError("attention: Q, K, V must share one shape")


def fine_forward(layout, q, k, v, sel):
    """fine_forward (fine.hpp:43-99) -> (out, row_max, row_lse)."""
    q, k, v, sel = _c(q), _c(k), _c(v), _c(sel, np.int32)
    _check_qkv(q, k, v)
    B, H, S, D = q.shape
    sb, sh, snc, kk = sel.shape
    out = np.empty_like(q)
    rmax = np.empty((B * H, S), q.dtype)
    lse = np.empty((B * H, S), q.dtype)
    _check(getattr(lib(), "orc_fine_forward_" + _suf(q.dtype))(
        *layout.cargs(), _p(q), _p(k), _p(v), C.c_int64(B), C.c_int64(H), C.c_int64(S), C.c_int64(D), _p(sel),
        C.c_int64(sb), C.c_int64(sh), C.c_int64(snc), C.c_int64(kk), _p(out), _p(rmax), _p(lse)))
    return out, rmax, lse


def fine_backward(layout, q, k, v, sel, dout, row_lse, return_delta=False):
    """fine_backward (fine.hpp:107-204) -> (dq, dk, dv[, delta])."""
    q, k, v, sel, dout, row_lse = _c(q), _c(k), _c(v), _c(sel, np.int32), _c(dout), _c(row_lse)
    _check_qkv(q, k, v)
    B, H, S, D = q.shape
    if dout.shape != q.shape:
        raise ValueError("fine_backward: dO shape mismatch")
    if row_lse.shape != (B * H, S):
        raise ValueError("fine_backward: saved statistics do not match shapes")
    sb, sh, snc, kk = sel.shape
    dq, dk, dv = (np.empty_like(q) for _ in range(3))
    delta = np.empty((B * H, S), q.dtype)
    _check(getattr(lib(), "orc_fine_backward_" + _suf(q.dtype))(
        *layout.cargs(), _p(q), _p(k), _p(v), C.c_int64(B), C.c_int64(H), C.c_int64(S), C.c_int64(D), _p(sel),
        C.c_int64(sb), C.c_int64(sh), C.c_int64(snc), C.c_int64(kk), _p(dout), _p(row_lse), _p(dq), _p(dk),
        _p(dv), _p(delta)))
    return (dq, dk, dv, delta) if return_delta else (dq, dk, dv)


# ----------------------------------------------------------------------------- VSA operator
IDENTITY, SIGMOID = 0, 1  # GateActivation (vsa.hpp:9)


@dataclass
class VsaParams:
    """VsaParams (vsa.hpp:16-52)."""

    gate_weight: np.ndarray  # [model_dim, 2*H*d]
    gate_bias: np.ndarray | None = None
    top_k: int = 1
    pool: int = KMEAN
    activation: int = IDENTITY
    adaptation: bool = False

    @staticmethod
    def random_init(model_dim, heads, head_dim, top_k, rng: Rng, dtype=np.float64):
        w = randn_matrix(rng, model_dim, 2 * heads * head_dim, dtype, 1.0 / np.sqrt(float(model_dim)))
        return VsaParams(w, None, top_k)

    @staticmethod
    def adaptation_init(model_dim, heads, head_dim, num_cubes, dtype=np.float64):
        return VsaParams(np.zeros((model_dim, 2 * heads * head_dim), dtype), None, num_cubes, adaptation=True)

    def check(self, model_dim, heads, head_dim):
        if self.gate_weight.shape != (model_dim, 2 * heads * head_dim):
            raise ValueError("VsaParams: gate projection must map model_dim -> 2*heads*head_dim")
        if self.gate_bias is not None and self.gate_bias.size not in (0, self.gate_weight.shape[1]):
            raise ValueError("VsaParams: gate bias size mismatch")
        if self.top_k < 1:
            raise ValueError("VsaParams: k must be >= 1")


@dataclass
class VsaOutput:
    """VsaOutput (vsa.hpp:56-63)."""

    out: np.ndarray
    coarse: CoarseArtifacts
    fine_out: np.ndarray
    fine_row_max: np.ndarray
    fine_row_lse: np.ndarray
    gate_coarse: np.ndarray
    gate_fine: np.ndarray
    fine_sel: np.ndarray


def gates_from_hidden(hidden, params: VsaParams, heads, dim):
    """Gate projection + split (vsa.hpp:100-112)."""
    B, _, S, md = hidden.shape
    dt = hidden.dtype
    gc = np.empty((B, heads, S, dim), dt)
    gf = np.empty((B, heads, S, dim), dt)
    for b in range(B):
        z = hidden[b, 0] @ params.gate_weight
        if params.gate_bias is not None and params.gate_bias.size:
            z = z + params.gate_bias.reshape(1, -1)
        if params.activation == SIGMOID:
            z = 1.0 / (1.0 + np.exp(-z))
        for h in range(heads):
            gc[b, h] = z[:, h * dim:(h + 1) * dim]
            gf[b, h] = z[:, (heads + h) * dim:(heads + h + 1) * dim]
    if params.adaptation:
        gf[...] = 1
    return gc, gf


def vsa_forward(layout, hidden, q, k, v, params: VsaParams, sel_override=None) -> VsaOutput:
    """vsa_forward (vsa.hpp:89-122)."""
    _check_qkv(q, k, v)
    if hidden.shape[1] != 1:
        raise ValueError("vsa: hidden states are [batch, 1, seq, model_dim]")
    if hidden.shape[0] != q.shape[0] or hidden.shape[2] != q.shape[2]:
        raise ValueError("vsa: hidden states do not match Q/K/V shapes")
    B, H, S, D = q.shape
    params.check(hidden.shape[3], H, D)
    gc, gf = gates_from_hidden(hidden, params, H, D)
    art = coarse_forward_select(layout, q, k, v, params.top_k, params.pool)
    fsel = art.sel if sel_override is None else sel_override
    fo, fmax, flse = fine_forward(layout, q, k, v, fsel)
    out = art.oc * gc + fo * gf
    return VsaOutput(out, art, fo, fmax, flse, gc, gf, fsel)


@dataclass
class VsaGrads:
    dq: np.ndarray
    dk: np.ndarray
    dv: np.ndarray
    dhidden: np.ndarray
    dgate_weight: np.ndarray
    dgate_bias: np.ndarray | None
    dgate_coarse: np.ndarray  # dL/dGc (post-activation), the attention-level gate grads
    dgate_fine: np.ndarray


def vsa_backward(layout, fwd: VsaOutput, hidden, q, k, v, params: VsaParams, dout) -> VsaGrads:
    """vsa_backward (vsa.hpp:129-189)."""
    _check_qkv(q, k, v)
    if dout.shape != q.shape:
        raise ValueError("vsa_backward: dO shape mismatch")
    if fwd is None or fwd.out is None or fwd.out.shape != q.shape or fwd.fine_sel is None or fwd.fine_sel.size == 0:
        raise ValueError("vsa_backward: missing or mismatched forward artifacts")
    B, H, S, D = q.shape
    params.check(hidden.shape[3], H, D)
    doc = dout * fwd.gate_coarse
    dof = dout * fwd.gate_fine
    dgc = dout * fwd.coarse.oc
    dgf = np.zeros_like(dout) if params.adaptation else dout * fwd.fine_out
    md = hidden.shape[3]
    dhidden = np.empty((B, 1, S, md), q.dtype)
    dW = np.zeros_like(params.gate_weight)
    db = None if params.gate_bias is None or params.gate_bias.size == 0 else np.zeros_like(params.gate_bias)
    for b in range(B):
        dz = np.empty((S, 2 * H * D), q.dtype)
        for h in range(H):
            dz[:, h * D:(h + 1) * D] = dgc[b, h]
            dz[:, (H + h) * D:(H + h + 1) * D] = dgf[b, h]
        if params.activation == SIGMOID:
            for h in range(H):
                g = fwd.gate_coarse[b, h]
                dz[:, h * D:(h + 1) * D] *= g * (1 - g)
                if not params.adaptation:
                    g = fwd.gate_fine[b, h]
                    dz[:, (H + h) * D:(H + h + 1) * D] *= g * (1 - g)
        dhidden[b, 0] = dz @ params.gate_weight.T
        dW += hidden[b, 0].T @ dz
        if db is not None:
            db += dz.sum(axis=0).reshape(db.shape)
    cdq, cdk, cdv = coarse_backward(fwd.coarse, layout, doc, q, k, v)
    fdq, fdk, fdv = fine_backward(layout, q, k, v, fwd.fine_sel, dof, fwd.fine_row_lse)
    return VsaGrads(cdq + fdq, cdk + fdk, cdv + fdv, dhidden, dW, db, dgc, dgf)


# ----------------------------------------------------------------------------- gradcheck helpers
def fd_gradient(data: np.ndarray, step: float, loss) -> np.ndarray:
    """fd_gradient (gradcheck.hpp:13-26): central differences, in place over `data`."""
    flat = data.reshape(-1)
    g = np.empty(flat.size)
    for i in range(flat.size):
        saved = flat[i]
        flat[i] = saved + step
        up = loss()
        flat[i] = saved - step
        down = loss()
        flat[i] = saved
        g[i] = (up - down) / (2.0 * step)
    return g.reshape(data.shape)


def max_rel_err(a, f) -> float:
    """max_rel_err (gradcheck.hpp:30-37)."""
    a = np.asarray(a, np.float64).reshape(-1)
    f = np.asarray(f, np.float64).reshape(-1)
    den = np.maximum(np.maximum(np.abs(a), np.abs(f)), 1.0)
    return float(np.max(np.abs(a - f) / den)) if a.size else 0.0


# ----------------------------------------------------------------------------- selection analytics
def dense_probs(q, k):
    """dense_probs (dense.hpp:214-240): row-stochastic [B,H,S,S] attention probabilities
    (no mask), max-subtracted exp / row sum, float64 here."""
    q = np.asarray(q, np.float64)
    k = np.asarray(k, np.float64)
    d = q.shape[-1]
    s = np.einsum("bhid,bhjd->bhij", q, k) * (1.0 / np.sqrt(d))
    s = np.exp(s - s.max(axis=-1, keepdims=True))
    return s / s.sum(axis=-1, keepdims=True)


def aggregate_probs_to_cubes(layout, probs_token):
    """aggregate_probs_to_cubes (analysis.hpp:130-147): [..,S,S] tile-ordered -> [..,S,nc]."""
    B, H, S, S2 = probs_token.shape
    if S != layout.seq_len or S2 != layout.seq_len:
        raise ValueError("aggregate_probs_to_cubes: expected [.., seq, seq] probabilities")
    return probs_token.reshape(B, H, S, layout.num_cubes, layout.cube_size).sum(axis=-1)


def selection_accuracy(layout, probs_cube, sel):
    """selection_accuracy (analysis.hpp:100-125): captured attention mass of the selected
    cubes, averaged over query tokens, per (b, h) -> float64 [B, H]."""
    B, H, S, nc = probs_cube.shape
    if S != layout.seq_len or nc != layout.num_cubes:
        raise ValueError("selection_accuracy: probabilities do not match layout")
    if sel.shape[:3] != (B, H, nc):
        raise ValueError("selection_accuracy: selection does not match shapes")
    cube = layout.cube_size
    qcube = np.arange(S) // cube
    acc = np.empty((B, H), np.float64)
    for b in range(B):
        for h in range(H):
            rows = sel[b, h][qcube]  # [S, K] selected cubes of each token's query cube
            acc[b, h] = np.take_along_axis(probs_cube[b, h].astype(np.float64), rows, axis=1).sum() / S
    return acc
