# SPDX-License-Identifier: Apache-2.0
"""Host-side mirror of the reference VSA API over the B200 C ABI.

Names, argument meaning and error behaviour follow /root/reference/proj/include/vsa:
``TileLayout`` (layout.hpp:14-33), ``tile``/``untile`` (layout.hpp:43-70),
``pool_cubes`` / ``coarse_forward_select`` / ``coarse_backward`` (coarse.hpp),
``fine_forward`` / ``fine_backward`` (fine.hpp), ``vsa_forward`` /
``vsa_backward`` (vsa.hpp). Tensors are CUDA ``torch.Tensor``s ``[B, H, S, d]``
(``AttnTensor``, tensor.hpp:44-123) in bf16 (tcgen05 path) or fp32 (parity
mode). torch is used only for device memory and the current stream; all
compute is in libvsa_b200.so. Precondition failures raise ``ValueError``
(the reference's ``std::invalid_argument``).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import torch

from . import _lib as L
from ._lib import check

POOL_MEAN, POOL_MAX = L.POOL_MEAN, L.POOL_MAX
GATE_IDENTITY, GATE_SIGMOID = 0, 1


def _p(t):
    return None if t is None else C.c_void_p(t.data_ptr())


def _stream():
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def _dt(t: torch.Tensor) -> int:
    if t.dtype == torch.bfloat16:
        return L.VSA_BF16
    if t.dtype == torch.float32:
        return L.VSA_F32
    raise ValueError(f"unsupported dtype {t.dtype} (bf16 or fp32)")


def _cuda4(t: torch.Tensor, name: str) -> None:
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise ValueError(f"{name}: expected a CUDA tensor")
    if t.dim() != 4:
        raise ValueError(f"{name}: expected [batch, heads, seq, head_dim]")
    if not t.is_contiguous():
        raise ValueError(f"{name}: must be contiguous")


# ----------------------------------------------------------------------------- layout
class TileLayout:
    """vsa::TileLayout (layout.hpp:14-33). ``pad=True`` enables the zero-pad
    extension for non-divisible grids (the reference rejects them, layout.cpp:10-11)."""

    def __init__(self, tokens_t, tokens_h, tokens_w, cube_t=4, cube_h=4, cube_w=4, pad=False):
        self._raw = L.vsa_layout_t()
        check(L.lib().vsa_layout_make(tokens_t, tokens_h, tokens_w, cube_t, cube_h, cube_w,
                                      L.PAD_ZERO if pad else L.PAD_REJECT, C.byref(self._raw)))

    def ref(self):
        return C.byref(self._raw)

    tokens_t = property(lambda s: s._raw.t)
    tokens_h = property(lambda s: s._raw.h)
    tokens_w = property(lambda s: s._raw.w)
    cube_t = property(lambda s: s._raw.ct)
    cube_h = property(lambda s: s._raw.ch)
    cube_w = property(lambda s: s._raw.cw)
    cubes_t = property(lambda s: s._raw.nt)
    cubes_h = property(lambda s: s._raw.nh)
    cubes_w = property(lambda s: s._raw.nw)
    cube_size = property(lambda s: s._raw.cube)
    num_cubes = property(lambda s: s._raw.nc)
    seq_len = property(lambda s: s._raw.seq)            # raster tokens
    seq_padded = property(lambda s: s._raw.seq_padded)  # tiled tokens (== seq_len unless padded)
    padded = property(lambda s: (s._raw.tp, s._raw.hp, s._raw.wp))

    def __repr__(self):
        r = self._raw
        return (f"TileLayout(({r.t},{r.h},{r.w}) cube ({r.ct},{r.ch},{r.cw}) -> padded ({r.tp},{r.hp},{r.wp}), "
                f"nc={r.nc}, L={r.seq}, Lp={r.seq_padded})")


def flatten_index(layout: TileLayout, t: int, h: int, w: int) -> int:
    """flatten_index (layout.cpp:40-42)."""
    out = C.c_int64()
    check(L.lib().vsa_flatten_index(layout.ref(), t, h, w, C.byref(out)))
    return out.value


def tile(layout: TileLayout, x: torch.Tensor) -> torch.Tensor:
    """tile<S> (layout.hpp:43-55): raster -> cube order (zero-padded)."""
    _cuda4(x, "tile")
    if x.shape[2] != layout.seq_len:
        raise ValueError("tile: sequence length does not match layout")
    B, H, _, d = x.shape
    out = torch.empty((B, H, layout.seq_padded, d), dtype=x.dtype, device=x.device)
    check(L.lib().vsa_tile(layout.ref(), B * H, d, _dt(x), _p(x), _p(out), _stream()))
    return out


def untile(layout: TileLayout, x: torch.Tensor) -> torch.Tensor:
    """untile<S> (layout.hpp:58-70): cube order -> raster (padded rows dropped)."""
    _cuda4(x, "untile")
    if x.shape[2] != layout.seq_padded:
        raise ValueError("untile: sequence length does not match layout")
    B, H, _, d = x.shape
    out = torch.empty((B, H, layout.seq_len, d), dtype=x.dtype, device=x.device)
    check(L.lib().vsa_untile(layout.ref(), B * H, d, _dt(x), _p(x), _p(out), _stream()))
    return out


def pool_cubes(layout: TileLayout, x: torch.Tensor, mode: int = POOL_MEAN) -> torch.Tensor:
    """pool_cubes (coarse.hpp:47-65) on a tile-ordered tensor -> fp32 [B,H,nc,d]."""
    _cuda4(x, "pool_cubes")
    if x.shape[2] != layout.seq_padded:
        raise ValueError("pool_cubes: sequence length does not match layout")
    B, H, _, d = x.shape
    out = torch.empty((B, H, layout.num_cubes, d), dtype=torch.float32, device=x.device)
    check(L.lib().vsa_pool_tiled(layout.ref(), B * H, d, _dt(x), _p(x), _p(out), mode, _stream()))
    return out


def tile_pool(layout: TileLayout, xs, mode: int = POOL_MEAN, want_tiled: bool = True):
    """K1+K2: tile and pool up to three raster tensors in one pass."""
    xs = list(xs)
    for x in xs:
        _cuda4(x, "tile_pool")
        if x.shape != xs[0].shape or x.dtype != xs[0].dtype:
            raise ValueError("attention: Q, K, V must share one shape")
        if x.shape[2] != layout.seq_len:
            raise ValueError("tile: sequence length does not match layout")
    B, H, _, d = xs[0].shape
    dev = xs[0].device
    tiled = [torch.empty((B, H, layout.seq_padded, d), dtype=xs[0].dtype, device=dev) for _ in xs] if want_tiled else None
    pooled = [torch.empty((B, H, layout.num_cubes, d), dtype=torch.float32, device=dev) for _ in xs]
    n = len(xs)
    xr = (C.c_void_p * n)(*[x.data_ptr() for x in xs])
    xt = (C.c_void_p * n)(*[t.data_ptr() for t in tiled]) if want_tiled else None
    pl = (C.c_void_p * n)(*[t.data_ptr() for t in pooled])
    check(L.lib().vsa_tile_pool(layout.ref(), B * H, d, _dt(xs[0]), n, xr, xt, pl, mode, _stream()))
    return tiled, pooled


# ----------------------------------------------------------------------------- block maps
def all_cubes(B: int, H: int, nc: int, device="cuda") -> torch.Tensor:
    """BlockSelection::all_cubes (selection.cpp:13-22) — the dense baseline map."""
    return torch.arange(nc, dtype=torch.int32, device=device).expand(B, H, nc, nc).contiguous()


def validate_selection(sel: torch.Tensor, num_cubes: int) -> None:
    """BlockSelection::validate (selection.cpp:24-37), on device; raises ValueError."""
    if sel is None or sel.numel() == 0:
        raise ValueError("BlockSelection: empty selection")
    if sel.dtype != torch.int32 or not sel.is_cuda or sel.dim() != 4 or not sel.is_contiguous():
        raise ValueError("BlockSelection: expected contiguous int32 [B, H, nc, k] on CUDA")
    B, H, nc, k = sel.shape
    if nc != num_cubes:
        raise ValueError("fine stage: selection does not match shapes")
    err = torch.empty(1, dtype=torch.int32, device=sel.device)
    check(L.lib().vsa_validate_selection(_p(sel), B * H * nc, k, nc, _p(err), _stream()))
    if int(err.item()) != 0:
        raise ValueError("BlockSelection: indices must be strictly ascending and in [0, num_cubes)")


def selection_transpose(layout: TileLayout, sel: torch.Tensor):
    """The transposed block map (fine.hpp:163-170 `rev`) as CSR: (offs [B*H, nc+1], idx [B*H, nc*k])."""
    B, H, nc, k = sel.shape
    offs = torch.empty((B * H, nc + 1), dtype=torch.int32, device=sel.device)
    idx = torch.empty((B * H, nc * k), dtype=torch.int32, device=sel.device)
    bm = torch.empty(max(1, L.lib().vsa_coarse_bitmap_bytes(layout.ref(), B * H)), dtype=torch.uint8, device=sel.device)
    check(L.lib().vsa_selection_transpose(layout.ref(), B * H, _p(sel), k, _p(offs), _p(idx), _p(bm), _stream()))
    return offs, idx


# ----------------------------------------------------------------------------- coarse
@dataclass
class CoarseArtifacts:
    """CoarseArtifacts (coarse.hpp:18-25). Oc is kept at cube level (oc_cube);
    ``oc`` materialises the reference's token-level broadcast on demand."""

    qc: torch.Tensor
    kc: torch.Tensor
    vc: torch.Tensor
    ac: torch.Tensor
    oc_cube: torch.Tensor
    sel: torch.Tensor
    selT_offs: torch.Tensor
    selT_idx: torch.Tensor
    pool: int
    cube_size: int

    @property
    def oc(self) -> torch.Tensor:
        return self.oc_cube.repeat_interleave(self.cube_size, dim=2)


def coarse_from_pooled(layout: TileLayout, qc, kc, vc, top_k: int, pool: int = POOL_MEAN) -> CoarseArtifacts:
    """K3 from pooled fp32 [B,H,nc,d] tensors."""
    B, H, nc, d = qc.shape
    dev = qc.device
    ac = torch.empty((B, H, nc, nc), dtype=torch.float32, device=dev)
    oc = torch.empty((B, H, nc, d), dtype=torch.float32, device=dev)
    k = max(int(top_k), 1)
    sel = torch.empty((B, H, nc, k), dtype=torch.int32, device=dev)
    offs = torch.empty((B * H, nc + 1), dtype=torch.int32, device=dev)
    idx = torch.empty((B * H, nc * k), dtype=torch.int32, device=dev)
    bm = torch.empty(max(1, L.lib().vsa_coarse_bitmap_bytes(layout.ref(), B * H)), dtype=torch.uint8, device=dev)
    check(L.lib().vsa_coarse_forward(layout.ref(), B * H, d, _p(qc), _p(kc), _p(vc), int(top_k), _p(ac), _p(oc),
                                     _p(sel), _p(offs), _p(idx), _p(bm), _stream()))
    return CoarseArtifacts(qc, kc, vc, ac, oc, sel, offs, idx, pool, layout.cube_size)


def coarse_forward_select(layout: TileLayout, q, k, v, top_k: int, mode: int = POOL_MEAN) -> CoarseArtifacts:
    """coarse_forward_select (coarse.hpp:71-117); q, k, v tile-ordered like the reference."""
    for t, n in ((q, "q"), (k, "k"), (v, "v")):
        _cuda4(t, n)
    if not (q.shape == k.shape == v.shape):
        raise ValueError("attention: Q, K, V must share one shape")
    if q.shape[2] != layout.seq_padded:
        raise ValueError("coarse_forward_select: shape/layout mismatch")
    if not (1 <= top_k <= layout.num_cubes):
        raise ValueError("coarse_forward_select: k must be in [1, num_cubes]")
    qc, kc, vc = (pool_cubes(layout, t, mode) for t in (q, k, v))
    return coarse_from_pooled(layout, qc, kc, vc, top_k, mode)


def coarse_backward(art: CoarseArtifacts, layout: TileLayout, doc, q, k, v):
    """coarse_backward (coarse.hpp:124-184): token-level dOc (tiled) -> tiled (dq, dk, dv)."""
    _cuda4(doc, "coarse_backward")
    if doc.shape != q.shape:
        raise ValueError("coarse_backward: dOc shape mismatch")
    if art is None or art.ac is None or art.ac.shape[2] != layout.num_cubes:
        raise ValueError("coarse_backward: artifacts do not match layout")
    B, H, _, d = q.shape
    nc = layout.num_cubes
    doc_cube = pool_cubes(layout, doc, POOL_MEAN) * float(layout.cube_size)  # sum over tokens
    dqc, dkc, dvc = (torch.empty((B, H, nc, d), dtype=torch.float32, device=q.device) for _ in range(3))
    scratch = torch.empty((B, H, nc, nc), dtype=torch.float32, device=q.device)
    check(L.lib().vsa_coarse_backward(layout.ref(), B * H, d, _p(art.qc), _p(art.kc), _p(art.vc), _p(art.ac),
                                      _p(doc_cube), _p(dqc), _p(dkc), _p(dvc), _p(scratch), _stream()))
    outs = []
    for dc, x in ((dqc, q), (dkc, k), (dvc, v)):
        if art.pool == POOL_MEAN:
            outs.append((dc / float(layout.cube_size)).repeat_interleave(layout.cube_size, dim=2).to(q.dtype))
        else:
            dx = torch.zeros_like(x)
            check(L.lib().vsa_unpool_max_add(layout.ref(), B * H, d, _dt(x), _p(x), _p(dc), 0, _p(dx), _stream()))
            outs.append(dx)
    return tuple(outs)


# ----------------------------------------------------------------------------- fine
@dataclass
class FineResult:
    """FineResult (fine.hpp:17-20): out + saved softmax stats [B*H, seq]."""

    out: torch.Tensor
    row_max: torch.Tensor
    row_lse: torch.Tensor


def _check_fine(layout, q, k, v, sel):
    for t, n in ((q, "q"), (k, "k"), (v, "v")):
        _cuda4(t, n)
    if q.numel() == 0:
        raise ValueError("attention: empty tensors")
    if not (q.shape == k.shape == v.shape) or not (q.dtype == k.dtype == v.dtype):
        raise ValueError("attention: Q, K, V must share one shape")
    if q.shape[2] != layout.seq_padded:
        raise ValueError("fine stage: sequence length does not match layout")
    if sel.dim() != 4 or sel.shape[0] != q.shape[0] or sel.shape[1] != q.shape[1] or sel.shape[2] != layout.num_cubes:
        raise ValueError("fine stage: selection does not match shapes")
    validate_selection(sel, layout.num_cubes)


def fine_forward(layout: TileLayout, q, k, v, sel, force_simt: bool = False) -> FineResult:
    """fine_forward (fine.hpp:43-99) on tile-ordered q, k, v."""
    _check_fine(layout, q, k, v, sel)
    B, H, S, d = q.shape
    out = torch.empty_like(q)
    lse = torch.empty((B * H, S), dtype=torch.float32, device=q.device)
    rmax = torch.empty((B * H, S), dtype=torch.float32, device=q.device)
    flags = L.FINE_FORCE_SIMT if force_simt else 0
    check(L.lib().vsa_fine_forward(layout.ref(), B * H, d, _dt(q), _p(q), _p(k), _p(v), _p(sel), sel.shape[3],
                                   _p(out), _p(lse), _p(rmax), None, None, None, flags, None, _stream()))
    return FineResult(out, rmax, lse)


def fine_backward(layout: TileLayout, q, k, v, sel, dout, row_lse, out=None, selT=None, force_simt=False,
                  workspace=True):
    """fine_backward (fine.hpp:107-204) -> tiled (dq, dk, dv). `out` (the forward
    output) lets delta be read as rowsum(dO*O); without it delta is recomputed
    by one extra pass. `workspace=True` uses the dS-materialising path (dQ as a
    GEMM over stored dS tiles); False recomputes S and dP for dQ."""
    _check_fine(layout, q, k, v, sel)
    if dout.shape != q.shape:
        raise ValueError("fine_backward: dO shape mismatch")
    B, H, S, d = q.shape
    if row_lse.numel() != B * H * S:
        raise ValueError("fine_backward: saved statistics do not match shapes")
    if out is None:
        out = fine_forward(layout, q, k, v, sel, force_simt).out
    offs, idx = selT if selT is not None else selection_transpose(layout, sel)
    delta = torch.empty((B * H, S), dtype=torch.float32, device=q.device)
    doc = torch.empty((B, H, layout.num_cubes, d), dtype=torch.float32, device=q.device)
    dof = torch.empty_like(q)
    ones = torch.ones_like(q)
    zoc = torch.zeros((B, H, layout.num_cubes, d), dtype=torch.float32, device=q.device)
    # prologue with Gf = 1, Gc = 1: dof = dout, delta = rowsum(dout*out)
    check(L.lib().vsa_backward_prologue(layout.ref(), B * H, d, _dt(q), 0, _p(dout), _p(ones), None, _p(zoc),
                                        _p(out), 1, _p(dof), _p(delta), _p(doc), None, None, _stream()))
    dq, dk, dv = torch.empty_like(q), torch.empty_like(q), torch.empty_like(q)
    flags = L.FINE_FORCE_SIMT if force_simt else 0
    wsb = L.lib().vsa_fine_backward_workspace_bytes(layout.ref(), B * H, sel.shape[3])
    ws = torch.empty(max(wsb, 1), dtype=torch.uint8, device=q.device) if workspace else None
    check(L.lib().vsa_fine_backward(layout.ref(), B * H, d, _dt(q), _p(q), _p(k), _p(v), _p(dof), _p(row_lse),
                                    _p(delta), _p(sel), sel.shape[3], _p(offs), _p(idx), None, None, None, 0, flags,
                                    _p(dq), _p(dk), _p(dv), _p(ws), wsb if workspace else 0, _stream()))
    return dq, dk, dv


# ----------------------------------------------------------------------------- the operator
class VsaOp:
    """The VSA attention operator on device-resident buffers: the hot path.

    forward(q, k, v, gc, gf) -> O and backward(dO) -> (dQ, dK, dV, dGc, dGf), all
    raster-ordered [B, H, t*h*w, d] (``raster=True``, tiling fused into K1 and the
    fine epilogue) or tile-ordered (``raster=False``, the reference's vsa_forward
    contract, vsa.hpp:86). Buffers are allocated once (HBM-resident artifacts,
    the VsaOutput of vsa.hpp:56-63).

    ``io="bshd"`` (raster only) reads and writes the raster tensors sequence-major
    instead: [B, S, H, d] (DiT-native), or with ``seq_chunks=P`` the
    Ulysses receive layout [P, B, S/P, H, d] (§8e) — consumed in place, no copies.
    """

    def __init__(self, layout: TileLayout, B: int, H: int, d: int, top_k: int, dtype=torch.bfloat16,
                 pool: int = POOL_MEAN, adaptation: bool = False, raster: bool = True, device="cuda",
                 force_simt: bool = False, bwd_workspace: bool = True, io: str = "bhsd", seq_chunks: int = 1):
        if not (1 <= top_k <= layout.num_cubes):
            raise ValueError("coarse_forward_select: k must be in [1, num_cubes]")
        if io not in ("bhsd", "bshd"):
            raise ValueError("io must be 'bhsd' or 'bshd'")
        if io == "bshd" and not raster:
            raise ValueError("sequence-major I/O needs raster=True")
        self.io, self.seq_chunks = io, int(seq_chunks)
        self.layout, self.B, self.H, self.d, self.top_k = layout, B, H, d, int(top_k)
        self.dtype, self.pool, self.adaptation, self.raster = dtype, pool, adaptation, raster
        self.force_simt = force_simt
        # dS-materialising backward workspace (B*H*nc*k bf16 64x64 tiles), allocated on first backward
        self.bwd_workspace = bwd_workspace
        self.ws = None
        nc, Lp = layout.num_cubes, layout.seq_padded
        e = lambda *s, dt=dtype: torch.empty(s, dtype=dt, device=device)
        f32, i32 = torch.float32, torch.int32
        self.q_t, self.k_t, self.v_t = e(B, H, Lp, d), e(B, H, Lp, d), e(B, H, Lp, d)
        self.qc, self.kc, self.vc = e(B, H, nc, d, dt=f32), e(B, H, nc, d, dt=f32), e(B, H, nc, d, dt=f32)
        self.ac = e(B, H, nc, nc, dt=f32)
        self.oc = e(B, H, nc, d, dt=f32)
        self.sel = e(B, H, nc, self.top_k, dt=i32)
        self.selT_offs = e(B * H, nc + 1, dt=i32)
        self.selT_idx = e(B * H, nc * self.top_k, dt=i32)
        self.bitmap = e(max(1, L.lib().vsa_coarse_bitmap_bytes(layout.ref(), B * H)), dt=torch.uint8)
        self.o_f = e(B, H, Lp, d)
        self.lse = e(B, H, Lp, dt=f32)
        self.dof = e(B, H, Lp, d)
        self.delta = e(B, H, Lp, dt=f32)
        self.doc = e(B, H, nc, d, dt=f32)
        self.dqc, self.dkc, self.dvc = e(B, H, nc, d, dt=f32), e(B, H, nc, d, dt=f32), e(B, H, nc, d, dt=f32)
        self.scratch = e(B, H, nc, nc, dt=f32)
        self.fine_sel = self.sel
        self.fine_k = self.top_k
        self._gc = self._gf = None
        self._lib = L.lib()
        self._lref = layout.ref()
        S = layout.seq_len
        if io == "bshd":
            if self.seq_chunks < 1 or S % self.seq_chunks:
                raise ValueError("seq_chunks must divide the raster sequence length")
            self._raw = L.vsa_layout_t.from_buffer_copy(layout._raw)
            check(self._lib.vsa_layout_set_io(C.byref(self._raw), L.IO_SEQ_MAJOR, B, H, S // self.seq_chunks))
            self._lref = C.byref(self._raw)
            self.io_shape = ((B, S, H, d) if self.seq_chunks == 1 else
                             (self.seq_chunks, B, S // self.seq_chunks, H, d))
        else:
            self.io_shape = (B, H, S if raster else layout.seq_padded, d)
        self.trace = None  # optional list: (stage, torch.cuda.Event) appended after each stage

    def _mark(self, name):
        if self.trace is not None:
            ev = torch.cuda.Event(enable_timing=True)
            ev.record()
            self.trace.append((name, ev))

    @property
    def seq_io(self) -> int:
        return self.layout.seq_len if self.raster else self.layout.seq_padded

    def _chk(self, t, name):
        if not isinstance(t, torch.Tensor) or not t.is_cuda:
            raise ValueError(f"{name}: expected a CUDA tensor")
        shp = tuple(t.shape)
        if self.io == "bshd" and len(shp) == 5 and shp[0] == 1:
            shp = shp[1:]  # [1, B, S, H, d]: the chunked layout with one chunk
        if shp != self.io_shape or t.dtype != self.dtype:
            raise ValueError(f"{name}: expected {self.io_shape} {self.dtype}")
        if not t.is_contiguous():
            raise ValueError(f"{name}: must be contiguous")

    def forward(self, q, k, v, gc, gf=None, out=None, sel_override=None, check_inputs=True, before_fine=None):
        """vsa_forward (vsa.hpp:89-122) at attention level: gates are given.

        ``before_fine``: optional callable run after the coarse stage, before the
        fine kernel (the first reader of the gates) — e.g. to wait for a gate
        exchange that overlapped K1-K3."""
        lib, lr, st = self._lib, self._lref, _stream()
        B, H, d = self.B, self.H, self.d
        bh = B * H
        dt = L.VSA_BF16 if self.dtype == torch.bfloat16 else L.VSA_F32
        if check_inputs:
            for t, n in ((q, "q"), (k, "k"), (v, "v"), (gc, "gate_coarse")):
                self._chk(t, n)
            if not self.adaptation:
                if gf is None:
                    raise ValueError("vsa_forward: missing fine gate")
                self._chk(gf, "gate_fine")
        if self.raster:
            xr = (C.c_void_p * 3)(q.data_ptr(), k.data_ptr(), v.data_ptr())
            xt = (C.c_void_p * 3)(self.q_t.data_ptr(), self.k_t.data_ptr(), self.v_t.data_ptr())
            pl = (C.c_void_p * 3)(self.qc.data_ptr(), self.kc.data_ptr(), self.vc.data_ptr())
            self._mark("start")
            check(lib.vsa_tile_pool(lr, bh, d, dt, 3, xr, xt, pl, self.pool, st))
            self._mark("tile_pool")
            qt, kt, vt = self.q_t, self.k_t, self.v_t
        else:
            qt, kt, vt = q, k, v
            self._mark("start")
            for x, p in ((q, self.qc), (k, self.kc), (v, self.vc)):
                check(lib.vsa_pool_tiled(lr, bh, d, dt, _p(x), _p(p), self.pool, st))
            self._mark("tile_pool")
        override = sel_override is not None
        check(lib.vsa_coarse_forward(lr, bh, d, _p(self.qc), _p(self.kc), _p(self.vc), self.top_k, _p(self.ac),
                                     _p(self.oc), _p(self.sel), None if override else _p(self.selT_offs),
                                     None if override else _p(self.selT_idx), _p(self.bitmap), st))
        self._mark("coarse_fwd")
        if override:
            validate_selection(sel_override, self.layout.num_cubes)
            if sel_override.shape[:3] != self.sel.shape[:3]:
                raise ValueError("fine stage: selection does not match shapes")
            self.fine_sel, self.fine_k = sel_override, int(sel_override.shape[3])
            if self.selT_idx.shape[1] < self.layout.num_cubes * self.fine_k:
                self.selT_idx = torch.empty((bh, self.layout.num_cubes * self.fine_k), dtype=torch.int32,
                                            device=q.device)
            check(lib.vsa_selection_transpose(lr, bh, _p(sel_override), self.fine_k, _p(self.selT_offs),
                                              _p(self.selT_idx), _p(self.bitmap), st))
        else:
            self.fine_sel, self.fine_k = self.sel, self.top_k
        if out is None:
            out = torch.empty(self.io_shape, dtype=self.dtype, device=q.device)
        if before_fine is not None:
            before_fine()
        flags = L.FINE_COMBINE | (L.FINE_UNTILE if self.raster else 0) | (L.FINE_ADAPTATION if self.adaptation else 0)
        if self.force_simt:
            flags |= L.FINE_FORCE_SIMT
        check(lib.vsa_fine_forward(lr, bh, d, dt, _p(qt), _p(kt), _p(vt), _p(self.fine_sel), self.fine_k,
                                   _p(self.o_f), _p(self.lse), None, _p(gc), _p(gf), _p(self.oc), flags, _p(out), st))
        self._mark("fine_fwd")
        self._gc, self._gf = gc, gf
        self._qkv = (qt, kt, vt)
        return out

    def backward(self, dout, dq=None, dk=None, dv=None, dgc=None, dgf=None, check_inputs=True):
        """vsa_backward (vsa.hpp:129-189) at attention level -> (dq, dk, dv, dgc, dgf)."""
        if self._gc is None:
            raise ValueError("vsa_backward: missing or mismatched forward artifacts")
        if check_inputs:
            self._chk(dout, "dO")
        lib, lr, st = self._lib, self._lref, _stream()
        B, H, d = self.B, self.H, self.d
        bh = B * H
        dt = L.VSA_BF16 if self.dtype == torch.bfloat16 else L.VSA_F32
        mk = lambda: torch.empty(self.io_shape, dtype=self.dtype, device=dout.device)
        dq = mk() if dq is None else dq
        dk = mk() if dk is None else dk
        dv = mk() if dv is None else dv
        dgc = mk() if dgc is None else dgc
        dgf = mk() if dgf is None else dgf
        raster = 1 if self.raster else 0
        if self.raster and self.layout.seq_padded != self.layout.seq_len:
            pass  # padded rows of dq/dk/dv are never written (dropped at untile)
        check(lib.vsa_backward_prologue(lr, bh, d, dt, raster, _p(dout), _p(self._gc), _p(self._gf), _p(self.oc),
                                        _p(self.o_f), 1 if self.adaptation else 0, _p(self.dof), _p(self.delta),
                                        _p(self.doc), _p(dgc), _p(dgf), st))
        self._mark("prologue")
        check(lib.vsa_coarse_backward(lr, bh, d, _p(self.qc), _p(self.kc), _p(self.vc), _p(self.ac), _p(self.doc),
                                      _p(self.dqc), _p(self.dkc), _p(self.dvc), _p(self.scratch), st))
        self._mark("coarse_bwd")
        mean = self.pool == POOL_MEAN
        qt, kt, vt = self._qkv
        flags = L.FINE_FORCE_SIMT if self.force_simt else 0
        wsb = lib.vsa_fine_backward_workspace_bytes(lr, bh, self.fine_k) if self.bwd_workspace else 0
        if wsb and (self.ws is None or self.ws.numel() < wsb):
            free, _ = torch.cuda.mem_get_info(dout.device)
            if wsb > 0.6 * free:  # e.g. the dense baseline at 14B (all cubes): dQ recomputes S / dP instead
                wsb = 0
            else:
                self.ws = torch.empty(wsb, dtype=torch.uint8, device=dout.device)
        check(lib.vsa_fine_backward(lr, bh, d, dt, _p(qt), _p(kt), _p(vt), _p(self.dof), _p(self.lse),
                                    _p(self.delta), _p(self.fine_sel), self.fine_k, _p(self.selT_offs),
                                    _p(self.selT_idx), _p(self.dqc) if mean else None, _p(self.dkc) if mean else None,
                                    _p(self.dvc) if mean else None, raster, flags, _p(dq), _p(dk), _p(dv),
                                    _p(self.ws) if wsb else None, wsb, st))
        self._mark("fine_bwd")
        if not mean:
            for x, dc, g in ((qt, self.dqc, dq), (kt, self.dkc, dk), (vt, self.dvc, dv)):
                check(lib.vsa_unpool_max_add(lr, bh, d, dt, _p(x), _p(dc), raster, _p(g), st))
        if self.adaptation:
            dgf.zero_()
        return dq, dk, dv, dgc, dgf

    @property
    def artifacts(self) -> CoarseArtifacts:
        return CoarseArtifacts(self.qc, self.kc, self.vc, self.ac, self.oc, self.sel, self.selT_offs, self.selT_idx,
                               self.pool, self.layout.cube_size)


class VsaHostPipeline:
    """Forward + backward on HOST (pinned) tensors with the H2D / D2H copies
    overlapped with the kernels.

    Every (b, h) unit is independent (fine.hpp:65,129,172), so the B*H units are
    split into `chunks` groups; group i+1 is copied in on one stream while group
    i computes, and group i-1 is copied out on a third — double-buffered device
    inputs/outputs, events for the hand-offs. Result == VsaOp on the whole batch.
    """

    def __init__(self, layout: TileLayout, B: int, H: int, d: int, top_k: int, chunks: int = 12,
                 dtype=torch.bfloat16, device="cuda", **op_kwargs):
        units = B * H
        chunks = max(1, min(chunks, units))
        self.bounds = [(units * i) // chunks for i in range(chunks + 1)]
        self.units, self.d, self.S, self.dtype = units, d, layout.seq_len, dtype
        cmax = max(b - a for a, b in zip(self.bounds[:-1], self.bounds[1:]))
        self.ops = [VsaOp(layout, 1, cmax, d, top_k, dtype=dtype, device=device, **op_kwargs) for _ in range(2)]
        e = lambda: torch.empty((1, cmax, self.S, d), dtype=dtype, device=device)
        self.din = [[e() for _ in range(6)] for _ in range(2)]
        self.dout = [[e() for _ in range(6)] for _ in range(2)]
        self.s_in, self.s_out = torch.cuda.Stream(device), torch.cuda.Stream(device)
        self.h2d_bytes = 6 * units * self.S * d * torch.tensor([], dtype=dtype).element_size()
        self.d2h_bytes = self.h2d_bytes

    def run(self, hin, hout):
        """hin = (q, k, v, gc, gf, dO), hout = (O, dQ, dK, dV, dGc, dGf): pinned host [B,H,S,d].

        Per group: the five forward inputs are copied first and the forward starts as
        soon as they land (dO follows on the copy stream); O is copied out while the
        backward runs, the five gradients after it."""
        flat = lambda t: t.view(self.units, self.S, self.d)
        hin, hout = [flat(t) for t in hin], [flat(t) for t in hout]
        comp = torch.cuda.current_stream()
        n = len(self.bounds) - 1
        ev_comp, ev_out = [None] * n, [None] * n
        ev = lambda: torch.cuda.Event()
        for i in range(n):
            a, b = self.bounds[i], self.bounds[i + 1]
            c, slot = b - a, i % 2
            di, do = self.din[slot], self.dout[slot]
            with torch.cuda.stream(self.s_in):
                if i >= 2:
                    self.s_in.wait_event(ev_comp[i - 2])      # slot's inputs consumed
                for dst, src in zip(di[:5], hin[:5]):
                    dst[0, :c].copy_(src[a:b], non_blocking=True)
                ev_fwd_in = ev()
                ev_fwd_in.record(self.s_in)
                di[5][0, :c].copy_(hin[5][a:b], non_blocking=True)
                ev_bwd_in = ev()
                ev_bwd_in.record(self.s_in)
            comp.wait_event(ev_fwd_in)
            if i >= 2:
                comp.wait_event(ev_out[i - 2])                # slot's outputs drained
            op = self.ops[slot]
            if c == op.H:
                op.forward(*di[:5], out=do[0], check_inputs=False)
                ev_fwd = ev()
                ev_fwd.record(comp)
                with torch.cuda.stream(self.s_out):
                    self.s_out.wait_event(ev_fwd)
                    hout[0][a:b].copy_(do[0][0, :c], non_blocking=True)
                comp.wait_event(ev_bwd_in)
                op.backward(di[5], *do[1:], check_inputs=False)
                first_out = 1
            else:  # ragged last group: run on views of the right head count
                comp.wait_event(ev_bwd_in)
                sub = VsaOp(op.layout, 1, c, self.d, op.top_k, dtype=self.dtype, device=di[0].device)
                v = lambda t: t[:, :c].contiguous()
                o = sub.forward(*(v(t) for t in di[:5]))
                g = sub.backward(v(di[5]))
                for dst, src in zip(do, (o, *g)):
                    dst[:, :c].copy_(src)
                first_out = 0
            ev_comp[i] = ev()
            ev_comp[i].record(comp)
            with torch.cuda.stream(self.s_out):
                self.s_out.wait_event(ev_comp[i])
                for dst, src in zip(hout[first_out:], do[first_out:]):
                    dst[a:b].copy_(src[0, :c], non_blocking=True)
                ev_out[i] = ev()
                ev_out[i].record(self.s_out)
        comp.wait_event(ev_out[n - 1])
        if n >= 2:
            comp.wait_event(ev_out[n - 2])


# ----------------------------------------------------------------------------- gate projection (vsa.hpp:100-112)
@dataclass
class VsaParams:
    """VsaParams (vsa.hpp:16-52) with torch tensors; the gate projection runs on the
    tcgen05 GEMM of csrc/gemm_sm100.cu."""

    gate_weight: torch.Tensor            # [model_dim, 2*H*d]
    gate_bias: torch.Tensor | None = None
    top_k: int = 1
    pool: int = POOL_MEAN
    activation: int = GATE_IDENTITY
    adaptation: bool = False

    def check(self, model_dim, heads, head_dim):
        if tuple(self.gate_weight.shape) != (model_dim, 2 * heads * head_dim):
            raise ValueError("VsaParams: gate projection must map model_dim -> 2*heads*head_dim")
        if self.gate_bias is not None and self.gate_bias.numel() not in (0, self.gate_weight.shape[1]):
            raise ValueError("VsaParams: gate bias size mismatch")
        if self.top_k < 1:
            raise ValueError("VsaParams: k must be >= 1")


def _gate_layout(layout, S):
    if layout is None:
        return TileLayout(1, 1, S, 1, 1, 1)  # head-major [B,H,S,d] gates, no tiling involved
    if layout.seq_len != S:
        raise ValueError("gates: layout sequence length does not match hidden")
    return layout


def _gate_bias(params: VsaParams):
    if params.gate_bias is None or params.gate_bias.numel() == 0:
        return None
    return params.gate_bias.float().contiguous()


def gates_from_hidden(hidden: torch.Tensor, params: VsaParams, H: int, d: int, layout=None, op=None):
    """z = hidden Wg (+b) [sigmoid]; split into Gc, Gf [B,H,S,d] (vsa.hpp:100-112).

    tcgen05 GEMM with the bias / activation / split fused in its epilogue
    (vsa_gate_forward). hidden: bf16 CUDA [B, 1, S, model_dim]; gate_weight bf16
    [model_dim, 2*H*d]. With ``op`` (a VsaOp) the gates are written in the op's raster
    I/O layout (e.g. sequence-major)."""
    _cuda4(hidden, "hidden")
    B, one, S, md = hidden.shape
    if one != 1:
        raise ValueError("vsa: hidden states are [batch, 1, seq, model_dim]")
    params.check(md, H, d)
    w = params.gate_weight
    if hidden.dtype != torch.bfloat16 or w.dtype != torch.bfloat16 or not w.is_cuda or not w.is_contiguous():
        raise ValueError("gates: bf16 CUDA hidden and gate_weight required")
    if op is not None:
        lref, shape = op._lref, op.io_shape
    else:
        lref, shape = _gate_layout(layout, S).ref(), (B, H, S, d)
    gc = torch.empty(shape, dtype=hidden.dtype, device=hidden.device)
    gf = torch.empty(shape, dtype=hidden.dtype, device=hidden.device)
    bias = _gate_bias(params)
    check(L.lib().vsa_gate_forward(lref, B, H, d, md, _p(hidden), _p(w), _p(bias) if bias is not None else None,
                                   int(params.activation), 1 if params.adaptation else 0, _p(gc), _p(gf), _stream()))
    return gc, gf


def gate_backward(hidden, params: VsaParams, gc, gf, dgc, dgf, layout=None, op=None):
    """dz -> dhidden, dWg, dbias (vsa.hpp:152-176) on tcgen05 (vsa_gate_backward):
    dz = [dGc, dGf] (x G(1-G) for sigmoid), dhidden = dz Wg^T (bf16), dWg = hidden^T dz
    and dbias = colsum(dz) (fp32)."""
    B, _, S, md = hidden.shape
    d = gc.shape[-1]
    H = params.gate_weight.shape[1] // (2 * d)
    lref = op._lref if op is not None else _gate_layout(layout, S).ref()
    lib = L.lib()
    wsb = lib.vsa_gate_backward_workspace_bytes(lref, B, H, d)
    ws = torch.empty(wsb, dtype=torch.uint8, device=hidden.device)
    dhidden = torch.empty_like(hidden)
    dW = torch.empty(params.gate_weight.shape, dtype=torch.float32, device=hidden.device)
    bias = _gate_bias(params)
    db = torch.empty(bias.shape, dtype=torch.float32, device=hidden.device) if bias is not None else None
    check(lib.vsa_gate_backward(lref, B, H, d, md, _p(hidden), _p(params.gate_weight), _p(gc), _p(gf), _p(dgc),
                                _p(dgf) if dgf is not None else None, int(params.activation),
                                1 if params.adaptation else 0, _p(ws), _p(dhidden), _p(dW),
                                _p(db) if db is not None else None, _stream()))
    return dhidden, dW, db


# ----------------------------------------------------------------------------- selection analytics (§8 f4)
def aggregate_probs_to_cubes(layout: TileLayout, probs: torch.Tensor) -> torch.Tensor:
    """aggregate_probs_to_cubes (analysis.hpp:130-147): fp32 [B,H,S,S] tile-ordered token
    probabilities -> [B,H,S,nc] (unpadded layouts, diagnostics at small S)."""
    _cuda4(probs, "probs")
    B, H, S, S2 = probs.shape
    if S != layout.seq_len or S2 != layout.seq_len or probs.dtype != torch.float32:
        raise ValueError("aggregate_probs_to_cubes: expected fp32 [.., seq, seq] probabilities")
    out = torch.empty((B, H, S, layout.num_cubes), dtype=torch.float32, device=probs.device)
    check(L.lib().vsa_aggregate_probs_to_cubes(layout.ref(), B * H, _p(probs), _p(out), _stream()))
    return out


def selection_accuracy(layout: TileLayout, probs_cube: torch.Tensor, sel: torch.Tensor) -> torch.Tensor:
    """selection_accuracy (analysis.hpp:100-125): mean captured mass per (b, h), float64 [B,H]."""
    _cuda4(probs_cube, "probs_cube")
    B, H, S, nc = probs_cube.shape
    if S != layout.seq_len or nc != layout.num_cubes or probs_cube.dtype != torch.float32:
        raise ValueError("selection_accuracy: probabilities do not match layout")
    if tuple(sel.shape[:3]) != (B, H, nc):
        raise ValueError("selection_accuracy: selection does not match shapes")
    acc = torch.empty((B, H), dtype=torch.float64, device=probs_cube.device)
    check(L.lib().vsa_selection_accuracy(layout.ref(), B * H, _p(probs_cube), _p(sel), sel.shape[3], _p(acc),
                                         _stream()))
    return acc


def selection_accuracy_qk(layout: TileLayout, q: torch.Tensor, k: torch.Tensor, sel: torch.Tensor) -> torch.Tensor:
    """Captured dense-attention mass of a block map straight from Q, K (tile-ordered):
    mean_i exp(lse_sel(i) - lse_all(i)) from two fine forwards (the selection and all
    cubes) — the same quantity as selection_accuracy(aggregate_probs_to_cubes(
    dense_probs(q, k)), sel) without the [S,S] matrix. float64 [B,H]."""
    if layout.seq_padded != layout.seq_len:
        raise ValueError("selection_accuracy_qk: padded layouts are not supported")
    B, H, S, d = q.shape
    lse_sel = fine_forward(layout, q, k, k, sel).row_lse
    lse_all = fine_forward(layout, q, k, k, all_cubes(B, H, layout.num_cubes, device=q.device)).row_lse
    acc = torch.empty((B, H), dtype=torch.float64, device=q.device)
    check(L.lib().vsa_selection_accuracy_from_lse(_p(lse_sel), _p(lse_all), B * H, S, _p(acc), _stream()))
    return acc
