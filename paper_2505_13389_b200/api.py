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
    """vsa::TileLayout (layout.hpp:14-33). The reference rejects non-divisible grids
    (layout.cpp:10-11); ``pad=True`` (or ``"zero"``) pads with zero tokens that are ordinary
    tokens (the parity mode), ``pad="mask"`` pads FastVideo-style: padded keys are excluded
    from attention and cube means / maxima are over the real tokens."""

    def __init__(self, tokens_t, tokens_h, tokens_w, cube_t=4, cube_h=4, cube_w=4, pad=False):
        modes = {False: L.PAD_REJECT, None: L.PAD_REJECT, True: L.PAD_ZERO, "zero": L.PAD_ZERO, "mask": L.PAD_MASK}
        if pad not in modes:
            raise ValueError("TileLayout: pad must be False, True / 'zero' or 'mask'")
        self._raw = L.vsa_layout_t()
        check(L.lib().vsa_layout_make(tokens_t, tokens_h, tokens_w, cube_t, cube_h, cube_w, modes[pad],
                                      C.byref(self._raw)))

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
    mask_pad = property(lambda s: s._raw.pad_mode == L.PAD_MASK)

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
    """coarse_backward (coarse.hpp:124-184): token-level dOc (tiled) -> tiled (dq, dk, dv).
    Cube sums, the cube-level backward and the unpool all run in the library
    (vsa_coarse_backward_tokens)."""
    _cuda4(doc, "coarse_backward")
    if doc.shape != q.shape:
        raise ValueError("coarse_backward: dOc shape mismatch")
    if art is None or art.ac is None or art.ac.shape[2] != layout.num_cubes:
        raise ValueError("coarse_backward: artifacts do not match layout")
    B, H, _, d = q.shape
    nc = layout.num_cubes
    f32 = lambda *s: torch.empty(s, dtype=torch.float32, device=q.device)
    doc_cube, dqc, dkc, dvc = (f32(B, H, nc, d) for _ in range(4))
    scratch = f32(B, H, nc, nc)
    dq, dk, dv = torch.empty_like(q), torch.empty_like(k), torch.empty_like(v)
    check(L.lib().vsa_coarse_backward_tokens(layout.ref(), B * H, d, _dt(q), _p(art.qc), _p(art.kc), _p(art.vc),
                                             _p(art.ac), int(art.pool), _p(doc), _p(q), _p(k), _p(v), _p(doc_cube),
                                             _p(dqc), _p(dkc), _p(dvc), _p(scratch), _p(dq), _p(dk), _p(dv),
                                             _stream()))
    return dq, dk, dv


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


@dataclass
class MacCounter:
    """MacCounter (tensor.hpp:36-39): executed tiles and MACs, counted ON THE DEVICE by the
    fine-forward kernels (vsa_debug_tile_counter); macs = tiles * 2 * cube^2 * d (fine.hpp:59-63)."""

    tiles: int = 0
    macs: int = 0


def fine_forward(layout: TileLayout, q, k, v, sel, force_simt: bool = False,
                 counter: MacCounter | None = None) -> FineResult:
    """fine_forward (fine.hpp:43-99) on tile-ordered q, k, v. ``counter`` (debug) adds the
    tiles the kernel executed, read back from a device counter (one sync)."""
    _check_fine(layout, q, k, v, sel)
    B, H, S, d = q.shape
    out = torch.empty_like(q)
    lse = torch.empty((B * H, S), dtype=torch.float32, device=q.device)
    rmax = torch.empty((B * H, S), dtype=torch.float32, device=q.device)
    flags = L.FINE_FORCE_SIMT if force_simt else 0
    lib = L.lib()
    ctr = torch.zeros(1, dtype=torch.int64, device=q.device) if counter is not None else None
    if ctr is not None:
        check(lib.vsa_debug_tile_counter(_p(ctr)))
    try:
        check(lib.vsa_fine_forward(layout.ref(), B * H, d, _dt(q), _p(q), _p(k), _p(v), _p(sel), sel.shape[3],
                                   _p(out), _p(lse), _p(rmax), None, None, None, flags, None, _stream()))
    finally:
        if ctr is not None:
            lib.vsa_debug_tile_counter(None)
    if ctr is not None:
        tiles = int(ctr.item())
        counter.tiles += tiles
        counter.macs += tiles * 2 * layout.cube_size * layout.cube_size * d
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

    A thin wrapper over the native operator context (``vsa_op_*`` in
    include/vsa_b200.h, csrc/op.cu), which orchestrates the stage kernels and keeps
    the forward artifacts (the VsaOutput of vsa.hpp:56-63) resident in HBM. Its
    device memory is one block from torch's caching allocator; the attributes
    (``sel``, ``lse``, ``ac``, ...) are views into it.

    forward(q, k, v, gc, gf) -> O and backward(dO) -> (dQ, dK, dV, dGc, dGf), all
    raster-ordered [B, H, t*h*w, d] (``raster=True``, tiling fused into K1 and the
    fine epilogue) or tile-ordered (``raster=False``, the reference's vsa_forward
    contract, vsa.hpp:86).

    ``io="bshd"`` (raster only) reads and writes the raster tensors sequence-major
    instead: [B, S, H, d] (DiT-native), or with ``seq_chunks=P`` the
    Ulysses receive layout [P, B, S/P, H, d] (§8e) — consumed in place, no copies.
    ``model_dim > 0`` adds the gate projection (``forward_hidden`` / ``backward_hidden``,
    the reference's vsa_forward / vsa_backward with hidden states and VsaParams).
    ``coarse="bf16"`` runs the coarse products on the tensor cores (tcgen05; the block map
    may differ from the reference's near the top-k boundary); the default ``"fp32"`` is
    the canonical-order mode whose map is bit-exact with the reference.
    """

    def __init__(self, layout: TileLayout, B: int, H: int, d: int, top_k: int, dtype=torch.bfloat16,
                 pool: int = POOL_MEAN, adaptation: bool = False, raster: bool = True, device="cuda",
                 force_simt: bool = False, bwd_workspace: bool = True, io: str = "bhsd", seq_chunks: int = 1,
                 max_sel_k: int = 0, model_dim: int = 0, activation: int = GATE_IDENTITY, coarse: str = "fp32",
                 task_range=None):
        if coarse not in ("fp32", "bf16"):
            raise ValueError("coarse must be 'fp32' (bit-exact block map) or 'bf16' (tcgen05)")
        self.coarse = coarse
        # sub-split: the fine stages compute only (unit, cube) tasks [t0, t1)
        self.task_range = (0, 0) if task_range is None else (int(task_range[0]), int(task_range[1]))
        if not (1 <= top_k <= layout.num_cubes):
            raise ValueError("coarse_forward_select: k must be in [1, num_cubes]")
        if io not in ("bhsd", "bshd"):
            raise ValueError("io must be 'bhsd' or 'bshd'")
        if io == "bshd" and not raster:
            raise ValueError("sequence-major I/O needs raster=True")
        if dtype not in (torch.bfloat16, torch.float32):
            raise ValueError(f"unsupported dtype {dtype} (bf16 or fp32)")
        self.io, self.seq_chunks = io, int(seq_chunks)
        self.layout, self.B, self.H, self.d, self.top_k = layout, B, H, d, int(top_k)
        self.dtype, self.pool, self.adaptation, self.raster = dtype, pool, adaptation, raster
        self.force_simt = force_simt
        self.model_dim, self.activation = int(model_dim), int(activation)
        # dS-materialising backward workspace (B*H*nc*k bf16 64x64 tiles), allocated on first backward
        self.bwd_workspace = bwd_workspace
        self.ws = None
        self.device = torch.device(device)
        self._lib = L.lib()
        S = layout.seq_len
        self._raw = L.vsa_layout_t.from_buffer_copy(layout._raw)
        if io == "bshd":
            if self.seq_chunks < 1 or S % self.seq_chunks:
                raise ValueError("seq_chunks must divide the raster sequence length")
            check(self._lib.vsa_layout_set_io(C.byref(self._raw), L.IO_SEQ_MAJOR, B, H, S // self.seq_chunks))
            self.io_shape = ((B, S, H, d) if self.seq_chunks == 1 else
                             (self.seq_chunks, B, S // self.seq_chunks, H, d))
        else:
            self.io_shape = (B, H, S if raster else layout.seq_padded, d)
        self._lref = C.byref(self._raw)
        self._h = None
        self._create(int(max_sel_k))
        self._timing = False

    # -- native context
    def _create(self, max_sel_k: int):
        lib = self._lib
        self.max_sel_k = max_sel_k
        flags = (L.OP_FORCE_SIMT if self.force_simt else 0) | (0 if self.bwd_workspace else L.OP_NO_DS_WORKSPACE)
        desc = L.vsa_op_desc_t(self.B, self.H, self.d, self.top_k, max_sel_k, self.model_dim,
                               L.VSA_BF16 if self.dtype == torch.bfloat16 else L.VSA_F32, int(self.pool),
                               self.activation, 1 if self.adaptation else 0, 1 if self.raster else 0, flags,
                               L.COARSE_BF16 if self.coarse == "bf16" else L.COARSE_F32, 0, *self.task_range)
        nbytes = lib.vsa_op_memory_bytes(self._lref, C.byref(desc))
        h = C.c_void_p()
        if nbytes == 0:  # invalid descriptor: let create report the reference's message
            check(lib.vsa_op_create(self._lref, C.byref(desc), None, 0, C.byref(h)))
        self._destroy()
        self._mem = torch.empty(nbytes, dtype=torch.uint8, device=self.device)
        check(lib.vsa_op_create(self._lref, C.byref(desc), C.c_void_p(self._mem.data_ptr()), nbytes, C.byref(h)))
        self._h = h
        self._views()

    def _destroy(self):
        if getattr(self, "_h", None) is not None:
            self._lib.vsa_op_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self._destroy()
        except Exception:
            pass

    def _bufs(self) -> L.vsa_op_buffers_t:
        b = L.vsa_op_buffers_t()
        check(self._lib.vsa_op_buffers(self._h, C.byref(b)))
        return b

    def _views(self):
        b = self._bufs()
        base = self._mem.data_ptr()
        B, H, d, nc, Lp = self.B, self.H, self.d, self.layout.num_cubes, self.layout.seq_padded
        kmax = max(self.top_k, self.max_sel_k)

        def view(ptr, shape, dt):
            if not ptr:
                return None
            n = 1
            for x in shape:
                n *= x
            es = torch.tensor([], dtype=dt).element_size()
            off = ptr - base
            return self._mem[off:off + n * es].view(dt).view(shape)

        f32, i32, dt = torch.float32, torch.int32, self.dtype
        self.q_t, self.k_t, self.v_t = (view(p, (B, H, Lp, d), dt) for p in (b.q_t, b.k_t, b.v_t))
        self.qc, self.kc, self.vc = (view(p, (B, H, nc, d), f32) for p in (b.qc, b.kc, b.vc))
        self.ac = view(b.ac, (B, H, nc, nc), f32)
        self.oc = view(b.oc_cube, (B, H, nc, d), f32)
        self.sel = view(b.sel, (B, H, nc, self.top_k), i32)
        self.selT_offs = view(b.selT_offs, (B * H, nc + 1), i32)
        self.selT_idx = view(b.selT_idx, (B * H, nc * kmax), i32)
        self.o_f = view(b.o_fine, (B, H, Lp, d), dt)
        self.lse = view(b.lse, (B, H, Lp), f32)
        self.dof = view(b.dof, (B, H, Lp, d), dt)
        self.delta = view(b.delta, (B, H, Lp), f32)
        self.doc = view(b.doc_cube, (B, H, nc, d), f32)
        self.dqc, self.dkc, self.dvc = (view(p, (B, H, nc, d), f32) for p in (b.dqc, b.dkc, b.dvc))
        self.gc, self.gf, self.dgc, self.dgf = (view(p, self.io_shape, dt) for p in (b.gc, b.gf, b.dgc, b.dgf))
        self.fine_sel, self.fine_k = self.sel, self.top_k

    # -- timing (native CUDA events between stages, no host gaps)
    def timing(self, enable: bool = True):
        check(self._lib.vsa_op_timing(self._h, 1 if enable else 0))
        self._timing = enable

    def stage_ms(self) -> dict:
        """Mean device time per stage over the calls since ``timing(True)`` (one sync)."""
        ms = (C.c_float * len(L.OP_STAGES))()
        calls = (C.c_int32 * 2)()
        check(self._lib.vsa_op_stage_ms(self._h, ms, calls))
        out = {n: float(ms[i]) for i, n in enumerate(L.OP_STAGES)}
        out["_calls"] = (int(calls[0]), int(calls[1]))
        return out

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

    def _override(self, sel_override):
        if sel_override is None:
            return None, 0
        if (not isinstance(sel_override, torch.Tensor) or sel_override.dtype != torch.int32 or not sel_override.is_cuda
                or sel_override.dim() != 4 or not sel_override.is_contiguous()):
            raise ValueError("BlockSelection: expected contiguous int32 [B, H, nc, k] on CUDA")
        if tuple(sel_override.shape[:3]) != tuple(self.sel.shape[:3]):
            raise ValueError("fine stage: selection does not match shapes")
        k = int(sel_override.shape[3])
        if not (1 <= k <= self.layout.num_cubes):
            raise ValueError("BlockSelection: k must be in [1, num_cubes]")
        if k > max(self.top_k, self.max_sel_k):  # grow the transposed-map capacity (control path)
            self._create(k)
        return _p(sel_override), k

    def forward(self, q, k, v, gc, gf=None, out=None, sel_override=None, check_inputs=True, before_fine=None):
        """vsa_forward (vsa.hpp:89-122) at attention level: gates are given.

        ``before_fine``: optional callable run after the coarse stage, before the
        fine kernel (the first reader of the gates) — e.g. to wait for a gate
        exchange that overlapped K1-K3."""
        if check_inputs:
            for t, n in ((q, "q"), (k, "k"), (v, "v"), (gc, "gate_coarse")):
                self._chk(t, n)
            if not self.adaptation:
                if gf is None:
                    raise ValueError("vsa_forward: missing fine gate")
                self._chk(gf, "gate_fine")
        ov, ok = self._override(sel_override)
        st = _stream()
        check(self._lib.vsa_op_forward_coarse(self._h, _p(q), _p(k), _p(v), ov, ok, st))
        self.fine_sel, self.fine_k = (sel_override, ok) if ov is not None else (self.sel, self.top_k)
        if out is None:
            out = torch.empty(self.io_shape, dtype=self.dtype, device=q.device)
        if before_fine is not None:
            before_fine()
        check(self._lib.vsa_op_forward_fine(self._h, _p(gc), _p(gf), _p(out), st))
        self._fwd = (q, k, v, gc, gf)  # the caller's tensors the artifacts point into stay alive
        return out

    def _ensure_workspace(self, device):
        if not self.bwd_workspace:
            return
        wsb = self._lib.vsa_op_workspace_bytes(self._h, self.fine_k)
        if self.ws is not None and self.ws.numel() >= wsb:
            return
        free, _ = torch.cuda.mem_get_info(device)
        if wsb > 0.6 * free:  # e.g. the dense baseline at 14B (all cubes): dQ recomputes S / dP instead
            self.ws = None
            check(self._lib.vsa_op_set_workspace(self._h, None, 0))
            return
        self.ws = torch.empty(wsb, dtype=torch.uint8, device=device)
        check(self._lib.vsa_op_set_workspace(self._h, _p(self.ws), wsb))

    @property
    def used_ds_workspace(self) -> bool:
        """Whether the last backward took the dS-materialising path (else dQ recomputed S / dP)."""
        return bool(self._bufs().bwd_used_workspace)

    def backward(self, dout, dq=None, dk=None, dv=None, dgc=None, dgf=None, check_inputs=True, before_finish=None):
        """vsa_backward (vsa.hpp:129-189) at attention level -> (dq, dk, dv, dgc, dgf).

        ``before_finish``: optional callable run between the prologue (dof, delta, gate and
        coarse gradients) and the fine backward."""
        if getattr(self, "_fwd", None) is None:
            raise ValueError("vsa_backward: missing or mismatched forward artifacts")
        if check_inputs:
            self._chk(dout, "dO")
        mk = lambda: torch.empty(self.io_shape, dtype=self.dtype, device=dout.device)
        dq = mk() if dq is None else dq
        dk = mk() if dk is None else dk
        dv = mk() if dv is None else dv
        dgc = mk() if dgc is None else dgc
        dgf = mk() if dgf is None else dgf
        self._ensure_workspace(dout.device)
        st = _stream()
        check(self._lib.vsa_op_backward_prologue(self._h, _p(dout), _p(dgc), _p(dgf), st))
        if before_finish is not None:  # e.g. complete delta with the other ranks' rows (sub-split)
            before_finish()
        check(self._lib.vsa_op_backward_finish(self._h, _p(dq), _p(dk), _p(dv), st))
        return dq, dk, dv, dgc, dgf

    # -- the reference's vsa_forward / vsa_backward with hidden states (model_dim > 0)
    def forward_hidden(self, hidden, params: "VsaParams", q, k, v, out=None, sel_override=None):
        """vsa_forward (vsa.hpp:89-122): gate projection (tcgen05 GEMM) + the operator."""
        if self.model_dim <= 0:
            raise ValueError("vsa_forward: the operator was created without model_dim (gate projection)")
        _check_hidden(hidden, self.B, self.seq_io, self.model_dim)
        params.check(self.model_dim, self.H, self.d)
        for t, n in ((q, "q"), (k, "k"), (v, "v")):
            self._chk(t, n)
        ov, ok = self._override(sel_override)
        if out is None:
            out = torch.empty(self.io_shape, dtype=self.dtype, device=q.device)
        bias = _gate_bias(params)
        check(self._lib.vsa_forward(self._h, _p(hidden), _p(params.gate_weight), _p(bias), _p(q), _p(k), _p(v), ov,
                                    ok, _p(out), _stream()))
        self.fine_sel, self.fine_k = (sel_override, ok) if ov is not None else (self.sel, self.top_k)
        self._fwd = (q, k, v, hidden, bias)
        return out

    def backward_hidden(self, hidden, params: "VsaParams", dout, dq=None, dk=None, dv=None):
        """vsa_backward (vsa.hpp:129-189): -> (dq, dk, dv, dhidden, dgate_weight, dgate_bias)."""
        if self.model_dim <= 0:
            raise ValueError("vsa_backward: the operator was created without model_dim (gate projection)")
        if getattr(self, "_fwd", None) is None:
            raise ValueError("vsa_backward: missing or mismatched forward artifacts")
        _check_hidden(hidden, self.B, self.seq_io, self.model_dim)
        self._chk(dout, "dO")
        mk = lambda: torch.empty(self.io_shape, dtype=self.dtype, device=dout.device)
        dq = mk() if dq is None else dq
        dk = mk() if dk is None else dk
        dv = mk() if dv is None else dv
        dhidden = torch.empty_like(hidden)
        dW = torch.empty(params.gate_weight.shape, dtype=torch.float32, device=dout.device)
        bias = _gate_bias(params)
        db = torch.empty(bias.shape, dtype=torch.float32, device=dout.device) if bias is not None else None
        self._ensure_workspace(dout.device)
        check(self._lib.vsa_backward(self._h, _p(hidden), _p(params.gate_weight), _p(dout), _p(dq), _p(dk), _p(dv),
                                     _p(dhidden), _p(dW), _p(db), _stream()))
        return dq, dk, dv, dhidden, dW, db

    @property
    def artifacts(self) -> CoarseArtifacts:
        return CoarseArtifacts(self.qc, self.kc, self.vc, self.ac, self.oc, self.sel, self.selT_offs, self.selT_idx,
                               self.pool, self.layout.cube_size)


def _check_hidden(hidden, B, S, md):
    """check_hidden (vsa.hpp:75-80)."""
    _cuda4(hidden, "hidden")
    if hidden.shape[1] != 1:
        raise ValueError("vsa: hidden states are [batch, 1, seq, model_dim]")
    if hidden.shape[0] != B or hidden.shape[2] != S or hidden.shape[3] != md:
        raise ValueError("vsa: hidden states do not match Q/K/V shapes")
    if hidden.dtype != torch.bfloat16:
        raise ValueError("gates: bf16 CUDA hidden and gate_weight required")


class VsaHostPipeline:
    """Forward + backward on HOST (pinned) tensors with the H2D / D2H copies
    overlapped with the kernels.

    Every (b, h) unit is independent (fine.hpp:65,129,172), so the B*H units are
    split into `chunks` groups; group i+1 is copied in on one stream while group
    i computes, and group i-1 is copied out on a third — `slots`-deep device
    input/output buffers, events for the hand-offs. Result == VsaOp on the whole batch.

    The copies are released at the operator's stage boundaries, so the PCIe fill
    and drain around the first and last group are as short as the data allows:
    q / k / v land before the gates (K1-K3 need only q / k / v; the gates are first
    read by the fine forward's combine), dO after them; O leaves after the forward,
    dGc / dGf after the backward prologue (K6a writes them), dQ / dK / dV last.
    """

    def __init__(self, layout: TileLayout, B: int, H: int, d: int, top_k: int, chunks: int = 6,
                 dtype=torch.bfloat16, device="cuda", slots: int = 3, **op_kwargs):
        units = B * H
        chunks = max(1, min(chunks, units))
        self.bounds = [(units * i) // chunks for i in range(chunks + 1)]
        self.units, self.d, self.S, self.dtype = units, d, layout.seq_len, dtype
        self.slots = max(2, int(slots))
        sizes = sorted({b - a for a, b in zip(self.bounds[:-1], self.bounds[1:])})
        cmax = sizes[-1]
        # one operator per group size, built here with the caller's options: run() never
        # allocates, and ragged groups compute the same operator. The compute stream runs
        # the groups in order, so one operator per size serves every buffer slot.
        self.ops = {c: VsaOp(layout, 1, c, d, top_k, dtype=dtype, device=device, **op_kwargs) for c in sizes}
        e = lambda: torch.empty((1, cmax, self.S, d), dtype=dtype, device=device)
        self.din = [[e() for _ in range(6)] for _ in range(self.slots)]
        self.dout = [[e() for _ in range(6)] for _ in range(self.slots)]
        self.s_in, self.s_out = torch.cuda.Stream(device), torch.cuda.Stream(device)
        self.h2d_bytes = 6 * units * self.S * d * torch.tensor([], dtype=dtype).element_size()
        self.d2h_bytes = self.h2d_bytes

    def run(self, hin, hout):
        """hin = (q, k, v, gc, gf, dO), hout = (O, dQ, dK, dV, dGc, dGf): pinned host [B,H,S,d]."""
        flat = lambda t: t.view(self.units, self.S, self.d)
        hin, hout = [flat(t) for t in hin], [flat(t) for t in hout]
        comp = torch.cuda.current_stream()
        n, ns = len(self.bounds) - 1, self.slots
        ev_comp, ev_out = [None] * n, [None] * n
        ev = torch.cuda.Event

        def copy_out(srcs, dsts, a, b, c, after):
            with torch.cuda.stream(self.s_out):
                self.s_out.wait_event(after)
                for dst, src in zip(dsts, srcs):
                    dst[a:b].copy_(src[0, :c], non_blocking=True)

        for i in range(n):
            a, b = self.bounds[i], self.bounds[i + 1]
            c, slot = b - a, i % ns
            di, do = self.din[slot], self.dout[slot]
            evs = []
            with torch.cuda.stream(self.s_in):
                if i >= ns:
                    self.s_in.wait_event(ev_comp[i - ns])     # slot's inputs consumed
                for grp in ((0, 1, 2), (3, 4), (5,)):         # q k v | gates | dO
                    for j in grp:
                        di[j][0, :c].copy_(hin[j][a:b], non_blocking=True)
                    evs.append(ev())
                    evs[-1].record(self.s_in)
            comp.wait_event(evs[0])
            if i >= ns:
                comp.wait_event(ev_out[i - ns])               # slot's outputs drained
            op = self.ops[c]
            v = lambda t: t[:, :c]  # [1, cmax, S, d] -> [1, c, S, d]: a contiguous prefix view
            op.forward(*(v(t) for t in di[:5]), out=v(do[0]), check_inputs=False,
                       before_fine=lambda: comp.wait_event(evs[1]))
            ev_fwd = ev()
            ev_fwd.record(comp)
            copy_out(do[:1], hout[:1], a, b, c, ev_fwd)
            comp.wait_event(evs[2])
            ev_pro = ev()
            op.backward(v(di[5]), *(v(t) for t in do[1:]), check_inputs=False,
                        before_finish=lambda: ev_pro.record(comp))
            copy_out(do[4:], hout[4:], a, b, c, ev_pro)
            ev_comp[i] = ev()
            ev_comp[i].record(comp)
            copy_out(do[1:4], hout[1:4], a, b, c, ev_comp[i])
            ev_out[i] = ev()
            ev_out[i].record(self.s_out)
        for i in range(max(0, n - ns), n):
            comp.wait_event(ev_out[i])


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

    @staticmethod
    def random_init(model_dim: int, heads: int, head_dim: int, top_k: int, rng=None, device="cuda",
                    dtype=torch.bfloat16) -> "VsaParams":
        """VsaParams::random_init (vsa.hpp:25-32): Wg ~ N(0, 1/model_dim), no bias.
        ``rng``: a numpy-compatible draw function f(rows, cols, std) -> array (e.g. the
        oracle's mt19937_64 randn_matrix for identical draws); default torch.randn."""
        std = 1.0 / float(model_dim) ** 0.5
        if rng is None:
            w = torch.randn((model_dim, 2 * heads * head_dim), device=device) * std
        else:
            w = torch.as_tensor(rng(model_dim, 2 * heads * head_dim, std), dtype=torch.float32).to(device)
        return VsaParams(w.to(dtype).contiguous(), None, int(top_k))

    @staticmethod
    def adaptation_init(model_dim: int, heads: int, head_dim: int, num_cubes: int, device="cuda",
                        dtype=torch.bfloat16) -> "VsaParams":
        """VsaParams::adaptation_init (vsa.hpp:35-42): Wg = 0, k = all cubes, Gf == 1."""
        return VsaParams(torch.zeros((model_dim, 2 * heads * head_dim), dtype=dtype, device=device), None,
                         int(num_cubes), adaptation=True)

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


# ----------------------------------------------------------------------------- vsa_forward / vsa_backward
@dataclass
class VsaOutput:
    """VsaOutput (vsa.hpp:56-63): the output plus the forward artifacts, resident in the
    operator context ``op`` (coarse artifacts, fine output / lse, gates, fine_sel)."""

    out: torch.Tensor
    op: VsaOp

    @property
    def coarse(self) -> CoarseArtifacts:
        return self.op.artifacts

    @property
    def fine(self) -> FineResult:
        return FineResult(self.op.o_f, None, self.op.lse.view(-1, self.op.layout.seq_padded))

    @property
    def gate_coarse(self) -> torch.Tensor:
        return self.op.gc

    @property
    def gate_fine(self) -> torch.Tensor:
        return self.op.gf

    @property
    def fine_sel(self) -> torch.Tensor:
        return self.op.fine_sel


@dataclass
class VsaGrads:
    """VsaGrads (vsa.hpp:65-71)."""

    dq: torch.Tensor
    dk: torch.Tensor
    dv: torch.Tensor
    dhidden: torch.Tensor
    dgate_weight: torch.Tensor
    dgate_bias: torch.Tensor | None


def vsa_forward(layout: TileLayout, hidden, q, k, v, params: VsaParams, sel_override=None,
                raster: bool = False) -> VsaOutput:
    """vsa_forward (vsa.hpp:89-122): gate projection, coarse stage (+ top-k), fine stage on
    the selection (or ``sel_override``), gated combine. Like the reference, q, k, v and
    hidden are tile-ordered ([B,H,Lp,d], [B,1,Lp,md]); ``raster=True`` takes raster-ordered
    tensors ([B,H,t*h*w,d], [B,1,t*h*w,md]) with the tiling fused into the kernels."""
    for t, n in ((q, "q"), (k, "k"), (v, "v")):
        _cuda4(t, n)
    if not (q.shape == k.shape == v.shape) or not (q.dtype == k.dtype == v.dtype):
        raise ValueError("attention: Q, K, V must share one shape")
    B, H, S, d = q.shape
    if S != (layout.seq_len if raster else layout.seq_padded):
        raise ValueError("vsa: sequence length does not match layout")
    _check_hidden(hidden, B, S, hidden.shape[3])
    params.check(hidden.shape[3], H, d)
    if not (1 <= params.top_k <= layout.num_cubes):
        raise ValueError("coarse_forward_select: k must be in [1, num_cubes]")
    op = VsaOp(layout, B, H, d, params.top_k, dtype=q.dtype, pool=params.pool, adaptation=params.adaptation,
               raster=raster, device=q.device, model_dim=hidden.shape[3], activation=int(params.activation),
               max_sel_k=0 if sel_override is None else int(sel_override.shape[3]))
    out = op.forward_hidden(hidden, params, q, k, v, sel_override=sel_override)
    return VsaOutput(out, op)


def vsa_backward(layout: TileLayout, fwd: VsaOutput, hidden, q, k, v, params: VsaParams, dout) -> VsaGrads:
    """vsa_backward (vsa.hpp:129-189): path split, gate gradients through the activation
    and projection, coarse + fine attention gradients."""
    if fwd is None or not isinstance(fwd, VsaOutput) or fwd.op is None:
        raise ValueError("vsa_backward: missing or mismatched forward artifacts")
    if dout.shape != q.shape:
        raise ValueError("vsa_backward: dO shape mismatch")
    op = fwd.op
    if tuple(q.shape) != op.io_shape:
        raise ValueError("vsa_backward: missing or mismatched forward artifacts")
    params.check(hidden.shape[3], op.H, op.d)
    dq, dk, dv, dh, dW, db = op.backward_hidden(hidden, params, dout)
    return VsaGrads(dq, dk, dv, dh, dW, db)
