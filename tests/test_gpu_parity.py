# SPDX-License-Identifier: Apache-2.0
"""GPU parity: the CUDA path through the C ABI (libvsa_b200.so) against the
oracle on the same seeded inputs. Bit-exact for tiling / pooling / the
fp32-coarse block map; north_star tolerances for outputs and gradients."""
import numpy as np
import pytest
import torch

import oracle as orc
from gpu_helpers import Problem, assert_close, host, rounded, to_dev

pytestmark = pytest.mark.gpu

TINY = dict(grid=(8, 16, 16), B=1, H=2, d=64, top_k=4)           # BASELINE configs[0]
PADDED = dict(grid=(9, 14, 22), B=2, H=2, d=64, top_k=6)          # non-divisible grid
D128 = dict(grid=(16, 16, 16), B=1, H=2, d=128, top_k=8)
ODD_NC = dict(grid=(12, 4, 20), B=1, H=3, d=64, top_k=5)         # nc = 15: odd row lengths everywhere
PADDED128 = dict(grid=(9, 14, 22), B=2, H=2, d=128, top_k=7)      # batch 2, padded, d = 128, odd k
DTYPES = [torch.float32, torch.bfloat16]


@pytest.fixture(scope="module")
def vsa():
    import paper_2505_13389_b200 as v

    v.lib()
    return v


def layout_of(vsa, p):
    return vsa.TileLayout(*p.grid, *p.cube, pad=True)


@pytest.mark.parametrize("cfg", [TINY, PADDED, D128], ids=["tiny", "padded", "d128"])
@pytest.mark.parametrize("dtype", DTYPES, ids=["f32", "bf16"])
def test_tile_pool_bitexact(vsa, cfg, dtype):
    p = Problem(**cfg, seed=11)
    L = layout_of(vsa, p)
    xs = [to_dev(x, dtype) for x in (p.q, p.k, p.v)]
    tiled, pooled = vsa.tile_pool(L, xs)
    for x, t, pl in zip((p.q, p.k, p.v), tiled, pooled):
        ref_t = p.pad_tile(rounded(x, dtype))
        np.testing.assert_array_equal(host(t), ref_t)
        np.testing.assert_array_equal(pl.cpu().numpy(), orc.pool_cubes(p.olayout, ref_t))
        np.testing.assert_array_equal(host(vsa.untile(L, t)), rounded(x, dtype))
    # max pooling
    _, pooled_max = vsa.tile_pool(L, xs[:1], vsa.POOL_MAX, want_tiled=False)
    np.testing.assert_array_equal(pooled_max[0].cpu().numpy(),
                                  orc.pool_cubes(p.olayout, p.pad_tile(rounded(p.q, dtype)), orc.KMAX))


def test_flatten_index_matches_oracle(vsa):
    L = vsa.TileLayout(4, 4, 4, 2, 2, 2)
    assert (vsa.flatten_index(L, 0, 0, 0), vsa.flatten_index(L, 1, 1, 1), vsa.flatten_index(L, 2, 0, 0)) == (0, 7, 32)
    with pytest.raises(ValueError):
        vsa.flatten_index(L, 4, 0, 0)
    with pytest.raises(ValueError):
        vsa.TileLayout(5, 4, 4, 2, 2, 2)


@pytest.mark.parametrize("cfg", [TINY, PADDED, D128, ODD_NC], ids=["tiny", "padded", "d128", "odd_nc"])
def test_coarse_blockmap_bitexact(vsa, cfg):
    """fp32 coarse stage: probabilities, Oc and the Top-K block map bit-exact."""
    p = Problem(**cfg, seed=31)
    L = layout_of(vsa, p)
    _, pooled = vsa.tile_pool(L, [to_dev(x, torch.float32) for x in (p.q, p.k, p.v)])
    art = vsa.coarse_from_pooled(L, *pooled, p.top_k)
    ref = orc.coarse_forward_select(p.olayout, p.pad_tile(p.q), p.pad_tile(p.k), p.pad_tile(p.v), p.top_k)
    np.testing.assert_array_equal(art.ac.cpu().numpy(), ref.ac)
    np.testing.assert_array_equal(art.sel.cpu().numpy(), ref.sel)
    np.testing.assert_array_equal(art.oc_cube.cpu().numpy(), ref.oc_cube)
    # transposed map == the reference's rev lists (fine.hpp:163-170)
    offs, idx = art.selT_offs.cpu().numpy(), art.selT_idx.cpu().numpy()
    nc, k = L.num_cubes, p.top_k
    sel = ref.sel.reshape(-1, nc, k)
    for u in range(sel.shape[0]):
        rev = [[] for _ in range(nc)]
        for qc in range(nc):
            for kc in sel[u, qc]:
                rev[kc].append(qc)
        for kc in range(nc):
            assert list(idx[u, offs[u, kc]:offs[u, kc + 1]]) == rev[kc]
        assert offs[u, nc] == nc * k


def test_topk_ties_lower_index(vsa):
    """Exact ties (identical pooled keys) go to the lower index (coarse.hpp:30-42)."""
    grid, d = (8, 16, 16), 64
    L = vsa.TileLayout(*grid)
    rng = orc.Rng(5)
    qc = orc.randn(rng, 1, 1, L.num_cubes, d, np.float32)
    kc = np.repeat(orc.randn(rng, 1, 1, 1, d, np.float32), L.num_cubes, axis=2)  # all keys equal
    kc[0, 0, 5] *= 1.5
    vc = orc.randn(rng, 1, 1, L.num_cubes, d, np.float32)
    art = vsa.coarse_from_pooled(L, *(to_dev(x, torch.float32) for x in (qc, kc, vc)), 3)
    ac = art.ac.cpu().numpy()[0, 0]
    assert (ac == ac[:, :1]).sum() >= ac.shape[1] - 2  # rows are genuinely tied
    ref_rows = np.stack([orc.topk_row(r, 3) for r in ac])
    np.testing.assert_array_equal(art.sel.cpu().numpy()[0, 0], ref_rows)


@pytest.mark.parametrize("cfg", [TINY, PADDED, D128, PADDED128], ids=["tiny", "padded", "d128", "padded128"])
@pytest.mark.parametrize("dtype", DTYPES, ids=["f32", "bf16"])
def test_fine_forward_backward(vsa, cfg, dtype):
    """fine_forward / fine_backward on tile-ordered inputs with a random block map."""
    p = Problem(**cfg, seed=51)
    L = layout_of(vsa, p)
    rng = orc.Rng(52)
    sel = orc.random_selection(p.B, p.H, L.num_cubes, p.top_k, rng)
    q, k, v, do = (p.pad_tile(rounded(x, dtype)) for x in (p.q, p.k, p.v, p.dout))
    fo, _, flse = orc.fine_forward(p.olayout, q, k, v, sel)
    fdq, fdk, fdv = orc.fine_backward(p.olayout, q, k, v, sel, do, flse)
    dq_, dk_, dv_, do_ = (to_dev(x, dtype) for x in (q, k, v, do))
    dsel = to_dev(sel, torch.int32)
    res = vsa.fine_forward(L, dq_, dk_, dv_, dsel)
    assert_close(host(res.out), fo, dtype, "fine out")
    # bf16: P is rounded to bf16 for the P.V product; at d = 64 the forward sums the
    # softmax denominator on the tensor core over the same bf16 P (row 64 of O^T,
    # fine_fwd_pp_sm100.cu), so lse carries that rounding (<= 2^-9 relative in l, a few
    # 1e-3 in log l where a few keys dominate a row); O itself is normalised consistently
    np.testing.assert_allclose(res.row_lse.cpu().numpy().reshape(flse.shape), flse,
                               atol=5e-3 if dtype != torch.float32 else 1e-4)
    g = vsa.fine_backward(L, dq_, dk_, dv_, dsel, do_, res.row_lse, out=res.out)
    for got, ref, n in zip(g, (fdq, fdk, fdv), ("dq", "dk", "dv")):
        assert_close(host(got), ref, dtype, n)
    # the recompute-dQ variant (no dS workspace) agrees as well
    g2 = vsa.fine_backward(L, dq_, dk_, dv_, dsel, do_, res.row_lse, out=res.out, workspace=False)
    for got, ref, n in zip(g2, (fdq, fdk, fdv), ("dq", "dk", "dv")):
        assert_close(host(got), ref, dtype, n + " (recompute)")
    # unselected key cubes: exactly zero dK/dV (test_fine.cpp:149-169)
    used = np.zeros((p.B, p.H, L.num_cubes), bool)
    for b in range(p.B):
        for h in range(p.H):
            used[b, h, np.unique(sel[b, h])] = True
    dk_h = host(g[1]).reshape(p.B, p.H, L.num_cubes, -1)
    assert (dk_h[~used] == 0).all()


@pytest.mark.parametrize("dtype", DTYPES, ids=["f32", "bf16"])
def test_dense_baseline_is_dense_attention(vsa, dtype):
    """Full selection (BlockSelection::all_cubes) == dense attention (test_fine.cpp:21-42)."""
    p = Problem(grid=(4, 8, 8), B=1, H=2, d=64, top_k=4, seed=53)
    L = layout_of(vsa, p)
    q, k, v = (p.pad_tile(rounded(x, dtype)) for x in (p.q, p.k, p.v))
    dense, _, _ = orc.dense_forward(q, k, v)
    res = vsa.fine_forward(L, *(to_dev(x, dtype) for x in (q, k, v)), vsa.all_cubes(p.B, p.H, L.num_cubes))
    assert_close(host(res.out), dense, dtype, "dense")


@pytest.mark.parametrize("cfg", [TINY, PADDED, D128, PADDED128], ids=["tiny", "padded", "d128", "padded128"])
@pytest.mark.parametrize("dtype", DTYPES, ids=["f32", "bf16"])
def test_vsa_op_end_to_end(vsa, cfg, dtype):
    """The full operator, raster in / raster out: forward, block map, backward incl. gate grads."""
    p = Problem(**cfg, seed=71)
    L = layout_of(vsa, p)
    op = vsa.VsaOp(L, p.B, p.H, p.d, p.top_k, dtype=dtype)
    ins = [to_dev(x, dtype) for x in (p.q, p.k, p.v, p.gc, p.gf)]
    out = op.forward(*ins)
    ref = p.oracle(dtype)
    if dtype == torch.float32:
        np.testing.assert_array_equal(op.sel.cpu().numpy(), ref["sel"])
    else:  # bf16 inputs: the block map is bit-exact against the oracle on the same rounded inputs
        np.testing.assert_array_equal(op.sel.cpu().numpy(), ref["sel"])
    assert_close(host(out), ref["out"], dtype, "out")
    dq, dk, dv, dgc, dgf = op.backward(to_dev(p.dout, dtype))
    for got, n in ((dq, "dq"), (dk, "dk"), (dv, "dv"), (dgc, "dgc"), (dgf, "dgf")):
        assert_close(host(got), ref[n], dtype, n)


def test_sel_override_and_adaptation(vsa):
    """sel_override (vsa.hpp:93,115) with adaptation (Gf == 1, k = nc): equals dense attention."""
    p = Problem(grid=(4, 8, 8), B=1, H=2, d=64, top_k=4, seed=73)
    L = layout_of(vsa, p)
    dt = torch.float32
    op = vsa.VsaOp(L, p.B, p.H, p.d, L.num_cubes, dtype=dt, adaptation=True)
    gc0 = torch.zeros((p.B, p.H, L.seq_len, p.d), dtype=dt, device="cuda")
    out = op.forward(*(to_dev(x, dt) for x in (p.q, p.k, p.v)), gc0, None)
    q, k, v = (p.pad_tile(x) for x in (p.q, p.k, p.v))
    dense, _, _ = orc.dense_forward(q, k, v)
    assert_close(host(out), p.untile_crop(dense), dt, "adaptation == dense")
    sel = orc.random_selection(p.B, p.H, L.num_cubes, 3, orc.Rng(74))
    op2 = vsa.VsaOp(L, p.B, p.H, p.d, 2, dtype=dt)
    out2 = op2.forward(*(to_dev(x, dt) for x in (p.q, p.k, p.v, p.gc, p.gf)), sel_override=to_dev(sel, torch.int32))
    ref = p.oracle(dt, sel_override=sel, backward=False)
    assert_close(host(out2), ref["out"], dt, "sel_override")


def test_invalid_inputs_raise(vsa):
    L = vsa.TileLayout(4, 8, 8)
    q = torch.zeros((1, 1, L.seq_padded, 64), dtype=torch.bfloat16, device="cuda")
    nc = L.num_cubes
    for bad in (torch.tensor([[3, 1]] * nc, dtype=torch.int32), torch.tensor([[1, 1]] * nc, dtype=torch.int32),
                torch.full((nc, 1), nc, dtype=torch.int32)):
        with pytest.raises(ValueError):
            vsa.fine_forward(L, q, q, q, bad.view(1, 1, nc, -1).cuda())
    with pytest.raises(ValueError):
        vsa.VsaOp(L, 1, 1, 64, 0)
    with pytest.raises(ValueError):
        vsa.VsaOp(L, 1, 1, 64, nc + 1)
    op = vsa.VsaOp(L, 1, 1, 64, 2)
    with pytest.raises(ValueError):
        op.backward(torch.zeros((1, 1, L.seq_len, 64), dtype=torch.bfloat16, device="cuda"))


@pytest.mark.parametrize("dtype", DTYPES, ids=["f32", "bf16"])
def test_backward_deterministic(vsa, dtype):
    p = Problem(**D128, seed=81)
    L = layout_of(vsa, p)
    op = vsa.VsaOp(L, p.B, p.H, p.d, p.top_k, dtype=dtype)
    ins = [to_dev(x, dtype) for x in (p.q, p.k, p.v, p.gc, p.gf)]
    do = to_dev(p.dout, dtype)
    o1 = op.forward(*ins).clone()
    g1 = [t.clone() for t in op.backward(do)]
    o2 = op.forward(*ins)
    g2 = op.backward(do)
    assert torch.equal(o1, o2)
    for a, b in zip(g1, g2):
        assert torch.equal(a, b)


def test_host_pipeline_matches_resident_op(vsa):
    """VsaHostPipeline (chunked, copy-overlapped, pinned host I/O) == VsaOp bitwise."""
    p = Problem(grid=(8, 16, 16), B=2, H=3, d=128, top_k=4, seed=91)
    L = layout_of(vsa, p)
    dt = torch.bfloat16
    ins = [to_dev(x, dt) for x in (p.q, p.k, p.v, p.gc, p.gf, p.dout)]
    op = vsa.VsaOp(L, p.B, p.H, p.d, p.top_k, dtype=dt)
    ref = [op.forward(*ins[:5]).clone()] + [t.clone() for t in op.backward(ins[5])]
    for chunks, slots in ((1, 2), (4, 2), (6, 3), (6, 4), (5, 3)):  # ragged groups at 5 chunks of 6 units
        pipe = vsa.VsaHostPipeline(L, p.B, p.H, p.d, p.top_k, chunks=chunks, dtype=dt, slots=slots)
        hin = [t.cpu().pin_memory() for t in ins]
        hout = [torch.empty(t.shape, dtype=dt, pin_memory=True) for t in ref]
        for _ in range(2):  # the second run reuses every slot's buffers and events
            pipe.run(hin, hout)
        torch.cuda.synchronize()
        for a, b in zip(hout, ref):
            assert torch.equal(a, b.cpu()), f"chunks={chunks} slots={slots}"


@pytest.mark.parametrize("d", [128, 64])
def test_fine_backward_skewed_transposed_map(vsa, d):
    """Persistent dK/dV with the dynamic key-cube hand-out (2048 tasks over the SMs,
    ring wrap-around, double-buffered accumulators, K/V reloads): a block map whose
    transposed lists are very uneven (8 hot key cubes in every other row, many key
    cubes selected by nobody) against the SIMT path on the same bf16 inputs, with and
    without the dS workspace; and run-to-run bitwise determinism."""
    g = torch.Generator(device="cuda").manual_seed(7)
    L = vsa.TileLayout(16, 32, 32)  # nc = 256
    B, H, k, nc = 1, 8, 8, 256
    rnd = lambda: (torch.randn((B, H, L.seq_len, d), generator=g, device="cuda")).bfloat16()
    q, kk, v, do = rnd(), rnd(), rnd(), rnd()
    gen = np.random.default_rng(8)
    rows = []
    for _ in range(B * H * nc):
        hot = gen.choice(8, 4, replace=False) if gen.random() < 0.5 else np.array([], dtype=np.int64)
        rest = gen.choice(np.arange(8 + 64, nc), k - len(hot), replace=False)  # cubes 8..71: never selected
        rows.append(np.sort(np.concatenate([hot, rest])))
    sel = torch.from_numpy(np.stack(rows).astype(np.int32)).view(B, H, nc, k).cuda()
    res = vsa.fine_forward(L, q, kk, v, sel)
    ref = vsa.fine_backward(L, q, kk, v, sel, do, res.row_lse, out=res.out, force_simt=True)
    a = vsa.fine_backward(L, q, kk, v, sel, do, res.row_lse, out=res.out)
    b = vsa.fine_backward(L, q, kk, v, sel, do, res.row_lse, out=res.out)
    c = vsa.fine_backward(L, q, kk, v, sel, do, res.row_lse, out=res.out, workspace=False)
    for got, r, n in zip(a, ref, ("dq", "dk", "dv")):
        assert_close(host(got), host(r), torch.bfloat16, n)
    for x, y in zip(a, b):
        assert torch.equal(x, y)
    for got, r, n in zip(c, ref, ("dq", "dk", "dv")):
        assert_close(host(got), host(r), torch.bfloat16, n + " (no workspace)")
    dk = a[1].view(B, H, nc, 64, d)
    assert (dk[:, :, 8:72] == 0).all()  # key cubes nobody selected


@pytest.mark.parametrize("top_k", [1, 3, 15], ids=["k1", "k3", "k15"])
def test_fine_odd_and_unit_k(vsa, top_k):
    """Single-cube last pairs on the tcgen05 path (k = 1: every pair is a single cube;
    odd k: one per row) in the forward, the transposed-map pairs of dK/dV and dQ."""
    p = Problem(grid=(16, 16, 16), B=1, H=2, d=128, top_k=top_k, seed=57)
    L = layout_of(vsa, p)
    sel = orc.random_selection(p.B, p.H, L.num_cubes, p.top_k, orc.Rng(58))
    q, k, v, do = (p.pad_tile(rounded(x, torch.bfloat16)) for x in (p.q, p.k, p.v, p.dout))
    fo, _, flse = orc.fine_forward(p.olayout, q, k, v, sel)
    fdq, fdk, fdv = orc.fine_backward(p.olayout, q, k, v, sel, do, flse)
    dq_, dk_, dv_, do_ = (to_dev(x, torch.bfloat16) for x in (q, k, v, do))
    dsel = to_dev(sel, torch.int32)
    res = vsa.fine_forward(L, dq_, dk_, dv_, dsel)
    assert_close(host(res.out), fo, torch.bfloat16, "fine out")
    g = vsa.fine_backward(L, dq_, dk_, dv_, dsel, do_, res.row_lse, out=res.out)
    for got, ref, n in zip(g, (fdq, fdk, fdv), ("dq", "dk", "dv")):
        assert_close(host(got), ref, torch.bfloat16, n)


@pytest.mark.parametrize("cfg", [TINY, PADDED128], ids=["tiny", "padded128"])
@pytest.mark.parametrize("dtype", DTYPES, ids=["f32", "bf16"])
def test_vsa_op_max_pool(vsa, cfg, dtype):
    """PoolMode::kMax end to end (coarse.hpp:47-65 forward, 172-176 first-argmax unpool)."""
    p = Problem(**cfg, seed=73)
    L = layout_of(vsa, p)
    op = vsa.VsaOp(L, p.B, p.H, p.d, p.top_k, dtype=dtype, pool=vsa.POOL_MAX)
    out = op.forward(*[to_dev(x, dtype) for x in (p.q, p.k, p.v, p.gc, p.gf)])
    ref = p.oracle(dtype, pool=orc.KMAX)
    np.testing.assert_array_equal(op.sel.cpu().numpy(), ref["sel"])
    assert_close(host(out), ref["out"], dtype, "out")
    for got, n in zip(op.backward(to_dev(p.dout, dtype)), ("dq", "dk", "dv", "dgc", "dgf")):
        assert_close(host(got), ref[n], dtype, n)


SWEEP_CUBES = [(4, 4, 4), (2, 4, 8), (1, 8, 8), (4, 2, 8), (8, 8, 1)]


@pytest.mark.parametrize("case", range(10))
def test_randomized_sweep_tcgen05(vsa, case):
    """Seeded sweep in the spirit of the reference's verify suite (verify.hpp:99-134):
    random grids (padded or not), 64-token cube shapes of every orientation, batch,
    heads, d in {64, 128} and k in [1, nc] through the full bf16 operator vs the oracle."""
    g = np.random.default_rng(1000 + case)
    cube = SWEEP_CUBES[case % len(SWEEP_CUBES)]
    grid = tuple(int(c * g.integers(1, 4) + (g.integers(0, c) if case % 3 == 0 else 0)) for c in cube)
    grid = tuple(max(x, 1) for x in grid)
    B, H, d = int(g.integers(1, 3)), int(g.integers(1, 4)), int(g.choice([64, 128]))
    nc = int(np.prod([(e + c - 1) // c for e, c in zip(grid, cube)]))
    p = Problem(grid=grid, B=B, H=H, d=d, top_k=int(g.integers(1, nc + 1)), seed=90 + case, cube=cube)
    L = layout_of(vsa, p)
    assert L.num_cubes == nc
    op = vsa.VsaOp(L, p.B, p.H, p.d, p.top_k)
    out = op.forward(*[to_dev(x, torch.bfloat16) for x in (p.q, p.k, p.v, p.gc, p.gf)])
    ref = p.oracle(torch.bfloat16)
    np.testing.assert_array_equal(op.sel.cpu().numpy(), ref["sel"])
    assert_close(host(out), ref["out"], torch.bfloat16, "out")
    for got, n in zip(op.backward(to_dev(p.dout, torch.bfloat16)), ("dq", "dk", "dv", "dgc", "dgf")):
        assert_close(host(got), ref[n], torch.bfloat16, n)
