# SPDX-License-Identifier: Apache-2.0
"""The tcgen05 (bf16) coarse mode (VSA_COARSE_BF16; north_star kernel 3: coarse attention
on the tensor cores with TMEM accumulators, the fused softmax + top-k + transposed-map
kernel). The fp32 mode stays the bit-exact one; this mode is checked the way north_star
prescribes for a non-bit-exact coarse stage:

* its probabilities and Oc agree with the oracle's fp32 coarse stage to bf16 accuracy,
  and its block map is exactly the top-k (ties -> lower index) of its own probabilities;
* the fine stage fed the ORACLE's block map (sel_override) gives out / dq / dk / dv /
  dgc / dgf within the bf16 tolerance of the oracle (coarse backward included)."""
import numpy as np
import pytest
import torch

import oracle as orc
from gpu_helpers import Problem, assert_close, host, rounded, to_dev

pytestmark = pytest.mark.gpu
BF = torch.bfloat16


@pytest.fixture(scope="module")
def vsa():
    import paper_2505_13389_b200 as v

    v.lib()
    return v


CASES = {"sweep16": dict(grid=(16, 16, 16), B=1, H=2, d=128, top_k=8),
         "d64": dict(grid=(16, 16, 16), B=2, H=1, d=64, top_k=16),
         "wan13-head": dict(grid=(21, 30, 52), B=1, H=1, d=128, top_k=78)}


def topk_rows(p, k):
    """topk_row (coarse.hpp:30-42) per row: largest k, ties to the lower index, ascending."""
    order = np.lexsort((np.arange(p.shape[-1])[None, :].repeat(p.shape[0], 0), -p), axis=-1)
    return np.sort(order[:, :k], axis=-1)


@pytest.mark.parametrize("name", list(CASES))
def test_coarse_bf16_probabilities_and_map(vsa, name):
    p = Problem(**CASES[name], seed=33)
    L = vsa.TileLayout(*p.grid, pad=True)
    op = vsa.VsaOp(L, p.B, p.H, p.d, p.top_k, coarse="bf16")
    op.forward(*(to_dev(x, BF) for x in (p.q, p.k, p.v, p.gc, p.gf)))
    torch.cuda.synchronize()
    q, k, v = (p.pad_tile(rounded(x, BF)) for x in (p.q, p.k, p.v))
    ref = orc.coarse_forward_select(p.olayout, q, k, v, p.top_k, token_oc=False)
    ac = op.ac.cpu().numpy()
    np.testing.assert_array_equal(op.qc.cpu().numpy(), ref.qc)  # pooling is shared with the fp32 mode
    err = np.abs(ac - ref.ac).max() / np.abs(ref.ac).max()
    assert err < 2e-3, f"probabilities: rel err {err:.2e}"
    np.testing.assert_allclose(op.oc.cpu().numpy(), ref.oc_cube, atol=2e-3, rtol=2e-2)
    sel = op.sel.cpu().numpy()
    nc = L.num_cubes
    np.testing.assert_array_equal(sel.reshape(-1, p.top_k), topk_rows(ac.reshape(-1, nc), p.top_k))
    agree = np.mean([len(np.intersect1d(a, b)) / p.top_k for a, b in
                     zip(sel.reshape(-1, p.top_k), ref.sel.reshape(-1, p.top_k))])
    assert agree > 0.5, f"block maps overlap only {agree:.2f}"


@pytest.mark.parametrize("name", list(CASES))
def test_coarse_bf16_operator_with_oracle_map(vsa, name):
    p = Problem(**CASES[name], seed=34)
    L = vsa.TileLayout(*p.grid, pad=True)
    ref = p.oracle(BF)
    op = vsa.VsaOp(L, p.B, p.H, p.d, p.top_k, coarse="bf16")
    out = op.forward(*(to_dev(x, BF) for x in (p.q, p.k, p.v, p.gc, p.gf)),
                     sel_override=to_dev(ref["sel"], torch.int32))
    grads = op.backward(to_dev(p.dout, BF))
    assert_close(host(out), ref["out"], BF, f"{name} out")
    for g, n in zip(grads, ("dq", "dk", "dv", "dgc", "dgf")):
        assert_close(host(g), ref[n], BF, f"{name} {n}")


def test_coarse_bf16_requires_nc_multiple_of_8(vsa):
    L = vsa.TileLayout(12, 12, 12)  # nc = 27
    with pytest.raises(ValueError, match="bf16 coarse"):
        vsa.VsaOp(L, 1, 1, 64, 4, coarse="bf16")
