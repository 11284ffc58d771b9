# SPDX-License-Identifier: Apache-2.0
"""MacCounter on the device (tensor.hpp:36-39, fine.hpp:59-63): the fine-forward kernels
count the tiles they execute. At density 1/8 the counted MACs are exactly 1/8 of the
dense (all-cubes) run (test_fine.cpp:251-270), on the tcgen05 (bf16) and SIMT (fp32) paths."""
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("dtype,d", [(torch.bfloat16, 128), (torch.bfloat16, 64), (torch.float32, 64)])
def test_mac_counter_density_eighth(dtype, d):
    import paper_2505_13389_b200 as vsa

    L = vsa.TileLayout(8, 16, 16)  # nc = 32
    B, H, nc = 2, 2, L.num_cubes
    g = torch.Generator(device="cuda").manual_seed(3)
    q, k, v = (torch.randn((B, H, L.seq_len, d), generator=g, device="cuda").to(dtype) for _ in range(3))
    sparse = torch.stack([torch.randperm(nc, generator=torch.Generator().manual_seed(i))[:nc // 8].sort().values
                          for i in range(B * H * nc)]).to(torch.int32).view(B, H, nc, nc // 8).cuda()
    c8, cd = vsa.MacCounter(), vsa.MacCounter()
    vsa.fine_forward(L, q, k, v, sparse, counter=c8)
    vsa.fine_forward(L, q, k, v, vsa.all_cubes(B, H, nc), counter=cd)
    assert c8.tiles == B * H * nc * (nc // 8)
    assert cd.tiles == B * H * nc * nc
    assert c8.macs * 8 == cd.macs == B * H * nc * nc * 2 * 64 * 64 * d
    # the counter is off outside a counted call
    c0 = vsa.MacCounter()
    vsa.fine_forward(L, q, k, v, sparse)
    assert c0.tiles == 0
