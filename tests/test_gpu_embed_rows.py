"""The tensor-core embed at every per-CTA round size it picks (kernels_embed_tc.cu):
rows per CTA = the smallest multiple of 16 that covers B over the SMs, so 1..8
subdomains per warp — pairs interleaved, an odd last one alone — and, past 148 x 128
subdomains, several rounds per CTA (the next round's perimeters staged by TMA while
the current one is embedded).  mfp_sdnet_batch at batch sizes that hit each of those
against the fp64 oracle forward on sampled rows, d = 128 and d = 256, bf16; same bars
as the other batch tests (3e-3 of S = sum|wo_i h_i|)."""
import numpy as np
import pytest

import oracle
from mfp_inputs import random_boundaries, random_weights
from tests._refnet import torch_sdnet

pytestmark = pytest.mark.gpu

TC_TOL = 3e-3


@pytest.fixture(scope="module")
def lib():
    import torch
    assert torch.cuda.is_available()
    import paper_2308_14258_b200 as mfp
    return mfp


# B -> rows per CTA on 148 SMs: 3000 -> 32 (2 per warp), 7000 -> 48 (3), 9000 -> 64 (4),
# 12000 -> 96 (6), 17000 -> 128 (8), 40000 -> 128 with 2-3 rounds per CTA
@pytest.mark.parametrize("d", [128, 256])
@pytest.mark.parametrize("B", [3000, 7000, 9000, 12000, 17000, 40000])
def test_embed_round_sizes_batch_parity(lib, d, B):
    import torch
    w = random_weights(2, d=d)
    cfg = lib.make_config(4096, 4096, precision=lib.BF16, subsolver=lib.SDNET, check_every=16)
    m = lib.Mfp(cfg, lib.make_net(d=d, gelu=1), w)
    gb = random_boundaries(B, seed=53)
    out = m.sdnet_batch(torch.from_numpy(gb).cuda(), 0).cpu().numpy()
    assert np.isfinite(out).all()
    rows = np.unique(np.concatenate([[0, 1, B - 2, B - 1], np.arange(0, B, max(1, B // 61)),
                                     np.arange(15, B, max(1, B // 37))]))
    q = oracle.writeset(0, 0)[1]
    ref = oracle.sdnet_forward(w.astype(np.float64), gb[rows].astype(np.float64), q, net=oracle.NetShape(d=d))
    _, S = torch_sdnet(w, gb[rows], q, d=d, return_scale=True)
    assert np.max(np.abs(out[rows] - ref) / S) <= TC_TOL
    m.close()
