"""GPU parity of the tensor-core paths with the EXACT erf GELU (mfp_sdnet_desc.gelu = 0).

The tensor-core embed keeps its conv weights in channel-pair order in the constant
bank, with the conv2 pairs halved only when the channel activation yields 2 GELU
(gelu = 1 / 2; api.cu); gelu = 0 takes the other branch (GELU proper, unscaled
pairs) in the embed (`ch_act2`) and the erf epilogues in the chains.  This file
pins that branch against the fp64 oracle (exact erf GELU) on every
tensor-core chain: d = 128 bf16 / fp16 (`k_chain_tc2`) and d = 256 bf16
(`k_chain_tc2w`), line lattice and final field after K iterations, 3e-3 per field
(north_star's 16-bit bar).  Inputs: seeded GP boundary, W-rand weights.
"""
import numpy as np
import pytest

import oracle
from mfp_inputs import gp_boundary, random_weights
from tests._lattice import lattice_to_global, line_mask

pytestmark = pytest.mark.gpu

TOL = 3e-3


@pytest.fixture(scope="module")
def lib():
    import torch
    assert torch.cuda.is_available()
    import paper_2308_14258_b200 as mfp
    return mfp


def rel_err(a, b, mask=None):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    if mask is not None:
        a, b = a[mask], b[mask]
    return np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-30)


@pytest.mark.parametrize("d,precision", [(128, 1), (128, 2), (256, 1)])
def test_tensorcore_erf_gelu_parity(lib, d, precision):
    nx = ny = 512
    t = 3
    g = gp_boundary(nx, ny, 3)
    w = random_weights(1, d=d)
    cfg = lib.make_config(nx, ny, precision=precision, subsolver=lib.SDNET)
    m = lib.Mfp(cfg, lib.make_net(d=d, gelu=0), w)
    u, rep = m.solve(g, t, 0.0)
    assert rep.iterations == t
    ocfg = oracle.MfpConfig(nx, ny, net=oracle.NetShape(d=d))
    ref = oracle.mfp_run(ocfg, g.astype(np.float64), t, params=w.astype(np.float64))
    L = lattice_to_global(m.lines(), nx, ny)
    assert rel_err(L, ref.lines, line_mask(nx, ny)) <= TOL
    assert rel_err(u, ref.u) <= TOL
    m.close()
