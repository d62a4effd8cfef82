"""The paper's accuracy criterion with fitted weights (NEXT-1): the bf16 MFP with
the SDNet fitted on MFP-iteration boundaries through the chain's bf16 operand
rounding (weights/sdnet_fit_d128_mfp.npy, tools/collect_mfp_boundaries.py +
tools/fit_sdnet.py --bank --qat bf16) reaches MAE < 0.05
against the discrete solution (P:179's stop rule) on a GP-boundary domain, and the
same weights through the fp32 SIMT path agree with the fp64 oracle (fixed K)."""
import os

import numpy as np
import pytest

import oracle
from mfp_inputs import gp_boundary
from tests._refsolve import dst_laplace

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
W = os.path.join(ROOT, "weights", "sdnet_fit_d128_mfp.npy")


@pytest.fixture(scope="module")
def lib():
    import torch
    assert torch.cuda.is_available()
    import paper_2308_14258_b200 as mfp
    return mfp


@pytest.mark.skipif(not os.path.exists(W), reason="weights/sdnet_fit_d128_mfp.npy not generated")
def test_bf16_mfp_reaches_paper_mae(lib):
    n = 1024
    w = np.load(W)
    g = gp_boundary(n, n, 0)
    ref = dst_laplace(n, n, g.astype(np.float64))
    cfg = lib.make_config(n, n, precision=lib.BF16, subsolver=lib.SDNET, check_every=50)
    m = lib.Mfp(cfg, lib.make_net(gelu=1), w)
    u, _ = m.solve(g, 50, 0.0)
    for _ in range(60):
        mae = float(np.mean(np.abs(u - ref)))
        if mae < 0.05:
            break
        u, _ = m.solve(None, 50, 0.0)
    assert mae < 0.05


@pytest.mark.skipif(not os.path.exists(W), reason="weights/sdnet_fit_d128_mfp.npy not generated")
def test_fitted_mfp_weights_fp32_parity(lib):
    n = 128
    w = np.load(W)
    g = gp_boundary(n, n, 2)
    cfg = lib.make_config(n, n, precision=lib.FP32, subsolver=lib.SDNET, check_every=1)
    m = lib.Mfp(cfg, lib.make_net(gelu=0), w)
    u, _ = m.solve(g, 8, 0.0)
    r = oracle.mfp_run(oracle.MfpConfig(n, n), g.astype(np.float64), 8, params=w.astype(np.float64))
    assert np.max(np.abs(u - r.u)) / np.max(np.abs(r.u)) <= 1e-5
