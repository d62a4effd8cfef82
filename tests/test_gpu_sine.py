"""The paper's evaluation problem g(x) = sin(2 pi x) on the GPU path.

The exact-subsolver MFP must converge to the grid's separable closed form
(tests/test_oracle_exact.py::sine_discrete_solution, itself pinned against the
DST solve); with the fitted SDNet (tools/fit_sdnet.py) the converged field is
held to the paper's accuracy criterion, MAE < 0.05 against that solution.
"""
import os

import numpy as np
import pytest

from mfp_inputs import sine_boundary
from tests.test_oracle_exact import sine_discrete_solution

pytestmark = pytest.mark.gpu
M = 32
H = 1.0 / 64.0
WFIT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "weights", "sdnet_fit_d128.npy")


@pytest.fixture(scope="module")
def lib():
    import torch
    assert torch.cuda.is_available()
    import paper_2308_14258_b200 as mfp
    return mfp


@pytest.mark.parametrize("nx,ny,grid", [(64, 128, (1, 1)), (256, 256, (1, 1)), (256, 256, (2, 2))])
def test_sine_exact_converges_to_closed_form(lib, nx, ny, grid):
    g = sine_boundary(nx, ny, H).astype(np.float32)
    cfg = lib.make_config(nx, ny, grid, precision=lib.FP32, subsolver=lib.EXACT_LAPLACE, check_every=8)
    m = lib.Mfp(cfg, lib.make_net(), None, rank=0 if grid == (1, 1) else lib.ALL_RANKS)
    u, rep = m.solve(g, 20000, 1e-7)
    assert rep.converged
    ref = sine_discrete_solution(nx, ny, H)
    assert np.max(np.abs(u - ref)) < 2e-4


@pytest.mark.skipif(not os.path.exists(WFIT), reason="fitted weights not generated (tools/fit_sdnet.py)")
@pytest.mark.parametrize("precision", [0, 2])
@pytest.mark.parametrize("nx,ny", [(64, 128), (256, 256)])
def test_sine_fitted_sdnet_mae(lib, precision, nx, ny):
    """Converged fitted-SDNet MFP vs the discrete solution: MAE < 0.05 (P:179's
    stop rule), the Fig. gfnet-eval quantity."""
    w = np.load(WFIT)
    g = sine_boundary(nx, ny, H).astype(np.float32)
    cfg = lib.make_config(nx, ny, precision=precision, subsolver=lib.SDNET, check_every=8)
    m = lib.Mfp(cfg, lib.make_net(gelu=1 if precision else 0), w)
    u, rep = m.solve(g, 4000, 1e-6)
    mae = float(np.mean(np.abs(u - sine_discrete_solution(nx, ny, H))))
    print(f"sine MAE nx={nx} ny={ny} precision={precision}: {mae:.4g} after {rep.iterations} iterations")
    assert mae < 0.05
