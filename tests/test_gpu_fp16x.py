"""GPU parity of the tensor-core accuracy mode MFP_FP16X (split fp16 activations,
fp16 weights, `k_chain_tc2s`) and of the accurate GELU form (mfp_sdnet_desc.gelu = 2).

VERDICT r1 "what's weak" 3 / "next" 7: with TRAINED weights the single-rounding
tensor-core modes miss north_star's 3e-3 per-field bar (bf16 1.5e-2, fp16 2.3e-3
per batch / 4e-3 per field).  The emulation that motivated the mode
(DESIGN.md §7): exact activations + fp16 weights + an accurate GELU = 4.6e-4 of
max|y| on the fitted network.  Here the same bar as the fp32 twin's companions:
3e-3 per batch AND per field with the fitted weights, against the fp64 oracle
(exact-erf GELU).
"""
import os

import numpy as np
import pytest

import oracle
from mfp_inputs import gp_boundary, random_boundaries, random_weights
from tests._lattice import lattice_to_global, line_mask

pytestmark = pytest.mark.gpu

TOL = 3e-3
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
WFIT = os.path.join(ROOT, "weights", "sdnet_fit_d128.npy")
WFIT_MFP = os.path.join(ROOT, "weights", "sdnet_fit_d128_mfp.npy")


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
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-30))


@pytest.mark.parametrize("wfile", [WFIT, WFIT_MFP])
@pytest.mark.parametrize("qs", [0, 1])
def test_fp16x_fitted_batch(lib, wfile, qs):
    import torch
    w = np.load(wfile)
    cfg = lib.make_config(128, 128, precision=lib.FP16X, subsolver=lib.SDNET, check_every=1)
    m = lib.Mfp(cfg, lib.make_net(gelu=2), w)
    gb = random_boundaries(500, seed=13)
    out = m.sdnet_batch(torch.from_numpy(gb).cuda(), qs).cpu().numpy()
    q = oracle.writeset(0, 0)[1] if qs == 0 else oracle.interior_queries()
    ref = oracle.sdnet_forward(w.astype(np.float64), gb.astype(np.float64), q)
    e = rel_err(out, ref)
    print(f"FP16X fitted batch ({os.path.basename(wfile)}, q set {qs}): {e:.2e}")
    assert e <= TOL
    m.close()


@pytest.mark.parametrize("wfile", [WFIT, WFIT_MFP])
@pytest.mark.parametrize("nx,ny,t,grid", [(128, 128, 10, (1, 1)), (512, 512, 6, (1, 1)), (256, 256, 8, (2, 2))])
def test_fp16x_fitted_field(lib, wfile, nx, ny, t, grid):
    """The north_star per-field bar with trained weights: lines and the final
    field after t iterations, 1x1 and the 2x2 D1 emulation."""
    w = np.load(wfile)
    cfg = lib.make_config(nx, ny, grid, precision=lib.FP16X, subsolver=lib.SDNET, check_every=1)
    rank = 0 if grid == (1, 1) else lib.ALL_RANKS
    m = lib.Mfp(cfg, lib.make_net(gelu=2), w, rank=rank)
    g = gp_boundary(nx, ny, 1)
    u, rep = m.solve(g, t, 0.0)
    r = oracle.mfp_run(oracle.MfpConfig(nx, ny, Py=grid[0], Px=grid[1]), g.astype(np.float64), t,
                       params=w.astype(np.float64))
    e = rel_err(u, r.u)
    print(f"FP16X fitted field {nx}x{ny} {grid}: {e:.2e}")
    assert e <= TOL
    if grid == (1, 1):
        assert rel_err(lattice_to_global(m.lines(), nx, ny), r.lines, line_mask(nx, ny)) <= TOL
    m.close()


@pytest.mark.parametrize("B", [1, 333, 16384])
def test_fp16x_wrand_batch_many_tiles(lib, B):
    """W-rand batches up to 16,384 subdomains (3,904 pair tiles: ~26 per tile slot
    of the two-slot kernel), sampled rows vs the oracle at the fp16 bar."""
    import torch
    w = random_weights(0)
    cfg = lib.make_config(4096, 4096, precision=lib.FP16X, subsolver=lib.SDNET, check_every=16)
    m = lib.Mfp(cfg, lib.make_net(gelu=2), w)
    gb = random_boundaries(B, seed=31)
    out = m.sdnet_batch(torch.from_numpy(gb).cuda(), 0).cpu().numpy()
    rows = np.unique(np.concatenate([[0, B - 1], np.arange(0, B, max(1, B // 89))]))
    ref = oracle.sdnet_forward(w.astype(np.float64), gb[rows].astype(np.float64), oracle.writeset(0, 0)[1])
    assert rel_err(out[rows], ref) <= TOL
    m.close()


def test_fp16x_rejects_d256(lib):
    cfg = lib.make_config(128, 128, precision=lib.FP16X, subsolver=lib.SDNET, check_every=1)
    with pytest.raises(lib.MfpError) as e:
        lib.Mfp(cfg, lib.make_net(d=256, gelu=2), random_weights(0, d=256))
    assert e.value.status == 1


@pytest.mark.parametrize("precision", [1, 2])
def test_accurate_gelu_single_rounding_modes(lib, precision):
    """gelu = 2 on the bf16 / fp16 chains (k_chain_tc2 GELU = 2): field parity at
    the per-field bar with W-rand weights (512^2, K = 4)."""
    nx = ny = 512
    w = random_weights(0)
    cfg = lib.make_config(nx, ny, precision=precision, subsolver=lib.SDNET, check_every=1)
    m = lib.Mfp(cfg, lib.make_net(gelu=2), w)
    g = gp_boundary(nx, ny, 3)
    u, _ = m.solve(g, 4, 0.0)
    r = oracle.mfp_run(oracle.MfpConfig(nx, ny), g.astype(np.float64), 4, params=w.astype(np.float64))
    assert rel_err(u, r.u) <= TOL
    m.close()
