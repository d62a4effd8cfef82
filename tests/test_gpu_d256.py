"""GPU parity of the d = 256 SDNet variant (SURVEY §8(b) d = 128 | 256, G7; PAPER.md
P:239-241 fixes the architecture's form, not its width).

The wide variant runs its own kernels: the tensor-core embed with two W1 halves
through one TMA-reloaded buffer, the SIMT embed and fp32 chain templated on d
(weights streamed through shared memory in K-chunks at d = 256), and the CTA-pair
tcgen05 chain `k_chain_tc2w` (M = N = 256, two tile slots, weight K-chunks streamed
by TMA through a four-stage ring).  Same bars as d = 128 (north_star): fp32
<= 1e-5 scale-relative, bf16 / fp16 <= 3e-3 per field after K iterations; batch
outputs as in test_gpu_parity.check_batch.
"""
import numpy as np
import pytest

import oracle
from mfp_inputs import gp_boundary, random_boundaries, random_weights
from tests._lattice import lattice_to_global, line_mask, owner_view
from tests._refnet import torch_sdnet

pytestmark = pytest.mark.gpu

D = 256
FP32_TOL = 1e-5
TC_TOL = 3e-3
NET = oracle.NetShape(d=D)


@pytest.fixture(scope="module")
def lib():
    import torch
    assert torch.cuda.is_available()
    import paper_2308_14258_b200 as mfp
    return mfp


@pytest.fixture(scope="module")
def w():
    return random_weights(0, d=D)


def rel_err(a, b, mask=None):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    if mask is not None:
        a, b = a[mask], b[mask]
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-30))


def check_batch(out, ref, precision, S):
    if precision == 0:
        assert rel_err(out, ref) <= FP32_TOL
    elif precision == 2:
        assert rel_err(out, ref) <= TC_TOL
    else:   # bf16: W-rand head cancellation, judged against S = sum|wo_i h_i|
        assert np.max(np.abs(out - ref) / S) <= TC_TOL


@pytest.mark.parametrize("precision", [0, 1, 2])
@pytest.mark.parametrize("qs,B", [(0, 1000), (0, 16384), (1, 37), (0, 1)])
def test_d256_batch_parity(lib, w, precision, qs, B):
    """mfp_sdnet_batch at d = 256 vs the fp64 oracle.  B = 16,384 at q = 61 is
    3,904 pair tiles over 74 CTA pairs: ~26 per tile slot, so the weight ring
    cycles through ~80 fills and every mbarrier parity flips many times."""
    import torch
    cfg = lib.make_config(4096, 4096, precision=precision, subsolver=lib.SDNET, check_every=16)
    m = lib.Mfp(cfg, lib.make_net(d=D, gelu=0 if precision == 0 else 1), w)
    gb = random_boundaries(B, seed=29)
    out = m.sdnet_batch(torch.from_numpy(gb).cuda(), qs).cpu().numpy()
    rows = np.unique(np.concatenate([[0, B - 1], np.arange(0, B, max(1, B // 97))]))
    q = oracle.writeset(0, 0)[1] if qs == 0 else oracle.interior_queries()
    ref = oracle.sdnet_forward(w.astype(np.float64), gb[rows].astype(np.float64), q, net=NET)
    _, S = torch_sdnet(w, gb[rows], q, d=D, return_scale=True)
    check_batch(out[rows], ref, precision, S)
    m.close()


@pytest.mark.parametrize("precision", [0, 1, 2])
@pytest.mark.parametrize("nx,ny,t,grid", [(64, 64, 12, (1, 1)), (512, 512, 4, (1, 1)), (128, 128, 6, (2, 2))])
def test_d256_field_parity(lib, w, precision, nx, ny, t, grid):
    """MFP at d = 256 after K iterations + the final phase vs the oracle (its D1
    emulation for the 2 x 2 grid, all ranks on this device)."""
    g = gp_boundary(nx, ny, 3)
    cfg = lib.make_config(nx, ny, grid, precision=precision, subsolver=lib.SDNET, check_every=1)
    rank = 0 if grid == (1, 1) else lib.ALL_RANKS
    m = lib.Mfp(cfg, lib.make_net(d=D, gelu=0 if precision == 0 else 1), w, rank=rank)
    u, rep = m.solve(g, t, 0.0)
    assert rep.iterations == t
    ref = oracle.mfp_run(oracle.MfpConfig(nx, ny, Py=grid[0], Px=grid[1], net=NET), g.astype(np.float64), t,
                         params=w.astype(np.float64))
    R = grid[0] * grid[1]
    L = lattice_to_global(m.lines(), nx, ny) if R == 1 else owner_view([m.lines(r) for r in range(R)], nx, ny, grid)
    tol = FP32_TOL if precision == 0 else TC_TOL
    assert rel_err(L, ref.lines, line_mask(nx, ny)) <= tol
    assert rel_err(u, ref.u) <= tol
    assert abs(rep.last_delta - ref.deltas[-1]) <= 2 * tol * np.max(np.abs(ref.u))
    m.close()


def test_d256_c3_lattice_bf16(lib, w):
    """C3 (2049^2, 16,129-16,384 subdomains per phase: ~52 pair tiles per slot)
    bf16 at d = 256, K = 2: the whole line lattice vs the oracle (the final phase
    is left out here: 1.5 TFLOP of fp64 at this width; the field tests above
    cover it)."""
    nx = ny = 2048
    g = gp_boundary(nx, ny, 4)
    cfg = lib.make_config(nx, ny, precision=lib.BF16, subsolver=lib.SDNET, check_every=2)
    m = lib.Mfp(cfg, lib.make_net(d=D, gelu=1), w)
    m.solve(g, 2, 0.0)
    ref = oracle.mfp_run(oracle.MfpConfig(nx, ny, net=NET), g.astype(np.float64), 2, params=w.astype(np.float64),
                         final=False)
    L = lattice_to_global(m.lines(), nx, ny)
    assert rel_err(L, ref.lines, line_mask(nx, ny)) <= TC_TOL
    m.close()


@pytest.mark.parametrize("d", [128, 256])
@pytest.mark.parametrize("nh", [1, 2])
@pytest.mark.parametrize("precision", [1, 3])
def test_fewer_hidden_layers(lib, d, nh, precision):
    """n_hidden = 1, 2 (mfp_sdnet_desc allows 1..3) through every tensor-core chain:
    the weight ring / resident images, the layer loop and the head after fewer
    layers, vs the oracle (FP16X is d = 128 only)."""
    import torch
    if precision == 3 and d == 256:
        pytest.skip("FP16X supports d = 128")
    w = random_weights(3, d=d, n_hidden=nh)
    cfg = lib.make_config(512, 512, precision=precision, subsolver=lib.SDNET, check_every=1)
    m = lib.Mfp(cfg, lib.make_net(d=d, n_hidden=nh, gelu=2 if precision == 3 else 1), w)
    gb = random_boundaries(2000, seed=41)
    out = m.sdnet_batch(torch.from_numpy(gb).cuda(), 0).cpu().numpy()
    q = oracle.writeset(0, 0)[1]
    net = oracle.NetShape(d=d, n_hidden=nh)
    ref = oracle.sdnet_forward(w.astype(np.float64), gb.astype(np.float64), q, net=net)
    _, S = torch_sdnet(w, gb, q, d=d, n_hidden=nh, return_scale=True)
    check_batch(out, ref, 2 if precision == 3 else precision, S)
    m.close()
