"""NEXT-2 peer-memory halo transport (mfp_p2p_open; kernels_p2p.cu) on one GPU.

With MFP_ALL_RANKS every rank's region lives on the same device, so the pack /
publish / pull / consumed protocol, the parity double buffer, the per-peer
segment table and the device-side epoch (graph replay) run exactly as across
GPUs, only without NVLink.  The transport moves the same floats as the copy
transport, so the two solves must be bit-identical; both are also checked
against the oracle's D1 emulation (communicate_new_boundaries).
"""
import numpy as np
import pytest

import oracle
from mfp_inputs import gp_boundary, random_weights
from tests._lattice import line_mask, owner_view

pytestmark = pytest.mark.gpu

M = 32
FP32_TOL = 1e-5


@pytest.fixture(scope="module")
def lib():
    import torch
    assert torch.cuda.is_available()
    import paper_2308_14258_b200 as mfp
    return mfp


def run(lib, nx, ny, grid, t, p2p, subsolver="exact", precision=0, ce=1, s_ex=1, seed=3):
    sub = lib.EXACT_LAPLACE if subsolver == "exact" else lib.SDNET
    cfg = lib.make_config(nx, ny, grid, precision=precision, subsolver=sub, check_every=ce)
    w = None if subsolver == "exact" else random_weights(seed)
    m = lib.Mfp(cfg, lib.make_net(), w, rank=lib.ALL_RANKS)
    if s_ex != 1:
        lib.mfp_set_exchange_every(m.ctx, s_ex)
    if p2p:
        lib.mfp_p2p_open(m.ctx)
    g = gp_boundary(nx, ny, seed)
    u, rep = m.solve(g, t, 0.0)
    R = grid[0] * grid[1]
    lines = owner_view([m.lines(r) for r in range(R)], nx, ny, grid)
    return u, lines, rep, g, w


@pytest.mark.parametrize("grid,kx,ky,t,ce,s_ex", [((1, 2), 4, 4, 10, 1, 1), ((2, 2), 4, 4, 9, 4, 1),
                                                  ((2, 4), 8, 4, 8, 2, 2), ((3, 3), 6, 6, 7, 1, 1),
                                                  ((2, 1), 2, 4, 12, 6, 3)])
def test_p2p_bit_identical_to_copy_transport(lib, grid, kx, ky, t, ce, s_ex):
    nx, ny = kx * M, ky * M
    u0, L0, _, g, _ = run(lib, nx, ny, grid, t, False, ce=ce, s_ex=s_ex)
    u1, L1, rep, _, _ = run(lib, nx, ny, grid, t, True, ce=ce, s_ex=s_ex)
    assert rep.iterations == t
    assert np.array_equal(u0, u1)
    assert np.array_equal(L0, L1, equal_nan=True)   # NaN = not a line point
    ref = oracle.mfp_run(oracle.MfpConfig(nx, ny, Py=grid[0], Px=grid[1], subsolver="exact", check_every=ce,
                                          exchange_every=s_ex), g.astype(np.float64), t)
    lm = line_mask(nx, ny)
    a, b = np.asarray(L1, np.float64)[lm], ref.lines[lm]
    assert np.max(np.abs(a - b)) / np.max(np.abs(b)) <= FP32_TOL


@pytest.mark.parametrize("precision", [0, 1])
def test_p2p_sdnet_2x4(lib, precision):
    """SDNet subsolver (fp32 SIMT and bf16 tcgen05 chain) on the 2x4 grid the
    8-GPU bench uses, with graph-replayed blocks: identical to the copy transport."""
    nx, ny = 16 * M, 8 * M
    u0, L0, _, _, _ = run(lib, nx, ny, (2, 4), 9, False, "sdnet", precision, ce=3)
    u1, L1, _, _, _ = run(lib, nx, ny, (2, 4), 9, True, "sdnet", precision, ce=3)
    assert np.array_equal(u0, u1)
    assert np.array_equal(L0, L1, equal_nan=True)   # NaN = not a line point


def test_p2p_to_convergence(lib):
    """Exact subsolver to a tolerance through the peer transport: same iteration
    count and field as the copy transport (epochs advance through many graphs)."""
    nx = ny = 8 * M
    out = []
    for p2p in (False, True):
        cfg = lib.make_config(nx, ny, (2, 2), subsolver=lib.EXACT_LAPLACE, check_every=8)
        m = lib.Mfp(cfg, lib.make_net(), None, rank=lib.ALL_RANKS)
        if p2p:
            lib.mfp_p2p_open(m.ctx)
        u, rep = m.solve(gp_boundary(nx, ny, 4), 20000, 1e-6)
        out.append((u, rep.iterations, rep.converged))
    assert out[0][1] == out[1][1] and out[1][2]
    assert np.array_equal(out[0][0], out[1][0])


def test_p2p_errors(lib):
    nx = ny = 4 * M
    cfg = lib.make_config(nx, ny, (2, 2), subsolver=lib.EXACT_LAPLACE)
    m = lib.Mfp(cfg, lib.make_net(), None, rank=lib.ALL_RANKS)
    with pytest.raises(lib.MfpError) as e:          # handles must be NULL for ALL_RANKS
        lib.mfp_p2p_open(m.ctx, [b"\0" * 64] * 4)
    assert e.value.status == 1
    with pytest.raises(lib.MfpError) as e:          # export is for one-process-per-GPU contexts
        lib.mfp_p2p_export(m.ctx)
    assert e.value.status == 1
    with pytest.raises(lib.MfpError) as e:          # a short handle list (R = 4) is rejected in C
        from paper_2308_14258_b200 import mfp as binding
        binding._check(binding._lib.mfp_p2p_open(m.ctx, None, 3), m.ctx)
    assert e.value.status == 1
    lib.mfp_p2p_open(m.ctx)
    with pytest.raises(lib.MfpError) as e:          # once per context
        lib.mfp_p2p_open(m.ctx)
    assert e.value.status == 1
    m1 = lib.Mfp(lib.make_config(nx, ny, (1, 1), subsolver=lib.EXACT_LAPLACE), lib.make_net(), None, rank=0)
    with pytest.raises(lib.MfpError) as e:          # a 1x1 grid has no halo
        lib.mfp_p2p_open(m1.ctx)
    assert e.value.status == 1
