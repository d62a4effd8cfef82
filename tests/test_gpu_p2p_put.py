"""NEXT-2 put transport (mfp_p2p_set_mode(MFP_P2P_PUT)): the SDNet chain's
epilogue stores every owned cell a stencil peer holds as a halo cell straight
into that peer's put buffer, and the iteration's exchange is a publish + a local
unpack (kernels_p2p.cu k_put_publish / k_put_unpack).

PAPER.md P:43 (communicate_new_boundaries), P:48 (once per iteration)
(direct GPU-GPU transfers).  With MFP_ALL_RANKS every rank's region is on this
device, so the protocol (parity buffers, put-done / consumed epochs, graph
replay, communication-avoiding s > 1, convergence loops) runs as across GPUs.
The puts move the same floats the pack would (the last write of the iteration
wins), so every solve must be bit-identical to the copy transport.
"""
import numpy as np
import pytest

from mfp_inputs import gp_boundary, random_weights
from tests._lattice import owner_view

pytestmark = pytest.mark.gpu

M = 32


@pytest.fixture(scope="module")
def lib():
    import torch
    assert torch.cuda.is_available()
    import paper_2308_14258_b200 as mfp
    return mfp


def run(lib, nx, ny, grid, t, mode, precision=1, ce=1, s_ex=1, tol=0.0, d=128, seed=5):
    cfg = lib.make_config(nx, ny, grid, precision=precision, subsolver=lib.SDNET, check_every=ce)
    w = random_weights(seed, d=d)
    m = lib.Mfp(cfg, lib.make_net(d=d, gelu=0 if precision == 0 else 1), w, rank=lib.ALL_RANKS)
    if s_ex != 1:
        lib.mfp_set_exchange_every(m.ctx, s_ex)
    if mode is not None:
        lib.mfp_p2p_open(m.ctx)
        lib.mfp_p2p_set_mode(m.ctx, mode)
    g = gp_boundary(nx, ny, seed)
    u, rep = m.solve(g, t, tol)
    R = grid[0] * grid[1]
    lines = owner_view([m.lines(r) for r in range(R)], nx, ny, grid)
    m.close()
    return u, lines, rep


@pytest.mark.parametrize("grid,kx,ky,t,ce,s_ex,precision", [
    ((1, 2), 4, 4, 8, 1, 1, 1), ((2, 2), 4, 4, 9, 3, 1, 0), ((2, 4), 16, 8, 6, 2, 1, 1),
    ((3, 3), 6, 6, 7, 1, 1, 2), ((2, 1), 2, 4, 12, 6, 3, 1), ((2, 2), 6, 6, 8, 4, 2, 3)])
def test_put_bit_identical_to_copy_transport(lib, grid, kx, ky, t, ce, s_ex, precision):
    nx, ny = kx * M, ky * M
    u0, L0, _ = run(lib, nx, ny, grid, t, None, precision, ce, s_ex)
    u1, L1, rep = run(lib, nx, ny, grid, t, lib.P2P_PUT, precision, ce, s_ex)
    assert rep.iterations == t
    assert np.array_equal(u0, u1)
    assert np.array_equal(L0, L1, equal_nan=True)


def test_put_d256_and_convergence(lib):
    """The wide chain's epilogue puts too; and a tolerance solve (host-checked
    blocks under ALL_RANKS use the device loop) stops at the same iteration."""
    nx = ny = 8 * M
    u0, L0, _ = run(lib, nx, ny, (2, 2), 5, None, d=256)
    u1, L1, _ = run(lib, nx, ny, (2, 2), 5, lib.P2P_PUT, d=256)
    assert np.array_equal(u0, u1) and np.array_equal(L0, L1, equal_nan=True)
    a = run(lib, nx, ny, (2, 2), 400, None, precision=0, ce=4, tol=1e-4)
    b = run(lib, nx, ny, (2, 2), 400, lib.P2P_PUT, precision=0, ce=4, tol=1e-4)
    assert a[2].iterations == b[2].iterations
    assert np.array_equal(a[0], b[0])


def test_put_mode_switching_and_errors(lib):
    nx = ny = 4 * M
    cfg = lib.make_config(nx, ny, (2, 2), precision=1, subsolver=lib.SDNET, check_every=2)
    m = lib.Mfp(cfg, lib.make_net(gelu=1), random_weights(0), rank=lib.ALL_RANKS)
    with pytest.raises(lib.MfpError) as e:          # p2p must be open first
        lib.mfp_p2p_set_mode(m.ctx, lib.P2P_PUT)
    assert e.value.status == 1
    lib.mfp_p2p_open(m.ctx)
    with pytest.raises(lib.MfpError) as e:
        lib.mfp_p2p_set_mode(m.ctx, 7)
    assert e.value.status == 1
    g = gp_boundary(nx, ny, 2)
    lib.mfp_p2p_set_mode(m.ctx, lib.P2P_PUT)
    u_put, _ = m.solve(g, 6, 0.0)
    lib.mfp_p2p_set_mode(m.ctx, lib.P2P_PULL)
    u_pull, _ = m.solve(g, 6, 0.0)
    assert np.array_equal(u_put, u_pull)
    m.close()
    x = lib.Mfp(lib.make_config(nx, ny, (2, 2), subsolver=lib.EXACT_LAPLACE), lib.make_net(), None,
                rank=lib.ALL_RANKS)
    lib.mfp_p2p_open(x.ctx)
    with pytest.raises(lib.MfpError) as e:          # puts come from the SDNet epilogue
        lib.mfp_p2p_set_mode(x.ctx, lib.P2P_PUT)
    assert e.value.status == 1
    x.close()
