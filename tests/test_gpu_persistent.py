"""The persistent exact-subsolver iteration (NEXT-2: "a fully
persistent 4-phase kernel; dataflow flags replace grid barriers";
kernels_lattice.cu k_exact_iter, opt-in with MFP_PERSIST=1 read at mfp_init).

PAPER.md P:43-44: the four phases of an iteration in class order.  One launch per
iteration; a group of 8 subdomains starts a phase as soon as the groups of other
phases that write its perimeter (RAW), read or write its centre lines (WAR, WAW)
have finished their latest earlier stage — per-group stamps instead of phase
barriers.  It performs the same FMAs per output as the per-phase kernels, so the
field must be bit-identical to them, for fixed iterations, through the CUDA-graph
blocks, the on-device convergence loop, resumed solves, and several solves on one
context (the stamps and the device iteration counter carry over).
"""
import os

import numpy as np
import pytest

import oracle
from mfp_inputs import gp_boundary

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def lib():
    import torch
    assert torch.cuda.is_available()
    import paper_2308_14258_b200 as mfp
    return mfp


def ctx(lib, nx, ny, ce, persist):
    cfg = lib.make_config(nx, ny, subsolver=lib.EXACT_LAPLACE, check_every=ce)
    old = os.environ.get("MFP_PERSIST")
    os.environ["MFP_PERSIST"] = "1" if persist else "0"
    try:
        return lib.Mfp(cfg, lib.make_net(), None)
    finally:
        if old is None:
            del os.environ["MFP_PERSIST"]
        else:
            os.environ["MFP_PERSIST"] = old


@pytest.mark.parametrize("nx,ny,t,ce", [(64, 64, 7, 1), (96, 160, 12, 4), (512, 512, 33, 16), (4096, 4096, 20, 16)])
def test_persistent_bit_identical(lib, nx, ny, t, ce):
    g = gp_boundary(nx, ny, 1)
    a, b = ctx(lib, nx, ny, ce, False), ctx(lib, nx, ny, ce, True)
    ua, ra = a.solve(g, t, 0.0)
    ub, rb = b.solve(g, t, 0.0)
    assert ra.iterations == rb.iterations == t
    assert np.array_equal(ua, ub)
    # a second solve on the same contexts (stamps and the iteration counter carry over)
    g2 = gp_boundary(nx, ny, 2)
    ua, _ = a.solve(g2, t + 3, 0.0)
    ub, _ = b.solve(g2, t + 3, 0.0)
    assert np.array_equal(ua, ub)
    # resumed (g = None): continue from the current lattice
    ua, _ = a.solve(None, 5, 0.0)
    ub, _ = b.solve(None, 5, 0.0)
    assert np.array_equal(ua, ub)
    a.close()
    b.close()


def test_persistent_converges_to_oracle_stop(lib):
    nx = ny = 256
    g = gp_boundary(nx, ny, 3)
    tol = 1e-6 * float(np.max(np.abs(g)))
    b = ctx(lib, nx, ny, 8, True)
    u, rep = b.solve(g, 20000, tol)
    assert rep.converged == 1
    a = ctx(lib, nx, ny, 8, False)
    u0, rep0 = a.solve(g, 20000, tol)
    assert rep.iterations == rep0.iterations and np.array_equal(u, u0)
    ref = oracle.mfp_run(oracle.MfpConfig(nx, ny, subsolver="exact", check_every=8), g.astype(np.float64), 20000, tol,
                         final=False)
    assert abs(ref.iterations - rep.iterations) <= 8
    a.close()
    b.close()
