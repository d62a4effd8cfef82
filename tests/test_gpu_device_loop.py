"""The on-device convergence loop (api.cu run_loop: a CUDA graph WHILE node whose
body is a block of c iterations + delta + the stopping rule k_loop_ctl).

PAPER.md P:43-44 (Algorithm 2: iterate until the convergence threshold eps or t
iterations).  A solve with tol > 0 on a single-process context runs its whole
sequence of check blocks in ONE graph launch; these tests check it against the
host-checked fixed-iteration path: the same stop iteration as the oracle's stop
rule (tests/test_gpu_delta.py does too), and a bit-identical field to a solve
of exactly that many iterations with tol = 0 (same kernels, same order).
"""
import numpy as np
import pytest

import oracle
from mfp_inputs import gp_boundary, random_weights

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def lib():
    import torch
    assert torch.cuda.is_available()
    import paper_2308_14258_b200 as mfp
    return mfp


@pytest.mark.parametrize("subsolver,precision,grid,ce", [("exact", 0, (1, 1), 4), ("exact", 0, (2, 2), 3),
                                                         ("sdnet", 1, (1, 1), 2), ("sdnet", 0, (1, 2), 5)])
def test_device_loop_matches_fixed_iterations(lib, subsolver, precision, grid, ce):
    nx = ny = 128
    g = gp_boundary(nx, ny, 2)
    sub = lib.EXACT_LAPLACE if subsolver == "exact" else lib.SDNET
    w = None if subsolver == "exact" else random_weights(0)
    cfg = lib.make_config(nx, ny, grid, precision=precision, subsolver=sub, check_every=ce)
    rank = 0 if grid == (1, 1) else lib.ALL_RANKS
    net = lib.make_net(gelu=0 if precision == 0 else 1)
    tol = 1e-4 * float(np.max(np.abs(g)))
    m = lib.Mfp(cfg, net, w, rank=rank)
    u, rep = m.solve(g, 5000, tol)
    assert rep.converged == 1
    assert rep.iterations % ce == 0 and rep.last_delta <= tol
    # the stop rule decided on the device agrees with the oracle's (G5)
    ocfg = oracle.MfpConfig(nx, ny, Py=grid[0], Px=grid[1], subsolver=subsolver, check_every=ce)
    ref = oracle.mfp_run(ocfg, g.astype(np.float64), 5000, tol, params=None if w is None else w.astype(np.float64),
                         final=False)
    if ref.iterations != rep.iterations:
        # only a check whose oracle delta sits within rounding of tol may differ
        k = min(ref.iterations, rep.iterations)
        assert abs(ref.deltas[k - 1] - tol) <= 1e-2 * tol, (ref.iterations, rep.iterations)
    # bit-identical to the same number of iterations run with tol = 0
    m2 = lib.Mfp(cfg, net, w, rank=rank)
    u2, rep2 = m2.solve(g, rep.iterations, 0.0)
    assert rep2.iterations == rep.iterations
    assert np.array_equal(u, u2)
    m.close()
    m2.close()


def test_device_loop_budget_and_remainder(lib):
    """t not a multiple of c: the loop stops when no whole block fits, the host
    runs the remaining iterations; not converged -> MFP_NOT_CONVERGED with the
    field written, exactly t iterations."""
    nx = ny = 96
    g = gp_boundary(nx, ny, 1)
    cfg = lib.make_config(nx, ny, subsolver=lib.EXACT_LAPLACE, check_every=4)
    m = lib.Mfp(cfg, lib.make_net(), None)
    u1, rep1 = m.solve(g, 11, 1e-30)          # MFP_NOT_CONVERGED: field and report written
    assert rep1.converged == 0 and rep1.iterations == 11
    u, rep = m.solve(g, 11, 0.0)
    assert rep.iterations == 11
    assert np.array_equal(u, u1)
    m.close()
