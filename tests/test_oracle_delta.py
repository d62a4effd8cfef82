"""Pins for the oracle's convergence quantity delta_k (reading G5, a8).

PAPER.md P:43 (§4.2, Algorithm 2: input "convergence threshold epsilon") and
P:44 (the second phase starts "upon reaching the convergence threshold") fix a
stopping rule but not its norm; reading G5 takes
delta_k = max over OWNED interior line points of |U_k - U_{k-1}|, tested every
c iterations.  These tests pin the oracle's delta_log (orc_mfp_run) against
things other than the oracle's own delta loop:
  * the definition applied in numpy to the oracle's owner views after t - 1
    and t iterations (separate runs; every line point, interior only) — bit
    exact, on 1x1, 2x2 and 2x4 emulated grids, exact and SDNet subsolvers;
  * a closed form: a domain that is one atomic subdomain has
    delta_1 = max |discrete solution| on its centre lines (sparse LU) and
    delta_2 = 0 exactly (same boundary, same prediction);
  * linearity of the exact-subsolver iteration: delta(2 g) = 2 delta(g) bit for
    bit (scaling by a power of two commutes with every rounding);
  * the stopping rule: with tol > 0 the run stops at the first multiple of c
    whose delta is <= tol, read off a tol = 0 run.
"""
import numpy as np
import pytest

import oracle
from mfp_inputs import gp_boundary, random_weights
from tests._refsolve import sparse_laplace

M = 32


def interior_line_mask(nx, ny):
    X, Y = np.meshgrid(np.arange(nx + 1), np.arange(ny + 1))
    line = (X % (M // 2) == 0) | (Y % (M // 2) == 0)
    inner = (X > 0) & (X < nx) & (Y > 0) & (Y < ny)
    return line & inner


def definition_delta(cfg, g, t, params):
    """delta_t from the owner views after t - 1 and t iterations (reading G5)."""
    cur = oracle.mfp_run(cfg, g, t, params=params, final=False).lines
    if t == 1:
        prev = np.zeros_like(cur)          # interior initial guess 0
    else:
        prev = oracle.mfp_run(cfg, g, t - 1, params=params, final=False).lines
    mk = interior_line_mask(cfg.nx, cfg.ny)
    return float(np.max(np.abs(cur[mk] - prev[mk])))


@pytest.mark.parametrize("grid,kx,ky", [((1, 1), 3, 2), ((2, 2), 4, 4), ((2, 4), 8, 4)])
@pytest.mark.parametrize("subsolver", ["exact", "sdnet"])
@pytest.mark.parametrize("t", [1, 2, 5])
def test_delta_equals_definition(grid, kx, ky, subsolver, t):
    nx, ny = kx * M, ky * M
    g = gp_boundary(nx, ny, 4).astype(np.float64)
    params = None if subsolver == "exact" else random_weights(0).astype(np.float64)
    cfg = oracle.MfpConfig(nx, ny, Py=grid[0], Px=grid[1], subsolver=subsolver)
    log = oracle.mfp_run(cfg, g, t, params=params, final=False).deltas
    assert log.shape == (t,)
    assert log[t - 1] == definition_delta(cfg, g, t, params)     # bit-exact
    assert np.all(log >= 0.0)


def test_delta_single_subdomain_closed_form():
    """one atomic subdomain; the first iteration writes the discrete
    solution onto the centre lines, the second reproduces it bit for bit."""
    g = gp_boundary(M, M, 3).astype(np.float64)
    cfg = oracle.MfpConfig(M, M, subsolver="exact")
    r = oracle.mfp_run(cfg, g, 3, final=False)
    from mfp_inputs import boundary_points
    bp = boundary_points(M, M)
    bval = {(int(x), int(y)): g[k] for k, (x, y) in enumerate(bp)}
    U = sparse_laplace(M, M, lambda x, y: bval[(x, y)])
    wr, _ = oracle.writeset(0, 0)
    assert abs(r.deltas[0] - np.max(np.abs(U[wr[:, 1], wr[:, 0]]))) < 1e-12
    assert r.deltas[1] == 0.0 and r.deltas[2] == 0.0


@pytest.mark.parametrize("grid", [(1, 1), (2, 2)])
def test_delta_linear_in_boundary(grid):
    nx = ny = 4 * M
    g = gp_boundary(nx, ny, 1).astype(np.float64)
    cfg = oracle.MfpConfig(nx, ny, Py=grid[0], Px=grid[1], subsolver="exact")
    a = oracle.mfp_run(cfg, g, 9, final=False).deltas
    b = oracle.mfp_run(cfg, 2.0 * g, 9, final=False).deltas
    assert np.array_equal(b, 2.0 * a)


@pytest.mark.parametrize("grid,c", [((1, 1), 1), ((1, 1), 4), ((2, 2), 3)])
def test_stop_rule_first_check_below_tol(grid, c):
    nx = ny = 4 * M
    g = gp_boundary(nx, ny, 2).astype(np.float64)
    cfg = oracle.MfpConfig(nx, ny, Py=grid[0], Px=grid[1], subsolver="exact", check_every=c)
    full = oracle.mfp_run(cfg, g, 120, final=False).deltas
    tol = float(full[40])                      # a value the sequence passes
    want = next(k for k in range(c, 121, c) if full[k - 1] <= tol)
    r = oracle.mfp_run(cfg, g, 120, tol=tol, final=False)
    assert r.iterations == want
    assert np.array_equal(r.deltas, full[:want])
