"""Input-generator pins and SDNet-driven oracle MFP invariants."""
import numpy as np
import pytest

import oracle
from mfp_inputs import gp_boundary, gp_hyperparameters, random_weights, sobol_2d
from tests.conftest import load_golden

M = 32


def test_sobol_spec_example():
    """dim 1, n = 4 -> 0, .5, .75, .25 (unscrambled Sobol)."""
    from scipy.stats import qmc
    want = load_golden("sobol_dim1.txt")[:, 0]
    got = qmc.Sobol(d=1, scramble=False).random(4)[:, 0]
    assert np.array_equal(got, want)
    assert sobol_2d(0) == (0.0, 0.0)


def test_gp_boundary_deterministic_and_in_box():
    a, b = gp_boundary(128, 64, 3), gp_boundary(128, 64, 3)
    assert a.dtype == np.float32 and a.size == 2 * (128 + 64)
    assert np.array_equal(a, b)
    var, ls = gp_hyperparameters(3)
    assert 0.1 <= var <= 1.0 and 0.1 <= ls <= 0.5
    big = gp_boundary(4096, 4096, 0)
    assert big.size == 16384 and np.all(np.isfinite(big))


def test_sdnet_mfp_batched_equals_sequential():
    """batching the disjoint subdomains of a class does not change results."""
    nx, ny = 3 * M, 2 * M
    g = gp_boundary(nx, ny, 1).astype(np.float64)
    w = random_weights(0).astype(np.float64)
    a = oracle.mfp_run(oracle.MfpConfig(nx, ny), g, t=3, params=w)
    b = oracle.mfp_run(oracle.MfpConfig(nx, ny, sequential=True), g, t=3, params=w)
    assert np.array_equal(a.lines, b.lines) and np.array_equal(a.u, b.u)


def test_sdnet_mfp_boundary_immutable_and_lines_only():
    nx, ny = 2 * M, 2 * M
    g = gp_boundary(nx, ny, 2).astype(np.float64)
    w = random_weights(1).astype(np.float64)
    r = oracle.mfp_run(oracle.MfpConfig(nx, ny, Px=2), g, t=4, params=w)
    from mfp_inputs import boundary_points
    bp = boundary_points(nx, ny)
    assert np.array_equal(r.lines[bp[:, 1], bp[:, 0]], g)
    assert np.array_equal(r.u[bp[:, 1], bp[:, 0]], g)
    X, Y = np.meshgrid(np.arange(nx + 1), np.arange(ny + 1))
    off = (X % 16 != 0) & (Y % 16 != 0)
    assert np.all(r.lines[off] == 0.0)                              # only line points touched
    assert np.all(np.isfinite(r.u))


def test_sdnet_mfp_final_phase_is_interior_prediction():
    """the final field's interior points are SDNet predictions on the last
    boundaries, its atomic-subdomain lines the lattice values."""
    nx, ny = 2 * M, 2 * M
    g = gp_boundary(nx, ny, 0).astype(np.float64)
    w = random_weights(2).astype(np.float64)
    cfg = oracle.MfpConfig(nx, ny)
    r = oracle.mfp_run(cfg, g, t=2, params=w)
    anc = oracle.anchors(nx, ny, 0)
    pred = oracle.predict_from_field(cfg, r.lines, anc, query_set=1, params=w)
    q = np.rint(oracle.interior_queries() * M).astype(int)
    for k, (ax, ay) in enumerate(anc):
        assert np.array_equal(r.u[ay + q[:, 1], ax + q[:, 0]], pred[k])
    assert np.array_equal(r.u[:, ::M], r.lines[:, ::M]) and np.array_equal(r.u[::M, :], r.lines[::M, :])
