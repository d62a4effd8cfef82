"""Pins for the oracle's exact discrete-Laplace subsolver and the exact-solver MFP.

With the SDNet replaced by the exact subdomain solve, the MF predictor is the
alternating (multiplicative) Schwarz method of §2.3 on the line
lattice, whose fixed point is the global 5-point discrete harmonic function
(P:512-519).  Pinned against DST-I and sparse-LU global solves (tests/_refsolve.py),
discrete-harmonic closed forms, and SPEC's examples.
"""
import numpy as np
import pytest

import oracle
from mfp_inputs import boundary_points, closed_form_boundary, gp_boundary
from tests._refsolve import dst_laplace, sparse_laplace

M = 32


@pytest.fixture(scope="module")
def Hc():
    return oracle.harmonic_matrix(0)


@pytest.fixture(scope="module")
def Hf():
    return oracle.harmonic_matrix(1)


def test_harmonic_matrix_invariants(Hc, Hf):
    for H in (Hc, Hf):
        assert H.min() >= -1e-15                                   # maximum principle
        assert np.max(np.abs(H.sum(1) - 1.0)) < 1e-12              # constants preserved
        corners = [0, M, 2 * M, 3 * M]                             # perimeter corner indices (G1)
        assert np.all(H[:, corners] == 0.0)                        # 5-point stencil never reads corners


def test_harmonic_matrix_vs_sparse_patch_solve(Hc, Hf):
    rng = np.random.default_rng(0)
    g = rng.standard_normal(4 * M)
    per = oracle.perimeter(0, 0)
    bval = {tuple(p): g[k] for k, p in enumerate(per)}
    U = sparse_laplace(M, M, lambda x, y: bval[(x, y)])
    wr, _ = oracle.writeset(0, 0)
    assert np.max(np.abs(Hc @ g - U[wr[:, 1], wr[:, 0]])) < 1e-12
    q = np.rint(oracle.interior_queries() * M).astype(int)
    assert np.max(np.abs(Hf @ g - U[q[:, 1], q[:, 0]])) < 1e-12


def test_harmonic_matrix_closed_form(Hc):
    # x^2 - y^2 is exactly discrete-harmonic for the 5-point stencil
    per = oracle.perimeter(0, 0).astype(float)
    g = per[:, 0] ** 2 - per[:, 1] ** 2
    wr, _ = oracle.writeset(0, 0)
    assert np.max(np.abs(Hc @ g - (wr[:, 0] ** 2 - wr[:, 1] ** 2))) < 1e-9


def test_single_subdomain_one_iteration_exact():
    """a domain that is one atomic subdomain -> after one iteration the
    centre lines equal the global discrete solution."""
    g = gp_boundary(M, M, 3).astype(np.float64)
    res = oracle.mfp_run(oracle.MfpConfig(M, M, subsolver="exact"), g, t=1)
    ref = dst_laplace(M, M, g)
    wr, _ = oracle.writeset(0, 0)
    assert np.max(np.abs(res.lines[wr[:, 1], wr[:, 0]] - ref[wr[:, 1], wr[:, 0]])) < 1e-12
    assert np.max(np.abs(res.u - ref)) < 1e-12


def test_dst_matches_sparse_lu():
    g = gp_boundary(64, 64, 1).astype(np.float64)
    from mfp_inputs import boundary_points
    bp = boundary_points(64, 64)
    bval = {(int(x), int(y)): g[k] for k, (x, y) in enumerate(bp)}
    assert np.max(np.abs(dst_laplace(64, 64, g) - sparse_laplace(64, 64, lambda x, y: bval[(x, y)]))) < 1e-12


@pytest.mark.parametrize("k", [0, 2])
def test_c1_converges_to_global_discrete_solution(k):
    nx = ny = 2 * M                                                # C1: 65^2, 9 predictions/iter
    g = gp_boundary(nx, ny, k).astype(np.float64)
    res = oracle.mfp_run(oracle.MfpConfig(nx, ny, subsolver="exact"), g, t=400, tol=1e-14)
    assert res.iterations < 400
    ref = dst_laplace(nx, ny, g)
    assert np.max(np.abs(res.u - ref)) < 1e-11
    # ∂Ω immutable, bit-exact
    from mfp_inputs import boundary_points
    bp = boundary_points(nx, ny)
    assert np.array_equal(res.u[bp[:, 1], bp[:, 0]], g)
    # maximum principle
    assert res.u.min() >= g.min() - 1e-12 and res.u.max() <= g.max() + 1e-12


@pytest.mark.parametrize("name,f", [("x2-y2", lambda x, y: x * x - y * y), ("xy", lambda x, y: x * y)])
def test_closed_forms_discrete_harmonic(name, f):
    """north_star: harmonic closed forms reproduced to 1e-8 (exactly
    discrete-harmonic, so the converged MFP must equal them)."""
    nx = ny = 2 * M
    h = 1.0 / 64.0
    g = closed_form_boundary(nx, ny, f, h)
    res = oracle.mfp_run(oracle.MfpConfig(nx, ny, subsolver="exact"), g, t=400, tol=1e-14)
    X, Y = np.meshgrid(np.arange(nx + 1) * h, np.arange(ny + 1) * h)
    assert np.max(np.abs(res.u - f(X, Y))) < 1e-8


def test_exp_sin_vs_discrete_solution():
    """e^x sin y is harmonic but not discrete-harmonic: pin 1e-8 against the
    discrete solve; against the closed form the floor is O(h^2)."""
    nx = ny = 2 * M
    h = 1.0 / 64.0
    f = lambda x, y: np.exp(x) * np.sin(y)
    g = closed_form_boundary(nx, ny, f, h)
    res = oracle.mfp_run(oracle.MfpConfig(nx, ny, subsolver="exact"), g, t=400, tol=1e-14)
    assert np.max(np.abs(res.u - dst_laplace(nx, ny, g))) < 1e-8
    X, Y = np.meshgrid(np.arange(nx + 1) * h, np.arange(ny + 1) * h)
    err = np.max(np.abs(res.u - f(X, Y)))
    assert 1e-8 < err < 1e-5


def sine_discrete_solution(nx, ny, h):
    """Closed-form solution of the 5-point Dirichlet problem with g = sin(2 pi x)
     when nx h is an integer: separation of variables on the grid,
    u_ij = sin(2 pi i h) v_j, v_{j+1} + v_{j-1} = (4 - 2 cos 2 pi h) v_j, v_0 = v_ny = 1
    => v_j = (sinh(l (ny - j)) + sinh(l j)) / sinh(l ny), cosh l = 2 - cos(2 pi h)."""
    lam = np.arccosh(2.0 - np.cos(2.0 * np.pi * h))
    j = np.arange(ny + 1)
    v = (np.sinh(lam * (ny - j)) + np.sinh(lam * j)) / np.sinh(lam * ny)
    return np.sin(2.0 * np.pi * np.arange(nx + 1) * h)[None, :] * v[:, None]


def test_sine_boundary_discrete_closed_form():
    """P:158's evaluation boundary sin(2 pi x): the converged exact-subsolver MFP
    equals the grid's separable closed form to 1e-8 (and that closed form is the
    continuous solution sin(2 pi x)(sinh 2pi(H-y) + sinh 2pi y)/sinh 2pi H to O(h^2))."""
    from mfp_inputs import sine_boundary
    nx, ny = 2 * M, 4 * M            # 1 x 2 units (the paper's smallest domain)
    h = 1.0 / 64.0
    g = sine_boundary(nx, ny, h)
    ref = sine_discrete_solution(nx, ny, h)
    bp = boundary_points(nx, ny)
    assert np.max(np.abs(ref[bp[:, 1], bp[:, 0]] - g)) < 1e-14   # the closed form meets g
    assert np.max(np.abs(ref - dst_laplace(nx, ny, g))) < 1e-12    # and is the discrete solution
    res = oracle.mfp_run(oracle.MfpConfig(nx, ny, subsolver="exact"), g, t=2000, tol=1e-14)
    assert np.max(np.abs(res.u - ref)) < 1e-8
    X, Y = np.meshgrid(np.arange(nx + 1) * h, np.arange(ny + 1) * h)
    H = ny * h
    cont = np.sin(2 * np.pi * X) * (np.sinh(2 * np.pi * (H - Y)) + np.sinh(2 * np.pi * Y)) / np.sinh(2 * np.pi * H)
    err = np.max(np.abs(ref - cont))
    assert 1e-6 < err < 2e-3                                     # O((2 pi h)^2) discretisation gap


def test_linearity():
    """the exact-solver MFP is linear in g at any fixed iteration count."""
    nx, ny = 3 * M, 2 * M
    g1 = gp_boundary(nx, ny, 0).astype(np.float64)
    g2 = gp_boundary(nx, ny, 1).astype(np.float64)
    cfg = oracle.MfpConfig(nx, ny, subsolver="exact")
    r1 = oracle.mfp_run(cfg, g1, t=7)
    r2 = oracle.mfp_run(cfg, g2, t=7)
    r3 = oracle.mfp_run(cfg, 2.0 * g1 - 0.5 * g2, t=7)
    assert np.max(np.abs(r3.u - (2.0 * r1.u - 0.5 * r2.u))) < 1e-12


def test_batched_equals_sequential_bit_exact():
    """P:23 / S:600: class members are disjoint, so batched == one-at-a-time."""
    nx, ny = 4 * M, 3 * M
    g = gp_boundary(nx, ny, 4).astype(np.float64)
    a = oracle.mfp_run(oracle.MfpConfig(nx, ny, subsolver="exact"), g, t=6)
    b = oracle.mfp_run(oracle.MfpConfig(nx, ny, subsolver="exact", sequential=True), g, t=6)
    assert np.array_equal(a.lines, b.lines) and np.array_equal(a.u, b.u)


@pytest.mark.parametrize("py,px", [(1, 2), (2, 1), (2, 2)])
def test_distributed_emulation_converges_to_same_solution(py, px):
    """P:48 (Lions): relaxed synchronisation changes the trajectory, not the limit."""
    nx = ny = 4 * M
    g = gp_boundary(nx, ny, 2).astype(np.float64)
    ref = dst_laplace(nx, ny, g)
    r1 = oracle.mfp_run(oracle.MfpConfig(nx, ny, subsolver="exact"), g, t=3000, tol=1e-13)
    rp = oracle.mfp_run(oracle.MfpConfig(nx, ny, Py=py, Px=px, subsolver="exact"), g, t=3000, tol=1e-13)
    assert r1.iterations < 3000 and rp.iterations < 3000
    assert np.max(np.abs(r1.u - ref)) < 1e-10
    assert np.max(np.abs(rp.u - ref)) < 1e-10
    assert rp.iterations >= r1.iterations                          # staleness never helps here


@pytest.mark.parametrize("s_ex", [2, 4])
def test_communication_avoiding_same_limit(s_ex):
    """The communication-avoiding variant (halos refreshed every s iterations)
    is still a relaxed Schwarz iteration: same limit (the global discrete solution),
    more iterations; s = 1 reproduces Algorithm 2 bit for bit."""
    nx = ny = 4 * M
    g = gp_boundary(nx, ny, 3).astype(np.float64)
    ref = dst_laplace(nx, ny, g)
    base = oracle.MfpConfig(nx, ny, Py=2, Px=2, subsolver="exact", check_every=4)
    r1 = oracle.mfp_run(base, g, t=4000, tol=1e-13)
    rs = oracle.mfp_run(oracle.MfpConfig(nx, ny, Py=2, Px=2, subsolver="exact", check_every=4,
                                         exchange_every=s_ex), g, t=4000, tol=1e-13)
    assert rs.iterations < 4000
    assert np.max(np.abs(rs.u - ref)) < 1e-10
    assert rs.iterations >= r1.iterations
    r1b = oracle.mfp_run(oracle.MfpConfig(nx, ny, Py=2, Px=2, subsolver="exact", check_every=4,
                                          exchange_every=1), g, t=30)
    r1c = oracle.mfp_run(base, g, t=30)
    assert np.array_equal(r1b.u, r1c.u)


def test_distributed_p1_is_plain():
    nx, ny = 2 * M, 4 * M
    g = gp_boundary(nx, ny, 0).astype(np.float64)
    a = oracle.mfp_run(oracle.MfpConfig(nx, ny, subsolver="exact"), g, t=5)
    b = oracle.mfp_run(oracle.MfpConfig(nx, ny, Py=1, Px=1, subsolver="exact", check_every=3), g, t=5)
    assert np.array_equal(a.u, b.u)
