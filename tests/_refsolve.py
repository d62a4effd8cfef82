"""Independent global references for the oracle pins (test code, not the oracle).

* ``dst_laplace``: the 5-point discrete Dirichlet Laplace solution on an
  (nx+1)x(ny+1) grid by the DST-I eigen-decomposition (scipy.fft.dstn).
* ``sparse_laplace``: the same system assembled with identity rows on the
  boundary and solved by a sparse direct solver (scipy.sparse.linalg.spsolve).
Neither shares code with ``oracle/``; they are two different algorithms for the
plain definition "discrete harmonic with the given boundary" (§2.1,
P:512-519, 5-point stencil SPEC S:120).
"""
import numpy as np
import scipy.fft
import scipy.sparse
import scipy.sparse.linalg

from mfp_inputs import boundary_points


def boundary_field(nx, ny, g):
    U = np.zeros((ny + 1, nx + 1))
    p = boundary_points(nx, ny)
    U[p[:, 1], p[:, 0]] = g
    return U


def dst_laplace(nx, ny, g):
    U = boundary_field(nx, ny, np.asarray(g, np.float64))
    b = np.zeros((ny - 1, nx - 1))
    b[:, 0] += U[1:ny, 0]
    b[:, -1] += U[1:ny, nx]
    b[0, :] += U[0, 1:nx]
    b[-1, :] += U[ny, 1:nx]
    bh = scipy.fft.dstn(b, type=1, norm="ortho")
    i = np.arange(1, nx)
    j = np.arange(1, ny)
    lam = 4.0 - 2.0 * np.cos(np.pi * i / nx)[None, :] - 2.0 * np.cos(np.pi * j / ny)[:, None]
    U[1:ny, 1:nx] = scipy.fft.idstn(bh / lam, type=1, norm="ortho")
    return U


def sparse_laplace(nx, ny, boundary_values_fn):
    """Solve on the full grid; boundary_values_fn(x, y) -> value for boundary points."""
    W, H = nx + 1, ny + 1
    n = W * H
    rows, cols, vals = [], [], []
    rhs = np.zeros(n)
    for y in range(H):
        for x in range(W):
            r = y * W + x
            if x in (0, nx) or y in (0, ny):
                rows.append(r); cols.append(r); vals.append(1.0)
                rhs[r] = boundary_values_fn(x, y)
            else:
                rows.append(r); cols.append(r); vals.append(4.0)
                for dx, dy in ((1, 0), (-1, 0), (0, 1), (0, -1)):
                    rows.append(r); cols.append((y + dy) * W + x + dx); vals.append(-1.0)
    A = scipy.sparse.csr_matrix((vals, (rows, cols)), shape=(n, n))
    return scipy.sparse.linalg.spsolve(A.tocsc(), rhs).reshape(H, W)
