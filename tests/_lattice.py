"""Test helpers: map exported local lattices to global (x, y) fields (layout only)."""
import numpy as np


def lattice_to_global(lat, nx, ny, fill=np.nan):
    """Global (ny+1, nx+1) array holding the lattice values of one rank."""
    info = lat.info
    U = np.full((ny + 1, nx + 1), fill, np.float64)
    for i in range(info.n_hlines):
        y = info.RY0 + 16 * i
        U[y, info.RX0: info.RX1 + 1] = lat.hl[i]
    for j in range(info.n_vlines):
        x = info.RX0 + 16 * j
        U[info.RY0: info.RY1 + 1, x] = lat.vl[j]
    return U


def crossings_consistent(lat):
    info = lat.info
    for i in range(info.n_hlines):
        for j in range(info.n_vlines):
            if lat.hl[i, 16 * j] != lat.vl[j, 16 * i]:
                return False
    return True


def owner_view(lats, nx, ny, grid):
    """Assemble the owner's value of every line point from per-rank lattices (D1)."""
    Py, Px = grid
    Lx, Ly = nx // Px, ny // Py
    U = np.full((ny + 1, nx + 1), np.nan)
    for r, lat in enumerate(lats):
        G = lattice_to_global(lat, nx, ny)
        ry, rx = divmod(r, Px)
        xs = np.arange(nx + 1)
        ys = np.arange(ny + 1)
        ox = np.minimum(xs // Lx, Px - 1) == rx
        oy = np.minimum(ys // Ly, Py - 1) == ry
        mask = oy[:, None] & ox[None, :] & ~np.isnan(G)
        U[mask] = G[mask]
    return U


def line_mask(nx, ny):
    X, Y = np.meshgrid(np.arange(nx + 1), np.arange(ny + 1))
    return (X % 16 == 0) | (Y % 16 == 0)
