"""mfp_inputs — seeded synthetic inputs shared by the oracle tests, the GPU tests and bench.py.

This module holds NONE of the method's arithmetic (no geometry of subdomains, no
SDNet, no Schwarz step).  It only draws inputs with the shapes and value
distributions of the paper's workloads (DESIGN.md §4 "input recipe"):

* GP boundaries (§5.1): a Sobol point (unscrambled, dim 2) sets the
  hyperparameters of a squared-exponential 1-D Gaussian process
  (variance in [0.1, 1], lengthscale in [0.1, 0.5] of the normalised perimeter,
  SPEC S:224 box); one curve is drawn along the whole global perimeter with
  numpy's PCG64 seeded 2308 + k.  Long perimeters are sampled at <= 1024 knots
  by Cholesky (jitter 1e-8 * variance, x10 escalation) and interpolated
  with a cubic spline.
* Closed-form boundaries: f(x, y) evaluated on the global perimeter at spacing
  h (default 1/64, the paper's 64 points per spatial unit).
* SDNet weights: U(+-1/sqrt(fan_in)) from PCG64(seed), fp64 drawn, stored fp32,
  in SPEC MFCK declaration order.
* Batches of boundary vectors: N(0, 1) fp32 (the C3 sweep).

The global boundary vector g has 2(nx+ny) entries walked counter-clockwise from
(0, 0) (reading G6): bottom x = 0..nx-1 (y = 0), right y = 0..ny-1 (x = nx),
top x = nx..1 (y = ny), left y = ny..1 (x = 0).
"""
from __future__ import annotations

import numpy as np

GP_VAR_RANGE = (0.1, 1.0)
GP_LEN_RANGE = (0.1, 0.5)
GP_SEED_BASE = 2308
GP_MAX_KNOTS = 1024


def boundary_points(nx: int, ny: int) -> np.ndarray:
    """(2(nx+ny), 2) integer points of the global perimeter in G6 order."""
    pts = []
    pts += [(x, 0) for x in range(0, nx)]
    pts += [(nx, y) for y in range(0, ny)]
    pts += [(x, ny) for x in range(nx, 0, -1)]
    pts += [(0, y) for y in range(ny, 0, -1)]
    return np.asarray(pts, np.int64)


def closed_form_boundary(nx: int, ny: int, f, h: float = 1.0 / 64.0) -> np.ndarray:
    """g = f(x h, y h) on the perimeter (fp64)."""
    p = boundary_points(nx, ny).astype(np.float64) * h
    return np.asarray(f(p[:, 0], p[:, 1]), np.float64)


def sine_boundary(nx: int, ny: int, h: float = 1.0 / 64.0) -> np.ndarray:
    """The paper's evaluation boundary g(x) = sin(2 pi x) (Fig. gfnet-eval),
    x in domain units (64 points per unit), on every boundary point (fp64)."""
    return closed_form_boundary(nx, ny, lambda x, y: np.sin(2.0 * np.pi * x), h)


def sobol_2d(k: int) -> tuple[float, float]:
    import warnings

    from scipy.stats import qmc

    with warnings.catch_warnings():
        warnings.simplefilter("ignore")   # balance warning for n not a power of 2
        pts = qmc.Sobol(d=2, scramble=False).random(k + 1)
    return float(pts[k, 0]), float(pts[k, 1])


def gp_hyperparameters(k: int) -> tuple[float, float]:
    u, v = sobol_2d(k)
    var = GP_VAR_RANGE[0] + u * (GP_VAR_RANGE[1] - GP_VAR_RANGE[0])
    ls = GP_LEN_RANGE[0] + v * (GP_LEN_RANGE[1] - GP_LEN_RANGE[0])
    return var, ls


def gp_curve(n: int, variance: float, lengthscale: float, seed: int) -> np.ndarray:
    """One draw of a 1-D SE-kernel GP at n equispaced positions of [0, 1] (fp64)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    nk = min(n, GP_MAX_KNOTS)
    s = np.linspace(0.0, 1.0, nk)
    K = variance * np.exp(-((s[:, None] - s[None, :]) ** 2) / (2.0 * lengthscale ** 2))
    jitter = 1e-8 * variance if variance > 0 else 1e-12
    for _ in range(4):
        try:
            L = np.linalg.cholesky(K + jitter * np.eye(nk))
            break
        except np.linalg.LinAlgError:
            jitter *= 10.0
    else:
        raise np.linalg.LinAlgError("GP covariance not positive definite after jitter escalation")
    knots = L @ rng.standard_normal(nk)
    if nk == n:
        return knots
    from scipy.interpolate import CubicSpline

    return CubicSpline(s, knots)(np.linspace(0.0, 1.0, n))


def gp_boundary(nx: int, ny: int, k: int = 0) -> np.ndarray:
    """Global GP boundary k (fp32 values returned as float32)."""
    var, ls = gp_hyperparameters(k)
    return gp_curve(2 * (nx + ny), var, ls, GP_SEED_BASE + k).astype(np.float32)


def sdnet_param_shapes(d: int = 128, n_hidden: int = 3, m: int = 32, conv_k=(5, 5), conv_ch=(1, 8, 1)):
    """[(name, shape, fan_in)] in SPEC MFCK declaration order."""
    nb = 4 * m
    out = []
    for l in range(len(conv_k)):
        fan = conv_ch[l] * conv_k[l]
        out.append((f"conv{l}.w", (conv_ch[l + 1], conv_ch[l], conv_k[l]), fan))
        out.append((f"conv{l}.b", (conv_ch[l + 1],), fan))
    fan = conv_ch[-1] * nb + 2   # the concat layer's fan-in (Eq. 3: 4N + 2)
    out.append(("W1", (d, conv_ch[-1] * nb), fan))
    out.append(("W2", (d, 2), fan))
    out.append(("b1", (d,), fan))
    for l in range(n_hidden):
        out.append((f"h{l}.W", (d, d), d))
        out.append((f"h{l}.b", (d,), d))
    out.append(("wo", (d,), d))
    out.append(("bo", (1,), d))
    return out


def random_weights(seed: int = 0, d: int = 128, n_hidden: int = 3, m: int = 32, conv_k=(5, 5),
                   conv_ch=(1, 8, 1)) -> np.ndarray:
    """W-rand: U(+-1/sqrt(fan_in)), PCG64(seed), flat fp32 in MFCK order."""
    rng = np.random.Generator(np.random.PCG64(seed))
    parts = []
    for _, shape, fan in sdnet_param_shapes(d, n_hidden, m, conv_k, conv_ch):
        bound = 1.0 / np.sqrt(fan)
        parts.append(rng.uniform(-bound, bound, size=int(np.prod(shape))))
    return np.concatenate(parts).astype(np.float32)


def split_params(flat: np.ndarray, d: int = 128, n_hidden: int = 3, m: int = 32, conv_k=(5, 5),
                 conv_ch=(1, 8, 1)) -> dict:
    """Named views of a flat MFCK-ordered parameter vector (layout only)."""
    out, off = {}, 0
    for name, shape, _ in sdnet_param_shapes(d, n_hidden, m, conv_k, conv_ch):
        n = int(np.prod(shape))
        out[name] = flat[off: off + n].reshape(shape)
        off += n
    assert off == flat.size, (off, flat.size)
    return out


def random_boundaries(B: int, m: int = 32, seed: int = 1) -> np.ndarray:
    rng = np.random.Generator(np.random.PCG64(seed))
    return rng.standard_normal((B, 4 * m)).astype(np.float32)
