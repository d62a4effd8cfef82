#!/usr/bin/env python
"""Minimax fit of the FMA-pipe GELU used for part of the tensor-core epilogue.

The epilogue computes h' = 2 GELU_tanh(x) = x + e(x) with
    e(x) = x tanh(G0 x + G1 x^3)          (even, 0 <= e <= |x|).
MUFU tanh is the binding unit of the chain, so a fraction of the
elements take a pure-FMA path instead:
    t = x^2,  e ~= min(t R(min(t, T)), |x|),   R a degree-(n-1) polynomial,
evaluated in fp32x2 (FFMA2).  This script finds R by linear-programming minimax
on x in [0, a] (T = a^2), weighting the error by 1 / max(|h'(x)|, floor) so the
relative error of h' is bounded where it is small (x < 0), and reports the
max error over the whole line including the clamped tails.

    python tools/fit_gelu_poly.py --n 6 --a 3.4
"""
import argparse

import numpy as np
from scipy.optimize import linprog

G0 = 0.7978845608028654
G1 = G0 * 0.044715


def e_true(x):
    return x * np.tanh(G0 * x + G1 * x ** 3)


def fit(n, a, floor=0.05, npts=3000):
    x = np.linspace(0.0, a, npts)
    t = x * x
    # unknowns: c_0..c_{n-1}, eps ; minimise eps s.t. |w (t R(t) - e)| <= eps, both signs of x
    w = np.maximum(1.0 / np.maximum(np.abs(x + e_true(x)), floor), 1.0 / np.maximum(np.abs(-x + e_true(x)), floor))
    V = (t[:, None] ** np.arange(n)[None, :]) * t[:, None]
    A = np.vstack([np.hstack([w[:, None] * V, -np.ones((npts, 1))]), np.hstack([-w[:, None] * V, -np.ones((npts, 1))])])
    b = np.concatenate([w * e_true(x), -w * e_true(x)])
    c = np.zeros(n + 1)
    c[-1] = 1.0
    res = linprog(c, A_ub=A, b_ub=b, bounds=[(None, None)] * (n + 1), method="highs")
    return res.x[:n], res.x[n]


def approx(coef, a, x):
    t = x * x
    tc = np.minimum(t, a * a)
    R = np.zeros_like(x)
    for ck in coef[::-1]:
        R = R * tc + ck
    return x + np.minimum(t * R, np.abs(x))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=6)
    ap.add_argument("--a", type=float, default=3.4)
    args = ap.parse_args()
    coef, eps = fit(args.n, args.a)
    x = np.linspace(-12, 12, 480001)
    h = x + e_true(x)
    err = np.abs(approx(coef.astype(np.float32).astype(np.float64), args.a, x) - h)
    print(f"n={args.n} a={args.a} weighted minimax eps={eps:.3e}  max|dh'|={err.max():.3e}  "
          f"max|dh'|/max(|h'|,0.05)={np.max(err / np.maximum(np.abs(h), 0.05)):.3e}")
    print("coefficients (R(t) = sum c_k t^k):")
    print(", ".join(f"{float(np.float32(c)):.9e}f" for c in coef))


if __name__ == "__main__":
    main()
