"""The tensor-core epilogues' GELU forms (device_common.cuh) against the exact
GELU x Phi(x) of PAPER.md P:241 (the oracle's, erf-based), in fp64 on the CPU:
the constants the kernels compile are read from the header and evaluated here.

* classic tanh form (mfp_sdnet_desc.gelu = 1): |2 GELU error| <= 9.5e-4;
* accurate form (gelu = 2, the FP16X accuracy mode): tanh(x (a0 + t (a1 + t a2))),
  t = min(x^2, 16): |2 GELU error| <= 5.1e-5 everywhere, and odd-symmetric.
"""
import os
import re

import numpy as np
from scipy.special import erf

HDR = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2308_14258_b200", "csrc",
                   "device_common.cuh")


def consts():
    src = open(HDR).read()
    out = {}
    for name in ("kGF0", "kGA0", "kGA1", "kGA2"):
        m = re.search(name + r"\s*=\s*([-0-9.eE+]+)f", src)
        out[name] = float(m.group(1))
    m = re.search(r"kGF1\s*=\s*([-0-9.eE+]+)f\s*\*\s*([-0-9.eE+]+)f", src)
    out["kGF1"] = float(m.group(1)) * float(m.group(2))
    return out


X = np.linspace(-12.0, 12.0, 480001)
EXACT2 = X + X * erf(X / np.sqrt(2.0))     # 2 GELU(x)


def test_classic_form_bound():
    c = consts()
    h = X + X * np.tanh(X * (c["kGF0"] + c["kGF1"] * X * X))
    assert np.max(np.abs(h - EXACT2)) <= 9.6e-4


def test_accurate_form_bound_and_symmetry():
    c = consts()
    t = np.minimum(X * X, 16.0)
    h = X + X * np.tanh(X * (c["kGA0"] + t * (c["kGA1"] + t * c["kGA2"])))
    err = np.abs(h - EXACT2)
    assert err.max() <= 5.1e-5
    # small arguments, where most pre-activations sit: relative accuracy too
    small = np.abs(X) < 0.5
    assert np.max(err[small] / np.maximum(np.abs(EXACT2[small]), 1e-30)) < 1e-3
    # 2 GELU(x) - x = x tanh(x P(x^2)) is even, as x erf(x / sqrt 2) is
    assert np.allclose(h[::-1] - X[::-1], h - X, rtol=0, atol=1e-12)
