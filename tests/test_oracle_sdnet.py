"""Pins for the oracle's SDNet forward (Eq. 5; reading G7).

The independent reference is torch fp64 library ops (F.conv1d with circular
padding, F.linear, F.gelu exact) — a different implementation of the same
definition; plus the algebraic identities the paper states (Eq. 5 == Eq. 3).
"""
import math

import numpy as np
import pytest
import torch
import torch.nn.functional as F

import oracle
from mfp_inputs import random_boundaries, random_weights, split_params
from tests.conftest import load_golden  # noqa: F401

M = 32


def torch_sdnet(flat, gb, queries, d=128, n_hidden=3):
    p = {k: torch.tensor(v, dtype=torch.float64) for k, v in split_params(flat.astype(np.float64), d, n_hidden).items()}
    x = torch.tensor(gb, dtype=torch.float64)[:, None, :]           # (B, 1, 4m)
    for l in range(2):
        x = F.gelu(F.conv1d(F.pad(x, (2, 2), mode="circular"), p[f"conv{l}.w"], p[f"conv{l}.b"]))
    e = x.flatten(1)                                                # (B, 4m)
    z = F.linear(e, p["W1"], p["b1"])                               # (B, d)
    X = torch.tensor(queries, dtype=torch.float64)                  # (q, 2)
    h = F.gelu(z[:, None, :] + F.linear(X, p["W2"])[None])          # broadcasted sum, Eq. 5
    for l in range(n_hidden):
        h = F.gelu(F.linear(h, p[f"h{l}.W"], p[f"h{l}.b"]))
    return (F.linear(h, p["wo"][None], p["bo"])[..., 0]).numpy()


@pytest.mark.parametrize("qs", [0, 1])
def test_sdnet_matches_torch_fp64(qs):
    flat = random_weights(0).astype(np.float64)
    gb = random_boundaries(6, seed=3).astype(np.float64)
    q = oracle.writeset(0, 0)[1] if qs == 0 else oracle.interior_queries()
    got = oracle.sdnet_forward(flat, gb, q)
    want = torch_sdnet(flat, gb, q)
    assert np.max(np.abs(got - want)) < 1e-12 * max(1.0, np.max(np.abs(want)))


@pytest.mark.parametrize("d,nh", [(64, 2), (256, 3)])
def test_sdnet_other_width(d, nh):
    """Other widths, including the wide variant the d = 256 kernels are checked
    against (SURVEY §8(b) d = 128 | 256)."""
    net = oracle.NetShape(d=d, n_hidden=nh)
    flat = random_weights(5, d=d, n_hidden=nh).astype(np.float64)
    gb = random_boundaries(3, seed=4).astype(np.float64)
    for q in (oracle.writeset(0, 0)[1], oracle.interior_queries()):
        got = oracle.sdnet_forward(flat, gb, q, net=net)
        want = torch_sdnet(flat, gb, q, d=d, n_hidden=nh)
        assert np.max(np.abs(got - want)) < 1e-12 * max(1.0, np.max(np.abs(want)))


def test_param_count_matches_layout():
    assert oracle.param_count(oracle.NetShape()) == random_weights(0).size == 66522


def test_zero_params_zero_output():
    """all-zero theta -> all-zero predictions (GELU(0) = 0)."""
    flat = np.zeros(oracle.param_count(oracle.NetShape()))
    out = oracle.sdnet_forward(flat, random_boundaries(2), oracle.writeset(0, 0)[1])
    assert np.all(out == 0.0)


def test_row_permutation_equivariance():
    """permuting query rows permutes predictions identically."""
    flat = random_weights(1).astype(np.float64)
    gb = random_boundaries(2, seed=9).astype(np.float64)
    q = oracle.interior_queries()[:50]
    perm = np.random.default_rng(0).permutation(50)
    a = oracle.sdnet_forward(flat, gb, q)
    b = oracle.sdnet_forward(flat, gb, q[perm])
    assert np.array_equal(a[:, perm], b)


def test_identity_conv_reduces_to_gelu():
    """S:322 special case: one 1x1 conv with unit weight, W1 = I, W2 = 0, no hidden
    layer, wo = e_j -> y = gelu(gelu(g_j)), the textbook GELU x*Phi(x)."""
    net = oracle.NetShape(n_conv=1, conv_k=(1,), conv_ch=(1, 1), d=4 * M, n_hidden=0)
    n = oracle.param_count(net)
    flat = np.zeros(n)
    flat[0] = 1.0                                   # conv w
    off = 2                                         # after conv w, conv b
    W1 = np.eye(4 * M)
    flat[off: off + W1.size] = W1.ravel()
    off += W1.size + 2 * 4 * M + 4 * M              # W1, W2, b1
    j = 37
    flat[off + j] = 1.0                             # wo = e_j
    g = random_boundaries(1, seed=2).astype(np.float64)
    y = oracle.sdnet_forward(flat, g, np.array([[0.3, 0.7]]), net=net)[0, 0]
    gelu = lambda x: 0.5 * x * (1.0 + math.erf(x / math.sqrt(2.0)))
    assert abs(y - gelu(gelu(g[0, j]))) < 1e-15


def test_gelu_special_values():
    """GELU(0) = 0 and GELU'(0) = 1/2 (through the identity network)."""
    net = oracle.NetShape(n_conv=1, conv_k=(1,), conv_ch=(1, 1), d=4 * M, n_hidden=0)
    flat = np.zeros(oracle.param_count(net))
    flat[0] = 1.0
    flat[2: 2 + (4 * M) ** 2] = np.eye(4 * M).ravel()
    g = np.zeros((1, 4 * M))
    eps = 1e-6
    g[0, 5] = eps
    # with wo = e_5 the output is gelu(gelu(eps)) ~ eps/4 for small eps
    off = 2 + (4 * M) ** 2 + 3 * 4 * M
    flat[off + 5] = 1.0
    y = oracle.sdnet_forward(flat, g, np.array([[0.5, 0.5]]), net=net)[0, 0]
    assert abs(y / eps - 0.25) < 1e-6


def test_split_equals_concat():
    """Eq. 5 is an algebraic identity with Eq. 3: <= 1e-12."""
    rng = np.random.default_rng(7)
    for _ in range(20):
        d, ne, q = 64, 4 * M, int(rng.integers(1, 200))
        W1, W2, b1 = rng.standard_normal((d, ne)) * 0.1, rng.standard_normal((d, 2)), rng.standard_normal(d)
        e = rng.standard_normal(ne)
        X = rng.random((q, 2))
        a = oracle.first_layer("split", W1, W2, b1, e, X)
        b = oracle.first_layer("concat", W1, W2, b1, e, X)
        assert np.max(np.abs(a - b)) <= 1e-12
