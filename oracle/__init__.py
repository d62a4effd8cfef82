"""oracle — TEST INFRASTRUCTURE ONLY: the fp64 CPU reference of the distributed MFP.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  The product path
(``paper_2308_14258_b200``) never imports it, and this package never imports the
product: they share no code.

The arithmetic lives in ``mfp_oracle.c`` (plain C, fp64, naive loops, OpenMP over
the disjoint subdomains of one class); this module only marshals numpy arrays
through ctypes.  Every C function cites the PAPER.md passage it follows.

Parity status: geometry, exact subsolver, exact-subsolver MFP
(P=1 and emulated P>1), SDNet forward, split layer and cost model are pinned by
``tests/test_oracle_*.py``.  The SDNet-driven MFP trajectory with random weights
has no paper value to pin against: "parity unpinned" beyond the batched ==
sequential, P=1 == plain, and component pins.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "mfp_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

M_DEFAULT = 32


def build(force: bool = False) -> str:
    """Compile mfp_oracle.c with gcc (-O2 -fopenmp).  Building the checker is not using it."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-std=c11", "-o", _LIB, _SRC, "-lm"]
        subprocess.run(cmd, check=True)
    return _LIB


_lib = None


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        P = ctypes.POINTER
        d, i, i64, sz = ctypes.c_double, ctypes.c_int, ctypes.c_int64, ctypes.c_size_t
        L.orc_perimeter.argtypes = [i, i, i, P(i), P(i)]
        L.orc_writeset.argtypes = [i, i, i, P(i), P(i), P(d), P(d)]
        L.orc_interior_queries.argtypes = [i, P(d), P(d)]
        L.orc_anchors.argtypes = [i, i, i, i, P(i), P(i)]
        L.orc_param_count.argtypes = [i, P(i), P(i), i, i, i]
        L.orc_param_count.restype = sz
        L.orc_sdnet_forward.argtypes = [i, P(i), P(i), i, i, i, P(d), i64, P(d), i, P(d), P(d), P(d)]
        L.orc_first_layer_concat.argtypes = [i, i, P(d), P(d), P(d), P(d), i, P(d), P(d), P(d)]
        L.orc_first_layer_split.argtypes = [i, i, P(d), P(d), P(d), P(d), i, P(d), P(d), P(d)]
        L.orc_harmonic_matrix.argtypes = [i, i, P(d)]
        L.orc_mfp_run.argtypes = [ctypes.c_void_p, P(d), P(d), i, d, P(d), P(d), P(d), P(i)]
        L.orc_predict_from_field.argtypes = [ctypes.c_void_p, P(d), P(d), i64, P(i), P(i), i, P(d)]
        L.orc_cost_model.argtypes = [d] * 8 + [P(d)] * 3
        L.orc_num_threads.restype = i
        _lib = L
    return _lib


def _p(a, ct):
    return a.ctypes.data_as(ctypes.POINTER(ct))


def _dp(a):
    return _p(a, ctypes.c_double)


def _ip(a):
    return _p(a, ctypes.c_int)


# --------------------------------------------------------------------------- geometry
def perimeter(ax: int, ay: int, m: int = M_DEFAULT) -> np.ndarray:
    """(4m, 2) global points of a subdomain perimeter in G1 order."""
    px = np.zeros(4 * m, np.int32)
    py = np.zeros(4 * m, np.int32)
    n = lib().orc_perimeter(m, ax, ay, _ip(px), _ip(py))
    return np.stack([px[:n], py[:n]], 1)


def writeset(ax: int, ay: int, m: int = M_DEFAULT):
    """((2m-3, 2) points, (2m-3, 2) local query coords) of the centre lines (G3)."""
    q = 2 * m - 3
    px, py = np.zeros(q, np.int32), np.zeros(q, np.int32)
    qx, qy = np.zeros(q), np.zeros(q)
    lib().orc_writeset(m, ax, ay, _ip(px), _ip(py), _dp(qx), _dp(qy))
    return np.stack([px, py], 1), np.stack([qx, qy], 1)


def interior_queries(m: int = M_DEFAULT) -> np.ndarray:
    q = (m - 1) ** 2
    qx, qy = np.zeros(q), np.zeros(q)
    lib().orc_interior_queries(m, _dp(qx), _dp(qy))
    return np.stack([qx, qy], 1)


def anchors(nx: int, ny: int, cls: int, m: int = M_DEFAULT) -> np.ndarray:
    n = lib().orc_anchors(nx, ny, m, cls, None, None)
    ax, ay = np.zeros(max(n, 1), np.int32), np.zeros(max(n, 1), np.int32)
    lib().orc_anchors(nx, ny, m, cls, _ip(ax), _ip(ay))
    return np.stack([ax[:n], ay[:n]], 1)


# --------------------------------------------------------------------------- SDNet
@dataclass
class NetShape:
    n_conv: int = 2
    conv_k: tuple = (5, 5)
    conv_ch: tuple = (1, 8, 1)
    d: int = 128
    n_hidden: int = 3

    def arrays(self):
        k = np.zeros(8, np.int32)
        k[: self.n_conv] = self.conv_k
        ch = np.zeros(9, np.int32)
        ch[: self.n_conv + 1] = self.conv_ch
        return k, ch


def param_count(net: NetShape, m: int = M_DEFAULT) -> int:
    k, ch = net.arrays()
    return int(lib().orc_param_count(net.n_conv, _ip(k), _ip(ch), net.d, net.n_hidden, m))


def sdnet_forward(params: np.ndarray, gb: np.ndarray, queries: np.ndarray, net: NetShape = NetShape(),
                  m: int = M_DEFAULT) -> np.ndarray:
    """fp64 SDNet forward: gb (B, 4m), queries (q, 2) -> (B, q)."""
    params = np.ascontiguousarray(params, np.float64)
    gb = np.ascontiguousarray(gb, np.float64).reshape(-1, 4 * m)
    qx = np.ascontiguousarray(queries[:, 0], np.float64)
    qy = np.ascontiguousarray(queries[:, 1], np.float64)
    B, q = gb.shape[0], qx.shape[0]
    out = np.zeros((B, q))
    k, ch = net.arrays()
    assert params.size == param_count(net, m)
    lib().orc_sdnet_forward(net.n_conv, _ip(k), _ip(ch), net.d, net.n_hidden, m, _dp(params), B,
                            _dp(gb), q, _dp(qx), _dp(qy), _dp(out))
    return out


def first_layer(kind: str, W1, W2, b1, e, queries) -> np.ndarray:
    W1, W2, b1, e = (np.ascontiguousarray(a, np.float64) for a in (W1, W2, b1, e))
    qx = np.ascontiguousarray(queries[:, 0], np.float64)
    qy = np.ascontiguousarray(queries[:, 1], np.float64)
    d, ne = W1.shape
    U = np.zeros((qx.size, d))
    fn = lib().orc_first_layer_concat if kind == "concat" else lib().orc_first_layer_split
    fn(d, ne, _dp(W1), _dp(W2), _dp(b1), _dp(e), qx.size, _dp(qx), _dp(qy), _dp(U))
    return U


def harmonic_matrix(query_set: int = 0, m: int = M_DEFAULT) -> np.ndarray:
    q = 2 * m - 3 if query_set == 0 else (m - 1) ** 2
    H = np.zeros((q, 4 * m))
    r = lib().orc_harmonic_matrix(m, query_set, _dp(H))
    assert r == q
    return H


# --------------------------------------------------------------------------- MFP
class _Cfg(ctypes.Structure):
    _fields_ = [("nx", ctypes.c_int), ("ny", ctypes.c_int), ("m", ctypes.c_int),
                ("Py", ctypes.c_int), ("Px", ctypes.c_int), ("subsolver", ctypes.c_int),
                ("check_every", ctypes.c_int), ("sequential", ctypes.c_int),
                ("n_conv", ctypes.c_int), ("conv_k", ctypes.c_int * 8),
                ("conv_ch", ctypes.c_int * 9), ("d", ctypes.c_int), ("n_hidden", ctypes.c_int),
                ("exchange_every", ctypes.c_int)]


@dataclass
class MfpConfig:
    nx: int
    ny: int
    m: int = M_DEFAULT
    Py: int = 1
    Px: int = 1
    subsolver: str = "sdnet"   # or "exact"
    check_every: int = 1
    sequential: bool = False
    net: NetShape = field(default_factory=NetShape)
    exchange_every: int = 1    # communication-avoiding variant: halo refresh every s iterations

    def c(self) -> _Cfg:
        k, ch = self.net.arrays()
        return _Cfg(self.nx, self.ny, self.m, self.Py, self.Px, 1 if self.subsolver == "exact" else 0,
                    self.check_every, int(self.sequential), self.net.n_conv,
                    (ctypes.c_int * 8)(*k), (ctypes.c_int * 9)(*ch), self.net.d, self.net.n_hidden,
                    self.exchange_every)


@dataclass
class MfpResult:
    lines: np.ndarray       # (ny+1, nx+1) owner view after the last iteration
    u: np.ndarray | None    # (ny+1, nx+1) final field or None
    deltas: np.ndarray      # delta_k per iteration run
    iterations: int


def mfp_run(cfg: MfpConfig, g: np.ndarray, t: int, tol: float = 0.0, params: np.ndarray | None = None,
            final: bool = True) -> MfpResult:
    """Algorithm 2 in fp64 on a Py x Px emulated processor grid (D1)."""
    assert cfg.m <= 64
    g = np.ascontiguousarray(g, np.float64)
    assert g.size == 2 * (cfg.nx + cfg.ny)
    if params is None:
        assert cfg.subsolver == "exact"
        params = np.zeros(1)
    params = np.ascontiguousarray(params, np.float64)
    lines = np.zeros((cfg.ny + 1, cfg.nx + 1))
    u = np.zeros((cfg.ny + 1, cfg.nx + 1)) if final else None
    deltas = np.zeros(t)
    it = ctypes.c_int(0)
    c = cfg.c()
    r = lib().orc_mfp_run(ctypes.byref(c), _dp(params), _dp(g), t, tol, _dp(lines),
                          _dp(u) if final else None, _dp(deltas), ctypes.byref(it))
    assert r == 0
    return MfpResult(lines, u, deltas[: it.value], it.value)


def predict_from_field(cfg: MfpConfig, U: np.ndarray, anchors_xy: np.ndarray, query_set: int = 0,
                       params: np.ndarray | None = None) -> np.ndarray:
    U = np.ascontiguousarray(U, np.float64)
    ax = np.ascontiguousarray(anchors_xy[:, 0], np.int32)
    ay = np.ascontiguousarray(anchors_xy[:, 1], np.int32)
    q = 2 * cfg.m - 3 if query_set == 0 else (cfg.m - 1) ** 2
    out = np.zeros((ax.size, q))
    params = np.zeros(1) if params is None else np.ascontiguousarray(params, np.float64)
    c = cfg.c()
    r = lib().orc_predict_from_field(ctypes.byref(c), _dp(params), _dp(U), ax.size, _ip(ax), _ip(ay),
                                     query_set, _dp(out))
    assert r == 0
    return out


def cost_model(N, P, m, d, I, alpha, beta, c):
    o = [ctypes.c_double() for _ in range(3)]
    lib().orc_cost_model(N, P, m, d, I, alpha, beta, c, *[ctypes.byref(x) for x in o])
    return tuple(x.value for x in o)


def num_threads() -> int:
    return int(lib().orc_num_threads())
