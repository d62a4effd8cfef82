"""Thin ctypes binding of libmfp (include/mfp.h) — argument marshalling only.

Every numeric step runs inside libmfp's sm_100a kernels; this module converts
Python/numpy/torch arguments to C pointers and status codes to exceptions.
PyTorch is used for device memory (the caller-owned workspace) and streams.
There is no CPU fallback: if libmfp.so is missing, importing this module raises.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libmfp.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(f"libmfp.so not built at {LIB_PATH}: run `python paper_2308_14258_b200/build.py`")

_lib = ctypes.CDLL(LIB_PATH)

ABI_VERSION = 1
ALL_RANKS = -1
FP32, BF16, FP16, FP16X = 0, 1, 2, 3
SDNET, EXACT_LAPLACE = 0, 1
QUERY_CENTRE, QUERY_INTERIOR = 0, 1

STATUS = {0: "OK", 1: "ERR_INVALID", 2: "ERR_NOT_TILEABLE", 3: "ERR_NONFINITE", 4: "NOT_CONVERGED",
          5: "ERR_CUDA", 6: "ERR_NCCL", 7: "ERR_WORKSPACE", 8: "ERR_STATE"}
OK, NOT_CONVERGED = 0, 4


class MfpError(RuntimeError):
    def __init__(self, status: int, msg: str = ""):
        super().__init__(f"mfp status {status} ({STATUS.get(status, '?')}): {msg}")
        self.status = status


class mfp_config(ctypes.Structure):
    _fields_ = [("abi", ctypes.c_uint32), ("nx", ctypes.c_int32), ("ny", ctypes.c_int32),
                ("m", ctypes.c_int32), ("stride", ctypes.c_int32), ("grid_rows", ctypes.c_int32),
                ("grid_cols", ctypes.c_int32), ("precision", ctypes.c_int32),
                ("subsolver", ctypes.c_int32), ("check_every", ctypes.c_int32)]


class mfp_sdnet_desc(ctypes.Structure):
    _fields_ = [("n_conv", ctypes.c_int32), ("conv_k", ctypes.c_int32 * 4), ("conv_ch", ctypes.c_int32 * 5),
                ("d", ctypes.c_int32), ("n_hidden", ctypes.c_int32), ("gelu", ctypes.c_int32)]


class mfp_report(ctypes.Structure):
    _fields_ = [("iterations", ctypes.c_int32), ("converged", ctypes.c_int32), ("last_delta", ctypes.c_float),
                ("pad_", ctypes.c_float), ("predictions", ctypes.c_double),
                ("predictions_computed", ctypes.c_double), ("ms_total", ctypes.c_double),
                ("ms_final", ctypes.c_double), ("halo_bytes_sent", ctypes.c_int64),
                ("halo_msgs_per_iter", ctypes.c_int32), ("gpu_launches", ctypes.c_int32)]


class mfp_profile(ctypes.Structure):
    _fields_ = [("iterations", ctypes.c_int32), ("launches_per_iter", ctypes.c_int32),
                ("ms_per_iter", ctypes.c_double), ("ms_gather_embed", ctypes.c_double),
                ("ms_chain", ctypes.c_double), ("ms_exact", ctypes.c_double), ("ms_halo", ctypes.c_double),
                ("ms_delta", ctypes.c_double), ("chain_launches", ctypes.c_int64),
                ("chain_rows", ctypes.c_int64), ("chain_ms_total", ctypes.c_double),
                ("gather_launches", ctypes.c_int64), ("gather_subdomains", ctypes.c_int64),
                ("gather_ms_total", ctypes.c_double)]


class mfp_plan_info(ctypes.Structure):
    _fields_ = [("rank", ctypes.c_int32), ("ry", ctypes.c_int32), ("rx", ctypes.c_int32),
                ("X0", ctypes.c_int32), ("X1", ctypes.c_int32), ("Y0", ctypes.c_int32), ("Y1", ctypes.c_int32),
                ("RX0", ctypes.c_int32), ("RX1", ctypes.c_int32), ("RY0", ctypes.c_int32), ("RY1", ctypes.c_int32),
                ("phase_count", ctypes.c_int64 * 4), ("final_count", ctypes.c_int64),
                ("n_peers", ctypes.c_int32), ("peers", ctypes.c_int32 * 8),
                ("send_count", ctypes.c_int64 * 8), ("recv_count", ctypes.c_int64 * 8),
                ("lattice_cells", ctypes.c_int64), ("n_hlines", ctypes.c_int32), ("n_vlines", ctypes.c_int32),
                ("hline_len", ctypes.c_int32), ("vline_len", ctypes.c_int32),
                ("phase0_interior", ctypes.c_int64)]


_P = ctypes.POINTER
_vp, _i32, _i64, _sz, _f32, _f64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_size_t, ctypes.c_float, ctypes.c_double
_SIGS = {
    "mfp_workspace_size": [_P(mfp_config), _P(mfp_sdnet_desc), ctypes.c_int, _P(_sz)],
    "mfp_param_count": [_P(mfp_sdnet_desc), _i32, _P(_sz)],
    "mfp_init": [_P(mfp_config), _P(mfp_sdnet_desc), _vp, _sz, ctypes.c_int, _vp, _vp, _sz, _vp, _P(_vp)],
    "mfp_destroy": [_vp],
    "mfp_last_error": [_vp],
    "mfp_solve": [_vp, _vp, _i32, _f32, _vp, _P(mfp_report)],
    "mfp_solve_device": [_vp, _vp, _i32, _f32, _vp, _P(mfp_report)],
    "mfp_sdnet_batch": [_vp, _vp, _i64, _i32, _vp, _vp],
    "mfp_step_phase": [_vp, _i32],
    "mfp_export_lines": [_vp, _i32, _vp, _vp],
    "mfp_import_lines": [_vp, _i32, _vp, _vp],
    "mfp_profile_iterations": [_vp, _i32, _P(mfp_profile)],
    "mfp_plan_query": [_P(mfp_config), _i32, _P(mfp_plan_info)],
    "mfp_plan_anchors": [_P(mfp_config), _i32, _i32, _P(_i32), _P(_i32), _i64, _P(_i64)],
    "mfp_plan_halo": [_P(mfp_config), _i32, _i32, _i32, _P(_i32), _P(_i32), _P(_i32), _i64, _P(_i64)],
    "mfp_cost_model": [_f64] * 8 + [_P(_f64)] * 3,
    "mfp_gather_phase": [_vp, _i32, _i32, _vp, _i64, _P(_i64), _P(_i32), _P(_i32)],
    "mfp_scatter_phase": [_vp, _i32, _i32, _vp, _i64, _P(ctypes.c_float)],
    "mfp_set_exchange_every": [_vp, _i32],
    "mfp_p2p_export": [_vp, _vp],
    "mfp_p2p_open": [_vp, _vp, _i32],
    "mfp_p2p_set_mode": [_vp, _i32],
    "mfp_nccl_get_unique_id": [_vp],
    "mfp_nccl_comm_init": [_i32, _vp, _i32, _P(_vp)],
    "mfp_nccl_comm_destroy": [_vp],
}
EXPORTS = tuple(_SIGS)
for _name, _args in _SIGS.items():
    _fn = getattr(_lib, _name)
    _fn.argtypes = _args
    _fn.restype = ctypes.c_char_p if _name == "mfp_last_error" else (None if _name == "mfp_destroy" else ctypes.c_int)


def _check(st: int, ctx=None, allow=(OK,)) -> int:
    if st not in allow:
        msg = _lib.mfp_last_error(ctx).decode() if ctx else ""
        raise MfpError(st, msg)
    return st


def _ptr(a) -> int | None:
    """Pointer of a numpy array or torch tensor (device or host)."""
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        assert a.flags["C_CONTIGUOUS"]
        return a.ctypes.data
    assert a.is_contiguous()
    return a.data_ptr()


# ------------------------------------------------------------------ config helpers
def make_config(nx: int, ny: int, grid=(1, 1), precision: int = FP32, subsolver: int = SDNET,
                check_every: int = 16, m: int = 32) -> mfp_config:
    return mfp_config(ABI_VERSION, nx, ny, m, m // 2, grid[0], grid[1], precision, subsolver, check_every)


def make_net(d: int = 128, n_hidden: int = 3, gelu: int = 0) -> mfp_sdnet_desc:
    return mfp_sdnet_desc(2, (ctypes.c_int32 * 4)(5, 5, 0, 0), (ctypes.c_int32 * 5)(1, 8, 1, 0, 0), d, n_hidden, gelu)


# ------------------------------------------------------------------ C-ABI mirrors
def mfp_workspace_size(cfg: mfp_config, net: mfp_sdnet_desc, rank: int) -> int:
    n = _sz(0)
    _check(_lib.mfp_workspace_size(ctypes.byref(cfg), ctypes.byref(net), rank, ctypes.byref(n)))
    return n.value


def mfp_param_count(net: mfp_sdnet_desc, m: int = 32) -> int:
    n = _sz(0)
    _check(_lib.mfp_param_count(ctypes.byref(net), m, ctypes.byref(n)))
    return n.value


def mfp_init(cfg, net, params, rank, nccl_comm, workspace, stream):
    """Returns the opaque context pointer.  params: host fp32 numpy or None."""
    ctx = _vp(None)
    if params is not None:
        params = np.ascontiguousarray(params, np.float32)
    ws_bytes = workspace.numel() * workspace.element_size()
    st = _lib.mfp_init(ctypes.byref(cfg), ctypes.byref(net), _ptr(params), 0 if params is None else params.size,
                       rank, nccl_comm, workspace.data_ptr(), ws_bytes, stream, ctypes.byref(ctx))
    if st != OK:
        msg = _lib.mfp_last_error(ctx).decode() if ctx.value else ""
        _lib.mfp_destroy(ctx)
        raise MfpError(st, msg)
    return ctx


def mfp_destroy(ctx) -> None:
    _lib.mfp_destroy(ctx)


def mfp_solve(ctx, g: np.ndarray | None, max_iters: int, tol: float, u_out: np.ndarray | None) -> mfp_report:
    rep = mfp_report()
    if g is not None:
        g = np.ascontiguousarray(g, np.float32)
    _check(_lib.mfp_solve(ctx, _ptr(g), max_iters, tol, _ptr(u_out), ctypes.byref(rep)), ctx, (OK, NOT_CONVERGED))
    return rep


def mfp_solve_device(ctx, g_dev, max_iters: int, tol: float, u_dev) -> mfp_report:
    rep = mfp_report()
    _check(_lib.mfp_solve_device(ctx, _ptr(g_dev), max_iters, tol, _ptr(u_dev), ctypes.byref(rep)), ctx,
           (OK, NOT_CONVERGED))
    return rep


def mfp_sdnet_batch(ctx, gb_dev, B: int, query_set: int, out_dev, stream=None) -> None:
    _check(_lib.mfp_sdnet_batch(ctx, _ptr(gb_dev), B, query_set, _ptr(out_dev), stream), ctx)


def mfp_gather_phase(ctx, rank: int, phase: int, gb_dev=None, cap: int = 0, want_anchors: bool = False):
    """a1 standalone: returns (B, anchors (B, 2) int32 (ax, ay) or None); gb_dev=None and
    want_anchors=False is a size query."""
    B = _i64(0)
    _check(_lib.mfp_gather_phase(ctx, rank, phase, None, 0, ctypes.byref(B), None, None), ctx)
    ax = ay = None
    if want_anchors:
        ax, ay = np.zeros(max(B.value, 1), np.int32), np.zeros(max(B.value, 1), np.int32)
    if gb_dev is not None or want_anchors:
        _check(_lib.mfp_gather_phase(ctx, rank, phase, _ptr(gb_dev), max(cap, B.value if gb_dev is None else cap),
                                     ctypes.byref(B), None if ax is None else ax.ctypes.data_as(_P(_i32)),
                                     None if ay is None else ay.ctypes.data_as(_P(_i32))), ctx)
    anchors = np.stack([ax[:B.value], ay[:B.value]], 1) if want_anchors else None
    return B.value, anchors


def mfp_scatter_phase(ctx, rank: int, phase: int, pred_dev, B: int, want_norm: bool = True):
    """a6 + a8 standalone: returns the update norm max |new - old| (syncs) or None."""
    v = ctypes.c_float(0.0)
    _check(_lib.mfp_scatter_phase(ctx, rank, phase, _ptr(pred_dev), B, ctypes.byref(v) if want_norm else None), ctx)
    return v.value if want_norm else None


def mfp_set_exchange_every(ctx, s: int) -> None:
    _check(_lib.mfp_set_exchange_every(ctx, s), ctx)


def mfp_p2p_export(ctx) -> bytes:
    """NEXT-2: this rank's 64-byte IPC handle of its peer-memory halo region."""
    h = ctypes.create_string_buffer(64)
    _check(_lib.mfp_p2p_export(ctx, h), ctx)
    return h.raw


def mfp_p2p_open(ctx, handles=None) -> None:
    """NEXT-2: switch to the peer-memory halo transport.  handles: the R
    exported handles in rank order (one process per GPU), None for ALL_RANKS."""
    if handles is not None:
        handles = list(handles)
        if any(len(h) != 64 for h in handles):
            raise MfpError(1, "p2p_open: every handle must be 64 bytes")
    buf = None if handles is None else ctypes.create_string_buffer(b"".join(handles), 64 * len(handles))
    _check(_lib.mfp_p2p_open(ctx, buf, 0 if handles is None else len(handles)), ctx)


P2P_PULL, P2P_PUT = 0, 1


def mfp_p2p_set_mode(ctx, mode: int) -> None:
    """NEXT-2: after mfp_p2p_open, P2P_PUT makes the chain epilogue store halo
    cells straight into the peers' put buffers (P2P_PULL: pack + pull)."""
    _check(_lib.mfp_p2p_set_mode(ctx, mode), ctx)


def mfp_step_phase(ctx, phase: int) -> None:
    _check(_lib.mfp_step_phase(ctx, phase), ctx)


def mfp_export_lines(ctx, rank: int, hl: np.ndarray, vl: np.ndarray) -> None:
    _check(_lib.mfp_export_lines(ctx, rank, _ptr(hl), _ptr(vl)), ctx)


def mfp_import_lines(ctx, rank: int, hl: np.ndarray, vl: np.ndarray) -> None:
    _check(_lib.mfp_import_lines(ctx, rank, _ptr(np.ascontiguousarray(hl, np.float32)),
                                 _ptr(np.ascontiguousarray(vl, np.float32))), ctx)


def mfp_profile_iterations(ctx, iters: int) -> mfp_profile:
    p = mfp_profile()
    _check(_lib.mfp_profile_iterations(ctx, iters, ctypes.byref(p)), ctx)
    return p


def mfp_plan_query(cfg: mfp_config, rank: int) -> mfp_plan_info:
    info = mfp_plan_info()
    _check(_lib.mfp_plan_query(ctypes.byref(cfg), rank, ctypes.byref(info)))
    return info


def mfp_plan_anchors(cfg: mfp_config, rank: int, phase: int) -> np.ndarray:
    n = _i64(0)
    _check(_lib.mfp_plan_anchors(ctypes.byref(cfg), rank, phase, None, None, 0, ctypes.byref(n)))
    ax = np.zeros(max(n.value, 1), np.int32)
    ay = np.zeros(max(n.value, 1), np.int32)
    _check(_lib.mfp_plan_anchors(ctypes.byref(cfg), rank, phase, ax.ctypes.data_as(_P(_i32)),
                                 ay.ctypes.data_as(_P(_i32)), ax.size, ctypes.byref(n)))
    return np.stack([ax[: n.value], ay[: n.value]], 1)


def mfp_plan_halo(cfg: mfp_config, rank: int, peer_idx: int, direction: int) -> np.ndarray:
    """(n, 3) rows (kind, x, y): kind 0 = horizontal-line cell, 1 = vertical."""
    n = _i64(0)
    _check(_lib.mfp_plan_halo(ctypes.byref(cfg), rank, peer_idx, direction, None, None, None, 0, ctypes.byref(n)))
    k, x, y = (np.zeros(max(n.value, 1), np.int32) for _ in range(3))
    _check(_lib.mfp_plan_halo(ctypes.byref(cfg), rank, peer_idx, direction, k.ctypes.data_as(_P(_i32)),
                              x.ctypes.data_as(_P(_i32)), y.ctypes.data_as(_P(_i32)), k.size, ctypes.byref(n)))
    return np.stack([k[: n.value], x[: n.value], y[: n.value]], 1)


def mfp_cost_model(N, P, m, d, I, alpha, beta, c):
    o = [_f64() for _ in range(3)]
    _check(_lib.mfp_cost_model(N, P, m, d, I, alpha, beta, c, *[ctypes.byref(v) for v in o]))
    return tuple(v.value for v in o)


def mfp_nccl_get_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(_lib.mfp_nccl_get_unique_id(buf))
    return buf.raw


def mfp_nccl_comm_init(nranks: int, uid: bytes, rank: int):
    comm = _vp(None)
    buf = ctypes.create_string_buffer(uid, 128)
    _check(_lib.mfp_nccl_comm_init(nranks, buf, rank, ctypes.byref(comm)))
    return comm


def mfp_nccl_comm_destroy(comm) -> None:
    _check(_lib.mfp_nccl_comm_destroy(comm))


# ------------------------------------------------------------------ convenience
@dataclass
class Lattice:
    hl: np.ndarray   # (n_hlines, hline_len): y = RY0 + 16 i, x = RX0 .. RX1
    vl: np.ndarray   # (n_vlines, vline_len): x = RX0 + 16 j, y = RY0 .. RY1
    info: mfp_plan_info


class Mfp:
    """Owns a context + its torch-allocated workspace on the current CUDA device."""

    def __init__(self, cfg: mfp_config, net: mfp_sdnet_desc | None = None, params=None, rank: int = 0,
                 nccl_comm=None, stream=None):
        import torch

        self.cfg = cfg
        self.net = net if net is not None else make_net()
        self.rank = rank
        nbytes = mfp_workspace_size(cfg, self.net, rank)
        self.workspace = torch.empty(nbytes + 256, dtype=torch.uint8, device="cuda")
        off = (-self.workspace.data_ptr()) % 256
        self.ws = self.workspace[off: off + nbytes]
        # a dedicated (capturable) stream by default: the library replays blocks
        # of iterations as CUDA graphs, which the legacy default stream forbids
        self.stream = stream if stream is not None else torch.cuda.Stream()
        self.ctx = mfp_init(cfg, self.net, params, rank, nccl_comm, self.ws, self.stream.cuda_stream)

    def _enter(self):
        import torch
        self.stream.wait_stream(torch.cuda.current_stream())

    def _leave(self):
        import torch
        torch.cuda.current_stream().wait_stream(self.stream)

    @property
    def ranks(self):
        R = self.cfg.grid_rows * self.cfg.grid_cols
        return list(range(R)) if self.rank == ALL_RANKS else [self.rank]

    def solve(self, g, max_iters, tol=0.0, want_u=True):
        nx, ny = self.cfg.nx, self.cfg.ny
        u = np.zeros((ny + 1, nx + 1), np.float32) if want_u else None
        rep = mfp_solve(self.ctx, g, max_iters, tol, u)
        return u, rep

    def solve_device(self, g_dev, max_iters, tol, u_dev):
        self._enter()
        rep = mfp_solve_device(self.ctx, g_dev, max_iters, tol, u_dev)
        self._leave()
        return rep

    def sdnet_batch(self, gb_dev, query_set=QUERY_CENTRE, out=None):
        import torch

        q = 61 if query_set == QUERY_CENTRE else 961
        B = gb_dev.shape[0]
        if out is None:
            out = torch.empty((B, q), dtype=torch.float32, device=gb_dev.device)
        self._enter()
        mfp_sdnet_batch(self.ctx, gb_dev, B, query_set, out, self.stream.cuda_stream)
        self._leave()
        return out

    def lines(self, rank: int | None = None) -> Lattice:
        r = self.ranks[0] if rank is None else rank
        info = mfp_plan_query(self.cfg, r)
        hl = np.zeros((info.n_hlines, info.hline_len), np.float32)
        vl = np.zeros((info.n_vlines, info.vline_len), np.float32)
        mfp_export_lines(self.ctx, r if self.rank == ALL_RANKS else 0, hl, vl)
        return Lattice(hl, vl, info)

    def set_lines(self, hl, vl, rank: int | None = None):
        r = self.ranks[0] if rank is None else rank
        mfp_import_lines(self.ctx, r if self.rank == ALL_RANKS else 0, hl, vl)

    def step_phase(self, phase: int):
        mfp_step_phase(self.ctx, phase)

    def _io_rank(self, rank):
        return 0 if self.rank != ALL_RANKS else (0 if rank is None else rank)

    def gather_phase(self, phase: int, out=None, rank: int | None = None, want_anchors: bool = False):
        """Perimeters (B, 128) of the phase's subdomains from the current lattice (a1)."""
        import torch

        r = self._io_rank(rank)
        B, _ = mfp_gather_phase(self.ctx, r, phase)
        if out is None:
            out = torch.empty((max(B, 1), 128), dtype=torch.float32, device="cuda")
        self._enter()
        _, anc = mfp_gather_phase(self.ctx, r, phase, out, out.shape[0], want_anchors)
        self._leave()
        return (out[:B], anc) if want_anchors else out[:B]

    def scatter_phase(self, phase: int, pred, rank: int | None = None, want_norm: bool = True):
        """Write (B, 61) centre-line predictions onto the lattice (a6); returns max |new - old|."""
        self._enter()
        v = mfp_scatter_phase(self.ctx, self._io_rank(rank), phase, pred, pred.shape[0], want_norm)
        self._leave()
        return v

    def profile(self, iters: int) -> mfp_profile:
        return mfp_profile_iterations(self.ctx, iters)

    def lines_bytes(self, rank: int | None = None) -> int:
        info = mfp_plan_query(self.cfg, self.ranks[0] if rank is None else rank)
        return 4 * (info.n_hlines * info.hline_len + info.n_vlines * info.vline_len)

    def close(self):
        if getattr(self, "ctx", None) is not None:
            mfp_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
