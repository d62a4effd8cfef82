"""CPU tests of libmfp's C ABI and host plan (no GPU): exported symbols, config
validation, D1 compute sets and halo lists against brute force,
cost model (§4.3)."""
import re

import numpy as np
import pytest

import oracle
import paper_2308_14258_b200 as mfp
from tests.conftest import ROOT, load_golden

M = 32


def header_functions():
    src = open(f"{ROOT}/include/mfp.h").read()
    return sorted(set(re.findall(r"^\s*(?:mfp_status|void|const char\*)\s+(mfp_\w+)\s*\(", src, re.M)))


def test_every_declared_symbol_is_exported():
    names = header_functions()
    assert len(names) >= 19
    import ctypes
    lib = ctypes.CDLL(mfp.LIB_PATH)
    for n in names:
        assert hasattr(lib, n), n
    assert set(names) == set(mfp.EXPORTS)


@pytest.mark.parametrize("nx,ny,grid,expect", [
    (65, 64, (1, 1), mfp.MfpError), (96, 64, (1, 2), mfp.MfpError), (64, 64, (1, 1), None),
])
def test_config_validation(nx, ny, grid, expect):
    cfg = mfp.make_config(nx, ny, grid)
    if expect is None:
        assert mfp.mfp_workspace_size(cfg, mfp.make_net(), 0) > 0
    else:
        with pytest.raises(expect) as e:
            mfp.mfp_workspace_size(cfg, mfp.make_net(), 0)
        assert e.value.status == 2                     # NOT_TILEABLE


def test_invalid_configs():
    for kw in [dict(m=16), dict(check_every=0)]:
        cfg = mfp.make_config(64, 64, **kw)
        with pytest.raises(mfp.MfpError) as e:
            mfp.mfp_plan_query(cfg, 0)
        assert e.value.status == 1
    cfg = mfp.make_config(64, 64)
    cfg.stride = 8
    with pytest.raises(mfp.MfpError):
        mfp.mfp_plan_query(cfg, 0)
    with pytest.raises(mfp.MfpError):
        mfp.mfp_plan_query(mfp.make_config(64, 64, (1, 2)), 2)     # rank out of range


def test_param_count():
    assert mfp.mfp_param_count(mfp.make_net()) == oracle.param_count(oracle.NetShape()) == 66522
    assert mfp.mfp_param_count(mfp.make_net(d=256)) == oracle.param_count(oracle.NetShape(d=256))


def test_net_and_precision_validation():
    """d = 128 | 256; gelu 0 / 1 / 2 (exact, classic tanh, accurate
    tanh); precisions FP32 / BF16 / FP16 / FP16X — anything else is INVALID."""
    cfg = mfp.make_config(64, 64)
    w128 = mfp.mfp_workspace_size(cfg, mfp.make_net(), 0)
    w256 = mfp.mfp_workspace_size(cfg, mfp.make_net(d=256), 0)
    assert w256 > w128 > 0
    for gelu in (0, 1, 2):
        assert mfp.mfp_workspace_size(cfg, mfp.make_net(gelu=gelu), 0) == w128
    for net in (mfp.make_net(d=192), mfp.make_net(d=64), mfp.make_net(gelu=3), mfp.make_net(n_hidden=4)):
        with pytest.raises(mfp.MfpError) as e:
            mfp.mfp_workspace_size(cfg, net, 0)
        assert e.value.status == 1
    for prec in (mfp.FP32, mfp.BF16, mfp.FP16, mfp.FP16X):
        assert mfp.mfp_workspace_size(mfp.make_config(64, 64, precision=prec), mfp.make_net(), 0) > 0
    with pytest.raises(mfp.MfpError) as e:
        mfp.mfp_workspace_size(mfp.make_config(64, 64, precision=4), mfp.make_net(), 0)
    assert e.value.status == 1


@pytest.mark.parametrize("K", [2, 4, 16])
def test_single_rank_phases_are_classes(K):
    nx = ny = K * M
    cfg = mfp.make_config(nx, ny)
    for c in range(4):
        got = mfp.mfp_plan_anchors(cfg, 0, c)
        want = oracle.anchors(nx, ny, c)
        assert np.array_equal(got, want)
    fin = mfp.mfp_plan_anchors(cfg, 0, 4)
    assert np.array_equal(fin, oracle.anchors(nx, ny, 0))


def brute_owner(nx, ny, grid, x, y):
    Py, Px = grid
    Lx, Ly = nx // Px, ny // Py
    return min(y // Ly, Py - 1) * Px + min(x // Lx, Px - 1)


def brute_read_region(nx, ny, grid, r):
    Py, Px = grid
    Lx, Ly = nx // Px, ny // Py
    ry, rx = divmod(r, Px)
    X0, Y0 = rx * Lx, ry * Ly
    return max(0, X0 - 16), min(nx, X0 + Lx + 16), max(0, Y0 - 16), min(ny, Y0 + Ly + 16)


GRIDS = [((1, 2), 4, 4), ((2, 2), 4, 4), ((2, 4), 8, 4), ((3, 3), 6, 6), ((2, 1), 2, 4)]


@pytest.mark.parametrize("grid,kx,ky", GRIDS)
def test_d1_compute_sets(grid, kx, ky):
    """D1: each rank computes every subdomain whose centre is in its closed block;
    together the ranks cover every subdomain, and every owned line point's
    writers are computed by its owner (the sequential writer set)."""
    nx, ny = kx * M, ky * M
    cfg = mfp.make_config(nx, ny, grid)
    R = grid[0] * grid[1]
    for c in range(4):
        allc = {tuple(a) for a in oracle.anchors(nx, ny, c)}
        seen = set()
        for r in range(R):
            info = mfp.mfp_plan_query(cfg, r)
            got = {tuple(a) for a in mfp.mfp_plan_anchors(cfg, r, c)}
            want = {(ax, ay) for ax, ay in allc
                    if info.X0 <= ax + 16 <= info.X1 and info.Y0 <= ay + 16 <= info.Y1}
            assert got == want
            seen |= got
            # owner computes every writer of its owned points
            for ax, ay in allc:
                wr, _ = oracle.writeset(ax, ay)
                if any(brute_owner(nx, ny, grid, x, y) == r for x, y in wr):
                    assert (ax, ay) in got
        assert seen == allc


@pytest.mark.parametrize("grid,kx,ky", GRIDS)
def test_halo_lists(grid, kx, ky):
    """owners send exactly the line points in the receiver's read region."""
    nx, ny = kx * M, ky * M
    cfg = mfp.make_config(nx, ny, grid)
    R = grid[0] * grid[1]
    infos = [mfp.mfp_plan_query(cfg, r) for r in range(R)]
    for r in range(R):
        info = infos[r]
        peers = list(info.peers[: info.n_peers])
        # stencil neighbours only
        for s in peers:
            assert abs(s // grid[1] - r // grid[1]) <= 1 and abs(s % grid[1] - r % grid[1]) <= 1
        RX0, RX1, RY0, RY1 = brute_read_region(nx, ny, grid, r)
        assert (info.RX0, info.RX1, info.RY0, info.RY1) == (RX0, RX1, RY0, RY1)
        for i, s in enumerate(peers):
            recv = mfp.mfp_plan_halo(cfg, r, i, 1)
            j = list(infos[s].peers[: infos[s].n_peers]).index(r)
            sent = mfp.mfp_plan_halo(cfg, s, j, 0)
            assert np.array_equal(recv, sent)                       # same cells, same order
            want = set()
            for y in range(RY0, RY1 + 1):
                for x in range(RX0, RX1 + 1):
                    if brute_owner(nx, ny, grid, x, y) != s:
                        continue
                    if y % 16 == 0:
                        want.add((0, x, y))
                    if x % 16 == 0:
                        want.add((1, x, y))
            assert {tuple(v) for v in recv} == want
        # every halo point of r is covered by some peer
        covered = set()
        for i in range(len(peers)):
            covered |= {tuple(v) for v in mfp.mfp_plan_halo(cfg, r, i, 1)}
        for y in range(RY0, RY1 + 1, 16):
            for x in range(RX0, RX1 + 1):
                if brute_owner(nx, ny, grid, x, y) != r:
                    assert (0, x, y) in covered


@pytest.mark.parametrize("grid,kx,ky", GRIDS)
def test_phase0_overlap_split(grid, kx, ky):
    """North_star overlap: the phase-0 subdomains run before the previous
    exchange completes are exactly those that neither read (perimeter) nor
    write (centre lines) a received halo cell."""
    nx, ny = kx * M, ky * M
    cfg = mfp.make_config(nx, ny, grid)
    for r in range(grid[0] * grid[1]):
        info = mfp.mfp_plan_query(cfg, r)
        halo = set()
        for i in range(info.n_peers):
            for kind, x, y in mfp.mfp_plan_halo(cfg, r, i, 1):
                halo.add((int(x), int(y)))
        n = 0
        for ax, ay in mfp.mfp_plan_anchors(cfg, r, 0):
            cells = {tuple(p) for p in oracle.perimeter(ax, ay)} | {tuple(p) for p in oracle.writeset(ax, ay)[0]}
            n += not (cells & halo)
        assert info.phase0_interior == n
        if grid == (1, 1):
            assert n == info.phase_count[0]


def test_message_counts_stencil():
    """interior rank of a 3x3 grid talks to 8 neighbours, corner to 3."""
    cfg = mfp.make_config(6 * M, 6 * M, (3, 3))
    assert mfp.mfp_plan_query(cfg, 4).n_peers == 8
    assert mfp.mfp_plan_query(cfg, 0).n_peers == 3
    assert mfp.mfp_plan_query(cfg, 1).n_peers == 5
    assert sorted(mfp.mfp_plan_query(mfp.make_config(2 * M, 2 * M, (2, 2)), 0).peers[:3]) == [1, 2, 3]


def test_c5_decomposition_sizes():
    """4097^2 on 2x4: D1 per-rank compute set and message counts."""
    cfg = mfp.make_config(4096, 4096, (2, 4))
    infos = [mfp.mfp_plan_query(cfg, r) for r in range(8)]
    assert max(sum(i.phase_count) for i in infos) == 8320
    assert max(i.n_peers for i in infos) == 5
    assert sum(sum(i.phase_count) for i in infos) >= 65025
    assert sum(infos[0].final_count for _ in [0]) == (1024 // 32) * (2048 // 32)


def test_cost_model_library():
    for N, P, m, d, I, a, b, c, spp, ccomm in load_golden("cost_model.txt"):
        s, cc, cp = mfp.mfp_cost_model(N, P, m, d, I, a, b, c)
        assert (s, cc, cp) == (spp, ccomm, c * spp)
