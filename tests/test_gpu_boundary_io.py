"""GPU tests of the standalone Boundaries IO through the C ABI:
mfp_gather_phase (a1), mfp_scatter_phase (a6 + the update-norm reduction a8),
and the unfused phase gather -> mfp_sdnet_batch -> scatter against the fused one.

Gather and scatter are pure data movement, so the bar is bit-exact: the
perimeter values are the lattice values at the oracle's G1 perimeter points
(oracle.perimeter, P:23 / SPEC perimeter order), the written cells are exactly
the oracle's G3 write sets (oracle.writeset), and the update norm equals
max |new - old| over them computed here from the exported lattices.
"""
import numpy as np
import pytest

import oracle
from mfp_inputs import gp_boundary, random_weights
from tests._lattice import crossings_consistent, lattice_to_global

pytestmark = pytest.mark.gpu
M = 32


@pytest.fixture(scope="module")
def lib():
    import torch
    assert torch.cuda.is_available()
    import paper_2308_14258_b200 as mfp
    return mfp


def random_lattice(m, seed, rank=None):
    lat = m.lines(rank)
    rng = np.random.default_rng(seed)
    hl = rng.standard_normal(lat.hl.shape).astype(np.float32)
    vl = rng.standard_normal(lat.vl.shape).astype(np.float32)
    for i in range(hl.shape[0]):
        vl[:, 16 * i] = hl[i, ::16]          # crossing points consistent
    m.set_lines(hl, vl, rank)


def exact_ctx(lib, nx, ny, grid=(1, 1)):
    cfg = lib.make_config(nx, ny, grid, precision=lib.FP32, subsolver=lib.EXACT_LAPLACE, check_every=1)
    return lib.Mfp(cfg, lib.make_net(), None, rank=0 if grid == (1, 1) else lib.ALL_RANKS)


@pytest.mark.parametrize("nx,ny", [(64, 64), (5 * M, 3 * M), (1024, 992)])
@pytest.mark.parametrize("phase", [0, 1, 2, 3])
def test_gather_phase_bit_exact(lib, nx, ny, phase):
    m = exact_ctx(lib, nx, ny)
    random_lattice(m, 10 + phase)
    U = lattice_to_global(m.lines(), nx, ny)
    gb, anc = m.gather_phase(phase, want_anchors=True)
    gb = gb.cpu().numpy()
    ref_anc = oracle.anchors(nx, ny, phase)
    assert gb.shape == (len(ref_anc), 4 * M)
    # same subdomain set as the oracle's class (order: the device list)
    assert sorted(map(tuple, anc)) == sorted(map(tuple, ref_anc))
    want = np.stack([U[oracle.perimeter(ax, ay)[:, 1], oracle.perimeter(ax, ay)[:, 0]] for ax, ay in anc])
    assert np.array_equal(gb, want.astype(np.float32))


@pytest.mark.parametrize("phase", [0, 1, 2, 3])
def test_scatter_phase_bit_exact(lib, phase):
    import torch
    nx, ny = 7 * M, 4 * M
    m = exact_ctx(lib, nx, ny)
    random_lattice(m, 20 + phase)
    before = lattice_to_global(m.lines(), nx, ny, fill=0.0)
    B, anc = lib.mfp_gather_phase(m.ctx, 0, phase, want_anchors=True)
    rng = np.random.default_rng(phase)
    pred = rng.standard_normal((B, 2 * M - 3)).astype(np.float32)
    norm = m.scatter_phase(phase, torch.from_numpy(pred).cuda())
    after = lattice_to_global(m.lines(), nx, ny, fill=0.0)
    expect = before.copy()
    written = np.zeros(before.shape, bool)
    for k, (ax, ay) in enumerate(anc):
        wr, _ = oracle.writeset(ax, ay)
        assert not written[wr[:, 1], wr[:, 0]].any()        # disjoint within a phase
        written[wr[:, 1], wr[:, 0]] = True
        expect[wr[:, 1], wr[:, 0]] = pred[k]
    assert np.array_equal(after, expect)
    assert crossings_consistent(m.lines())
    want_norm = np.max(np.abs(after[written].astype(np.float32) - before[written].astype(np.float32)))
    assert np.float32(norm) == want_norm


def test_scatter_empty_and_nonfinite(lib):
    import torch
    m = exact_ctx(lib, 64, 64)
    lat = m.lines()
    m.set_lines(np.zeros_like(lat.hl), np.zeros_like(lat.vl))
    B, _ = lib.mfp_gather_phase(m.ctx, 0, 3)
    assert B == 1                                         # C1: class (1,1) has one subdomain
    pred = torch.zeros((1, 2 * M - 3), device="cuda")
    assert m.scatter_phase(3, pred) == 0.0                # zero lattice, zero predictions
    pred[0, 7] = float("nan")
    with pytest.raises(lib.MfpError) as e:
        m.scatter_phase(3, pred)
    assert e.value.status == 3
    with pytest.raises(lib.MfpError) as e:                # wrong B
        lib.mfp_scatter_phase(m.ctx, 0, 3, torch.zeros((2, 61), device="cuda"), 2)
    assert e.value.status == 1


@pytest.mark.parametrize("n", [4096, 8192])
def test_scatter_many_blocks_norm_rearm(lib, n):
    """Phases of 16,384 / 65,536 subdomains: every block of the one-wave grid
    (8 per SM) takes part, so the last-block reduction (a8) combines >= 1,000
    block maxima; repeated calls re-arm its ticket, and a non-finite call is
    followed by a finite one whose flag must be clear.  The norm must equal
    max |after - before| over the whole exported lattice (unwritten cells do
    not change), bit for bit."""
    import torch
    m = exact_ctx(lib, n, n)
    random_lattice(m, 5)
    rng = np.random.default_rng(n)
    for rep, phase in enumerate([0, 1, 0, 3, 2]):
        b = m.lines()
        hl0, vl0 = b.hl.copy(), b.vl.copy()
        B, _ = lib.mfp_gather_phase(m.ctx, 0, phase)
        pred = (rng.standard_normal((B, 2 * M - 3)) * (rep + 1)).astype(np.float32)
        if rep == 2:
            pred[B // 2, 30] = float("inf")
            with pytest.raises(lib.MfpError) as e:
                m.scatter_phase(phase, torch.from_numpy(pred).cuda())
            assert e.value.status == 3
            m.set_lines(hl0, vl0)   # the inf was written; later phases overlap its cells
            continue
        norm = m.scatter_phase(phase, torch.from_numpy(pred).cuda())
        a = m.lines()
        want = max(np.max(np.abs(a.hl - hl0)), np.max(np.abs(a.vl - vl0)))
        assert np.float32(norm) == np.float32(want)
        assert np.count_nonzero(a.hl != hl0) + np.count_nonzero(a.vl != vl0) <= B * (2 * M - 2)


def test_gather_distributed_rank_view(lib):
    """MFP_ALL_RANKS 2x2: each rank gathers from its own lattice copy (D1)."""
    nx = ny = 8 * M
    m = exact_ctx(lib, nx, ny, grid=(2, 2))
    g = gp_boundary(nx, ny, 2)
    m.solve(g, 3, 0.0, want_u=False)
    for r in range(4):
        U = lattice_to_global(m.lines(r), nx, ny)
        for phase in range(4):
            gb, anc = m.gather_phase(phase, rank=r, want_anchors=True)
            ref = lib.mfp_plan_anchors(m.cfg, r, phase)
            assert sorted(map(tuple, anc)) == sorted(map(tuple, ref))
            want = np.stack([U[oracle.perimeter(ax, ay)[:, 1], oracle.perimeter(ax, ay)[:, 0]] for ax, ay in anc])
            assert np.array_equal(gb.cpu().numpy(), want.astype(np.float32))


@pytest.mark.parametrize("precision", [0, 1])
def test_unfused_phase_matches_fused(lib, precision):
    """gather -> mfp_sdnet_batch -> scatter (the paper's three steps) writes
    the same lattice as the fused phase kernels, on the same state."""
    nx, ny = 8 * M, 6 * M
    w = random_weights(0)
    cfg = lib.make_config(nx, ny, precision=precision, subsolver=lib.SDNET, check_every=1)
    net = lib.make_net(gelu=1 if precision else 0)
    fused, unfused = lib.Mfp(cfg, net, w), lib.Mfp(cfg, net, w)
    g = gp_boundary(nx, ny, 3)
    fused.solve(g, 2, 0.0, want_u=False)
    unfused.solve(g, 2, 0.0, want_u=False)
    for phase in range(4):
        fused.step_phase(phase)
        gb = unfused.gather_phase(phase)
        pred = unfused.sdnet_batch(gb)
        unfused.scatter_phase(phase, pred)
        a = lattice_to_global(fused.lines(), nx, ny, fill=0.0)
        b = lattice_to_global(unfused.lines(), nx, ny, fill=0.0)
        scale = np.max(np.abs(a))
        assert np.max(np.abs(a - b)) <= 1e-6 * scale, phase
