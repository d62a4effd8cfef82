"""Pins for the oracle's geometry (readings G1-G3).

Checked against SPEC's worked examples (tests/golden/, each cited) and brute
force over the lattice — never against the oracle itself.
"""
import itertools

import numpy as np
import pytest

import oracle
from tests.conftest import load_golden  # noqa: E402

M = 32


def test_perimeter_spec_example():
    # 3-point sides (m = 2 intervals under G1) walked CCW from the anchor
    want = load_golden("perimeter_m2.txt").astype(int)
    got = oracle.perimeter(0, 0, m=2)
    assert np.array_equal(got, want)
    # translation invariance
    assert np.array_equal(oracle.perimeter(16, 16, m=2), want + 16)


def test_perimeter_is_bijection_onto_square_boundary():
    p = oracle.perimeter(48, 16)
    assert len(p) == 4 * M
    pts = {tuple(x) for x in p}
    assert len(pts) == 4 * M                     # each corner exactly once
    ring = {(48 + i, 16 + j) for i in range(M + 1) for j in range(M + 1)
            if i in (0, M) or j in (0, M)}
    assert pts == ring
    # consecutive points are grid neighbours (a closed counter-clockwise walk)
    d = np.abs(np.diff(np.vstack([p, p[:1]]), axis=0)).sum(1)
    assert np.all(d == 1)
    # counter-clockwise: positive signed area (shoelace)
    x, y = p[:, 0].astype(float), p[:, 1].astype(float)
    assert 0.5 * np.sum(x * np.roll(y, -1) - np.roll(x, -1) * y) == M * M


def test_anchor_examples_spec():
    for npts, c0, c1, c2, c3 in load_golden("anchor_counts.txt").astype(int):
        n = npts - 1
        got = [len(oracle.anchors(n, n, c)) for c in range(4)]
        assert got == [c0, c1, c2, c3], (npts, got)
    rows = load_golden("anchors_65.txt").astype(int)
    for cls in (0, 3):
        want = sorted((x, y) for c, x, y in rows if c == cls)
        got = sorted(map(tuple, oracle.anchors(64, 64, cls)))
        assert got == want


@pytest.mark.parametrize("kx,ky", [(2, 2), (4, 4), (3, 5), (16, 16)])
def test_prediction_count_per_iteration(kx, ky):
    total = sum(len(oracle.anchors(kx * M, ky * M, c)) for c in range(4))
    assert total == (2 * kx - 1) * (2 * ky - 1)


def _brute_sets(nx, ny):
    """Brute force over the lattice: per class, per subdomain, perimeter & writes."""
    out = []
    for cls in range(4):
        subs = []
        for ax, ay in oracle.anchors(nx, ny, cls):
            per = {tuple(p) for p in oracle.perimeter(ax, ay)}
            wr, _ = oracle.writeset(ax, ay)
            subs.append((per, {tuple(p) for p in wr}))
        out.append(subs)
    return out


@pytest.mark.parametrize("kx,ky", [(2, 2), (3, 4)])
def test_classes_are_batchable(kx, ky):
    """subdomains of one class do not overlap -> reads and writes of a
    class are disjoint, so one batch == one-at-a-time."""
    nx, ny = kx * M, ky * M
    for subs in _brute_sets(nx, ny):
        writes = [w for _, w in subs]
        allw = set().union(*writes) if writes else set()
        assert sum(len(w) for w in writes) == len(allw)            # writes disjoint
        allr = set().union(*[p for p, _ in subs]) if subs else set()
        assert not (allw & allr)                                   # no write is read


def test_write_coverage_and_boundary_immutability():
    nx, ny = 4 * M, 3 * M
    count = {}
    for subs in _brute_sets(nx, ny):
        for _, w in subs:
            for p in w:
                count[p] = count.get(p, 0) + 1
    h = M // 2
    for (x, y), c in count.items():
        assert 0 < x < nx and 0 < y < ny                           # ∂Ω never written
        assert x % h == 0 or y % h == 0                            # only line points
    for x in range(1, nx):
        for y in range(1, ny):
            if x % h and y % h:
                continue
            c = count.get((x, y), 0)
            if x % h == 0 and y % h == 0:
                assert c == 1, (x, y)                               # crossings once
            elif (x % h == 0 and (y < h or y > ny - h)) or (y % h == 0 and (x < h or x > nx - h)):
                assert c == 1, (x, y)                               # near ∂Ω once
            else:
                assert c == 2, (x, y)


def test_centre_lines_are_boundaries_of_other_classes():
    """P:43 "the center lines of one subdomain are the boundary of another"."""
    nx = ny = 4 * M
    sets = _brute_sets(nx, ny)
    for cls in range(4):
        writes = set().union(*[w for _, w in sets[cls]])
        others = set().union(*[p for c2 in range(4) if c2 != cls for p, _ in sets[c2]])
        # every written point except those next to ∂Ω is read by another class
        inner = {p for p in writes if M // 2 < p[0] < nx - M // 2 and M // 2 < p[1] < ny - M // 2}
        assert inner <= others


def test_writeset_queries_normalised():
    pts, q = oracle.writeset(32, 64)
    assert len(pts) == 2 * M - 3
    local = (pts - np.array([32, 64])) / M
    assert np.allclose(local, q)
    assert np.all((q > 0) & (q < 1))
    assert len({tuple(p) for p in pts}) == len(pts)


def test_interior_queries_grid():
    q = oracle.interior_queries()
    assert q.shape == ((M - 1) ** 2, 2)
    ij = np.rint(q * M).astype(int)
    assert {tuple(x) for x in ij} == set(itertools.product(range(1, M), range(1, M)))
    assert np.array_equal(ij[:M - 1, 0], np.arange(1, M))      # i fastest


def test_cost_model_substitution():
    """§4.3 P:55-60 with SPEC S:626-628 substitutions."""
    for N, P, m, d, I, a, b, c, spp, ccomm in load_golden("cost_model.txt"):
        s, cc, cp = oracle.cost_model(N, P, m, d, I, a, b, c)
        assert s == spp and cc == ccomm and cp == c * spp
    s1, _, cp1 = oracle.cost_model(4096, 4, 32, 2, 1, 1, 1, 3.0)
    s2, _, cp2 = oracle.cost_model(4096, 8, 32, 2, 1, 1, 1, 3.0)
    assert cp2 == cp1 / 2
