"""The exact subsolver at full size on ONE rank: the path the bench's time-to-converge
leg runs (C5 = 4097^2, 16,256 subdomains per phase, so `k_exact_phase` takes 7
subdomains per warp on 146 blocks and is launched with PDL, DESIGN.md §8 session 3).

* line lattice and final field after K = 3 iterations vs the fp64 oracle (Algorithm 2,
  P:43-44, exact discrete-Laplace subsolver), fp32 bar 1e-5;
* bit-identical to the same solve with 8 subdomains per warp (MFP_EXACT_SUB=8, read
  once per process, so that run is a subprocess) and with PDL off (MFP_NO_PDL=1): the
  per-output FMA order does not depend on the grouping and the early launch only
  moves the H_c^T load.
"""
import os
import subprocess
import sys

import numpy as np
import pytest

import oracle
from mfp_inputs import gp_boundary
from tests._lattice import lattice_to_global, line_mask

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
N, K = 4096, 3

SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, {root!r})
import paper_2308_14258_b200 as lib
from mfp_inputs import gp_boundary
cfg = lib.make_config({n}, {n}, subsolver=lib.EXACT_LAPLACE, check_every=16)
m = lib.Mfp(cfg, lib.make_net(), None)
u, rep = m.solve(gp_boundary({n}, {n}, 0), {k}, 0.0)
np.save({out!r}, u)
m.close()
"""


def solve_in_subprocess(out, env_extra):
    env = dict(os.environ)
    for k in ("MFP_EXACT_SUB", "MFP_NO_PDL"):
        env.pop(k, None)
    env.update(env_extra)
    r = subprocess.run([sys.executable, "-c", SCRIPT.format(root=ROOT, n=N, k=K, out=out)], env=env,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    return np.load(out)


@pytest.fixture(scope="module")
def lib():
    import torch
    assert torch.cuda.is_available()
    import paper_2308_14258_b200 as mfp
    return mfp


def test_exact_c5_single_rank_parity(lib):
    g = gp_boundary(N, N, 0)
    m = lib.Mfp(lib.make_config(N, N, subsolver=lib.EXACT_LAPLACE, check_every=16), lib.make_net(), None)
    u, rep = m.solve(g, K, 0.0)
    assert rep.iterations == K
    ref = oracle.mfp_run(oracle.MfpConfig(N, N, subsolver="exact"), g.astype(np.float64), K)
    L = lattice_to_global(m.lines(), N, N)
    lm = line_mask(N, N)
    scale = np.max(np.abs(ref.u))
    assert np.max(np.abs(L[lm] - ref.lines[lm])) <= 1e-5 * scale
    assert np.max(np.abs(u - ref.u)) <= 1e-5 * scale
    m.close()


def test_exact_c5_grouping_and_pdl_bit_identical(tmp_path):
    base = solve_in_subprocess(str(tmp_path / "base.npy"), {})
    sub8 = solve_in_subprocess(str(tmp_path / "sub8.npy"), {"MFP_EXACT_SUB": "8"})
    nopdl = solve_in_subprocess(str(tmp_path / "nopdl.npy"), {"MFP_NO_PDL": "1"})
    assert np.array_equal(base, sub8)
    assert np.array_equal(base, nopdl)
