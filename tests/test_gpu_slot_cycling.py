"""Tile-slot protocols under many rounds: the tensor-core chains on a persistent grid
capped to 2 CTA pairs (MFP_MAX_PAIRS=2, read once per process, so the capped run is
a subprocess) against the same batch on the full grid, bit for bit.

With 2 pairs every tile slot of a 16,384-subdomain batch processes ~250 tiles, so the
per-slot mbarrier phases (operands written, MMA done, z staged), the two z staging
buffers (DESIGN.md §6 round 2 session 3) and, at d = 256, the TMA weight ring cycle
through hundreds of rounds; on the full grid each slot sees ~13.  A row's arithmetic
does not depend on which pair or slot computes it, so any protocol slip (a buffer
overwritten early, a stale phase, z of the wrong tile) shows up as a mismatch.
Covers k_chain_tc2 (bf16, fp16), k_chain_tc2w (d = 256) and k_chain_tc2s (FP16X),
centre-line and interior query sets.
"""
import os
import subprocess
import sys

import numpy as np
import pytest

from mfp_inputs import random_boundaries, random_weights

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CASES = [  # (d, precision, gelu, query set, B)
    (128, 1, 1, 0, 16384),
    (128, 2, 1, 1, 1200),
    (256, 1, 1, 0, 8192),
    (128, 3, 2, 0, 8192),
]

SCRIPT = r"""
import sys, numpy as np, torch
sys.path.insert(0, {root!r})
import paper_2308_14258_b200 as lib
from mfp_inputs import random_boundaries, random_weights
d, prec, gelu, qs, B = {case!r}
cfg = lib.make_config(4096, 4096, precision=prec, subsolver=lib.SDNET, check_every=16)
m = lib.Mfp(cfg, lib.make_net(d=d, gelu=gelu), random_weights(3, d=d))
gb = torch.from_numpy(random_boundaries(B, seed=41)).cuda()
np.save({out!r}, m.sdnet_batch(gb, qs).cpu().numpy())
m.close()
"""


def run_batch(case, out, max_pairs):
    env = dict(os.environ)
    env.pop("MFP_MAX_PAIRS", None)
    if max_pairs:
        env["MFP_MAX_PAIRS"] = str(max_pairs)
    src = SCRIPT.format(root=ROOT, case=case, out=out)
    r = subprocess.run([sys.executable, "-c", src], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    return np.load(out)


@pytest.mark.parametrize("case", CASES, ids=lambda c: f"d{c[0]}-p{c[1]}-q{c[3]}-B{c[4]}")
def test_capped_grid_bit_identical(case, tmp_path):
    full = run_batch(case, str(tmp_path / "full.npy"), 0)
    capped = run_batch(case, str(tmp_path / "capped.npy"), 2)
    assert np.isfinite(full).all()
    assert np.array_equal(full, capped)
