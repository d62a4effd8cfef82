"""Per-iteration device time of the MFP on one rank's share of the C5 domain for
each processor grid of the scaling runs (1x1: 4096^2, 1x2: 2048x4096, 2x2: 2048^2,
2x4: 1024x2048 points), run as a single-rank problem on one GPU: the compute part
of strong-scaling efficiency (no exchange, no D1 redundancy) — what bounds the
8-GPU efficiency once the per-rank batch is small.

    python tools/rank_share.py
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2308_14258_b200 as mfp  # noqa: E402
from mfp_inputs import gp_boundary, random_weights  # noqa: E402

w = random_weights(0)
rows = []
base = None
for n_gpu, (nx, ny) in [(1, (4096, 4096)), (2, (2048, 4096)), (4, (2048, 2048)), (8, (1024, 2048))]:
    cfg = mfp.make_config(nx, ny, precision=mfp.BF16, subsolver=mfp.SDNET, check_every=16)
    m = mfp.Mfp(cfg, mfp.make_net(gelu=1), w)
    g = torch.from_numpy(gp_boundary(nx, ny, 0)).cuda()
    m.solve_device(g, 32, 0.0, None)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(m.stream)
    m.solve_device(None, 128, 0.0, None)
    e1.record(m.stream)
    e1.synchronize()
    ms = e0.elapsed_time(e1) / 128
    if base is None:
        base = ms
    prof = m.profile(8)
    rows.append({"gpus": n_gpu, "share": f"{nx}x{ny}", "ms_per_iter": ms, "ideal_ms": base / n_gpu,
                 "compute_efficiency": base / n_gpu / ms, "chain_ms_per_phase": prof.ms_chain,
                 "embed_ms_per_phase_profiled": prof.ms_gather_embed})
    print(json.dumps(rows[-1]), file=sys.stderr, flush=True)
    m.close()
print(json.dumps({"experiment": "per-rank share of C5, compute only", "rows": rows}))
