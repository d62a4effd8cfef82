"""Chain roofline probe at d = 128 and d = 256 (GPU): C5 MFP, bf16 (or argv[1]
precision), mfp_profile_iterations -> chain ms per launch -> hidden-GEMM TFLOP/s
(algorithmic: rows x n_hidden x 2 d^2 per launch) and its fraction of the
measured sustained bf16 peak.  Usage: python tools/d_probe.py [precision] [iters]"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2308_14258_b200 as mfp  # noqa: E402
from mfp_inputs import gp_boundary, random_weights  # noqa: E402

prec = int(sys.argv[1]) if len(sys.argv) > 1 else 1
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 4
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pk = json.load(open(os.path.join(root, "MEASURED_PEAKS.json"))) if os.path.exists(
    os.path.join(root, "MEASURED_PEAKS.json")) else {}
peak = pk.get("bf16_tflops_sustained", 1400.0)
nx = ny = 4096
g = gp_boundary(nx, ny, 0)
for d in ((128,) if prec == 3 else (128, 256)):
    w = random_weights(0, d=d)
    m = mfp.Mfp(mfp.make_config(nx, ny, precision=prec, subsolver=mfp.SDNET, check_every=16),
                mfp.make_net(d=d, gelu=2 if prec == 3 else 1), w)
    m.solve(g, 2, 0.0)
    m.profile(2)
    p = m.profile(iters)
    chain_ms = p.chain_ms_total / max(p.chain_launches, 1)
    flop = p.chain_rows / max(p.chain_launches, 1) * 3 * 2 * d * d
    tf = flop / (chain_ms / 1e3) / 1e12
    print(json.dumps({"d": d, "precision": prec, "chain_ms_per_launch": chain_ms, "tflops": tf,
                      "frac_sustained": tf / peak, "ms_per_iter": p.ms_per_iter,
                      "gather_embed_per_phase_ms": p.ms_gather_embed, "chain_per_phase_ms": p.ms_chain,
                      "predictions_per_s": 65025 / (p.ms_per_iter / 1e3)}), flush=True)
    m.close()
