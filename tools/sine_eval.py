"""Fig. gfnet-eval analog: MAE of the converged MFP on the paper's evaluation
boundary g(x) = sin(2 pi x), for domains of 1x2 to 16x16 units (64 points per unit),
against the grid's separable closed form (tests/test_oracle_exact.py), with the
fitted SDNet (weights/sdnet_fit_d128_mfp.npy, bf16) and the round-1 W-fit (fp16).

    python tools/sine_eval.py > gpurun_out/sine_eval.json
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import paper_2308_14258_b200 as mfp  # noqa: E402
from mfp_inputs import sine_boundary  # noqa: E402
from tests.test_oracle_exact import sine_discrete_solution  # noqa: E402

H = 1.0 / 64.0
rows = []
for wname, prec in (("sdnet_fit_d128_mfp.npy", mfp.BF16), ("sdnet_fit_d128.npy", mfp.FP16)):
    w = np.load(os.path.join(ROOT, "weights", wname))
    for ux, uy in ((1, 2), (2, 2), (4, 4), (8, 8), (16, 16)):
        nx, ny = 64 * ux, 64 * uy
        cfg = mfp.make_config(nx, ny, precision=prec, subsolver=mfp.SDNET, check_every=16)
        m = mfp.Mfp(cfg, mfp.make_net(gelu=1), w)
        u, rep = m.solve(sine_boundary(nx, ny, H).astype(np.float32), 20000, 1e-5)
        mae = float(np.mean(np.abs(u - sine_discrete_solution(nx, ny, H))))
        rows.append({"weights": wname, "precision": "bf16" if prec == mfp.BF16 else "fp16", "units": f"{ux}x{uy}",
                     "iterations": rep.iterations, "converged": bool(rep.converged), "mae": mae})
        print(json.dumps(rows[-1]), file=sys.stderr, flush=True)
        m.close()
print(json.dumps({"experiment": "Fig. gfnet-eval analog: sin(2 pi x) boundary, MAE at convergence", "rows": rows}))
