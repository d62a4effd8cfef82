"""Diagnostic (GPU): where do the final-phase interior predictions differ from the
oracle?  Solves K iterations + the final phase on the GPU, then re-predicts the
worst subdomains' 961 interior points from the GPU's OWN line lattice with the
fp64 oracle network (oracle.predict_from_field), which separates final-phase
error from lattice error.  Usage: python tools/diag_final.py N precision K"""
import json
import sys

import numpy as np

sys.path.insert(0, ".")
import oracle  # noqa: E402
import paper_2308_14258_b200 as mfp  # noqa: E402
from mfp_inputs import gp_boundary, random_weights  # noqa: E402
from tests._lattice import lattice_to_global, line_mask  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
prec = int(sys.argv[2]) if len(sys.argv) > 2 else 1
K = int(sys.argv[3]) if len(sys.argv) > 3 else 3
g = gp_boundary(n, n, 0)
w = random_weights(0)
cfg = mfp.make_config(n, n, (1, 1), precision=prec, subsolver=mfp.SDNET, check_every=K)
m = mfp.Mfp(cfg, mfp.make_net(gelu=0 if prec == mfp.FP32 else 1), w)
u, rep = m.solve(g, K, 0.0)
L = lattice_to_global(m.lines(), n, n)
lm = line_mask(n, n)
Lf = np.where(lm, L, 0.0)
ref = oracle.mfp_run(oracle.MfpConfig(n, n), g.astype(np.float64), K, params=w.astype(np.float64))
inner = ~lm
d = np.abs(u.astype(np.float64) - ref.u)
out = {"n": n, "precision": prec, "K": K,
       "lines_abs": float(np.max(d[lm])), "inner_abs": float(np.max(d[inner])),
       "max_ref_inner": float(np.max(np.abs(ref.u[inner]))), "max_ref": float(np.max(np.abs(ref.u))),
       "inner_abs_p99": float(np.percentile(d[inner], 99)), "inner_abs_p50": float(np.percentile(d[inner], 50))}
# per subdomain (class 00 anchors, 32 x 32 blocks) max error
Kx = n // 32
blk = d[:n, :n].reshape(Kx, 32, Kx, 32).max(axis=(1, 3))
wi = np.argsort(blk.ravel())[::-1][:8]
out["worst_blocks"] = [[int(i // Kx), int(i % Kx), float(blk.ravel()[i])] for i in wi]
out["blocks_over_1e-3"] = int(np.sum(blk > 1e-3))
# position inside block of max error pattern
pos = d[:n, :n].reshape(Kx, 32, Kx, 32).max(axis=(0, 2))
out["pos_max_err_row"] = [float(x) for x in pos.max(axis=1)]
out["pos_max_err_col"] = [float(x) for x in pos.max(axis=0)]
# re-predict worst blocks from the GPU lattice in fp64
anc = np.array([[32 * (i % Kx), 32 * (i // Kx)] for i in wi], np.int32)
P = oracle.predict_from_field(oracle.MfpConfig(n, n), Lf, anc, 1, params=w.astype(np.float64))
rows = []
for k, (ax, ay) in enumerate(anc):
    gpu = u[ay + 1:ay + 32, ax + 1:ax + 32].astype(np.float64).ravel()
    rf = ref.u[ay + 1:ay + 32, ax + 1:ax + 32].ravel()
    rows.append({"anchor": [int(ax), int(ay)], "gpu_vs_refit": float(np.max(np.abs(gpu - P[k]))),
                 "refit_vs_oracle": float(np.max(np.abs(P[k] - rf))),
                 "gpu_vs_oracle": float(np.max(np.abs(gpu - rf)))})
out["repredict"] = rows
print(json.dumps(out))
