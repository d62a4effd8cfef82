"""E6 (Fig. batchedVunbatched): time per MFP iteration with every phase's
subdomains predicted as ONE batch (the library's solve) vs one SDNet call per
subdomain (the paper's original unbatched algorithm), for domains of 1x2 to
16x16 units (64 points per unit, m = 32).

The unbatched arm runs each phase through the library's standalone steps:
mfp_gather_phase (all perimeters), then mfp_sdnet_batch with B = 1 for every
subdomain in turn, then mfp_scatter_phase — the same arithmetic, one launch
pair per subdomain.  Device time with CUDA events; W-rand weights, bf16.

    python tools/e6_batching.py [--iters 20] > gpurun_out/e6.json
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2308_14258_b200 as mfp  # noqa: E402
from mfp_inputs import gp_boundary, random_weights  # noqa: E402

SIZES = [(1, 2), (2, 2), (2, 4), (4, 4), (4, 8), (8, 8), (8, 16), (16, 16)]   # units (x, y)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--unbatched-iters", type=int, default=2)
    a = ap.parse_args()
    w = random_weights(0)
    rows = []
    for ux, uy in SIZES:
        nx, ny = 64 * ux, 64 * uy
        cfg = mfp.make_config(nx, ny, precision=mfp.BF16, subsolver=mfp.SDNET, check_every=16)
        m = mfp.Mfp(cfg, mfp.make_net(gelu=1), w)
        g = torch.from_numpy(gp_boundary(nx, ny, 0)).cuda()
        m.solve_device(g, 1, 0.0, None)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        # batched: the library's iteration (graphs, fused kernels)
        torch.cuda.synchronize()
        e0.record(m.stream)
        m.solve_device(None, a.iters, 0.0, None)
        e1.record(m.stream)
        e1.synchronize()
        t_b = e0.elapsed_time(e1) / a.iters
        # unbatched: one SDNet launch pair per subdomain
        counts = [mfp.mfp_gather_phase(m.ctx, 0, ph)[0] for ph in range(4)]
        gbs = [torch.empty((max(c, 1), 128), device="cuda") for c in counts]
        preds = [torch.empty((max(c, 1), 61), device="cuda") for c in counts]
        torch.cuda.synchronize()
        e0.record(m.stream)
        for _ in range(a.unbatched_iters):
            for ph in range(4):
                mfp.mfp_gather_phase(m.ctx, 0, ph, gbs[ph], counts[ph])
                for i in range(counts[ph]):
                    mfp.mfp_sdnet_batch(m.ctx, gbs[ph][i:i + 1], 1, mfp.QUERY_CENTRE, preds[ph][i:i + 1],
                                        m.stream.cuda_stream)
                mfp.mfp_scatter_phase(m.ctx, 0, ph, preds[ph], counts[ph], want_norm=False)
        e1.record(m.stream)
        e1.synchronize()
        t_u = e0.elapsed_time(e1) / a.unbatched_iters
        n = sum(counts)
        rows.append({"units": f"{ux}x{uy}", "points": f"{nx}x{ny}", "subdomains_per_iter": n,
                     "batched_ms_per_iter": t_b, "unbatched_ms_per_iter": t_u, "speedup": t_u / t_b})
        print(json.dumps(rows[-1]), file=sys.stderr, flush=True)
        m.close()
    print(json.dumps({"experiment": "E6 batched vs unbatched (P:167)", "precision": "bf16", "rows": rows}))


if __name__ == "__main__":
    main()
