"""Iterations to the paper's stop rule, MAE < 0.05 against the discrete solution
(Table strongScalingIter: 3200 / 3250 / 3250 / 3300 iterations at 1 / 2 /
4 / 8 A30s on a 32 x 32-unit = 2049^2 domain), for the processor grids the bench
scales over (1x1, 1x2, 2x2, 2x4), emulated on ONE GPU with MFP_ALL_RANKS (same
plans, halo exchange by device copies: the convergence behaviour of D1 is the
same as with NCCL).  Subsolvers: exact discrete Laplace (fp32) and the fitted
SDNet (weights/sdnet_fit_d128.npy) in fp16 and bf16.

    python tools/iters_to_mae.py [--n 2048] [--chunk 50] [--max 20000] > gpurun_out/iters_to_mae.json
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2308_14258_b200 as mfp  # noqa: E402
from _refsolve import dst_laplace  # noqa: E402
from mfp_inputs import gp_boundary  # noqa: E402

GRIDS = [(1, 1), (1, 2), (2, 2), (2, 4)]


def run(n, grid, subsolver, precision, w, g, ref_dev, chunk, max_iters, target, s_ex=1):
    cfg = mfp.make_config(n, n, grid, precision=precision, subsolver=subsolver, check_every=chunk)
    rank = 0 if grid == (1, 1) else mfp.ALL_RANKS
    m = mfp.Mfp(cfg, mfp.make_net(gelu=1 if precision != mfp.FP32 else 0), w, rank=rank)
    mfp.mfp_set_exchange_every(m.ctx, s_ex)
    u = torch.empty((n + 1, n + 1), dtype=torch.float32, device="cuda")
    g_dev = torch.from_numpy(g.astype(np.float32)).cuda()
    done, mae, hist = 0, float("nan"), []
    t0 = time.perf_counter()
    g_arg = g_dev
    while done < max_iters:
        m.solve_device(g_arg, chunk, 0.0, u)      # chunk iterations + final phase (the field)
        g_arg = None                              # resume from the lattice
        done += chunk
        torch.cuda.synchronize()
        mae = float((u - ref_dev).abs().mean())
        hist.append((done, mae))
        if mae < target:
            break
    m.close()
    return {"grid": f"{grid[0]}x{grid[1]}", "exchange_every": s_ex, "iterations": done if mae < target else None, "mae": mae,
            "reached": mae < target, "wall_s": time.perf_counter() - t0,
            "mae_history": hist[:: max(1, len(hist) // 20)]}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=2048)
    ap.add_argument("--chunk", type=int, default=50)
    ap.add_argument("--max", type=int, default=20000)
    ap.add_argument("--target", type=float, default=0.05)
    ap.add_argument("--weights", default=os.path.join(ROOT, "weights", "sdnet_fit_d128.npy"))
    ap.add_argument("--only", default="", help="comma list of subsolver names to run (default all)")
    ap.add_argument("--grids", default="1x1,1x2,2x2,2x4")
    ap.add_argument("--exchange-every", default="1", help="comma list of s (NEXT-4); each must divide --chunk")
    a = ap.parse_args()
    g = gp_boundary(a.n, a.n, 0)
    ref = dst_laplace(a.n, a.n, g.astype(np.float64))
    ref_dev = torch.from_numpy(ref.astype(np.float32)).cuda()
    wfit = np.load(a.weights)
    grids = [tuple(int(v) for v in x.split("x")) for x in a.grids.split(",")]
    out = []
    for name, sub, prec, w in [("exact fp32", mfp.EXACT_LAPLACE, mfp.FP32, None),
                               ("sdnet W-fit fp16", mfp.SDNET, mfp.FP16, wfit),
                               ("sdnet W-fit bf16", mfp.SDNET, mfp.BF16, wfit)]:
        if a.only and name not in a.only.split(","):
            continue
        for grid in grids:
            for s_ex in [int(v) for v in a.exchange_every.split(",")]:
                if s_ex > 1 and grid == (1, 1):
                    continue
                r = run(a.n, grid, sub, prec, w, g, ref_dev, a.chunk, a.max, a.target, s_ex)
                r["subsolver"] = name
                print(json.dumps({k: v for k, v in r.items() if k != "mae_history"}), file=sys.stderr, flush=True)
                out.append(r)
    print(json.dumps({"experiment": "iterations to MAE < %g vs the discrete solution (P:179)" % a.target,
                      "domain": f"{a.n + 1}^2 (GP boundary k=0)", "rows": out}))


if __name__ == "__main__":
    main()
