"""Collect the boundary vectors the MFP iteration actually feeds its subsolver
(NEXT-1 training data): run the exact-subsolver MFP on GP-boundary domains and, at
a range of iteration counts (zero-interior start to near convergence), gather every
phase's perimeters with mfp_gather_phase.  Labels are not stored — they are the
exact harmonic extension H g, recomputed by the trainer.

    python tools/collect_mfp_boundaries.py --out gpurun_out/mfp_boundaries.npy
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2308_14258_b200 as mfp  # noqa: E402
from mfp_inputs import gp_boundary  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=2048)
    ap.add_argument("--seeds", type=int, default=4)
    ap.add_argument("--at", default="0,2,8,32,128,512,1024,2048")
    ap.add_argument("--per", type=int, default=4000, help="boundaries kept per (seed, iteration, phase)")
    ap.add_argument("--out", required=True)
    a = ap.parse_args()
    rng = np.random.default_rng(0)
    bank = []
    for k in range(a.seeds):
        cfg = mfp.make_config(a.n, a.n, precision=mfp.FP32, subsolver=mfp.EXACT_LAPLACE, check_every=1)
        m = mfp.Mfp(cfg, mfp.make_net(), None)
        g = torch.from_numpy(gp_boundary(a.n, a.n, 10 + k)).cuda()
        done = 0
        for t in [int(v) for v in a.at.split(",")]:
            if t > done:
                m.solve_device(g if done == 0 else None, t - done, 0.0, None)
                done = t
            elif t == 0:
                m.solve_device(g, 1, 0.0, None)     # init the lattice, then count from 1
                done = 1
            for ph in range(4):
                gb = m.gather_phase(ph).cpu().numpy()
                pick = rng.choice(len(gb), min(a.per, len(gb)), replace=False)
                bank.append(gb[pick])
        m.close()
        print(f"seed {k}: {sum(len(b) for b in bank)} boundaries", file=sys.stderr, flush=True)
    bank = np.concatenate(bank).astype(np.float32)
    np.save(a.out, bank)
    print(bank.shape, float(np.abs(bank).max()))


if __name__ == "__main__":
    main()
