"""Print the fitted-weights batch error of one precision (env MFP_GELU_POLY picks the GELU split)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402  (test/diagnostic tool)
from mfp_inputs import random_boundaries  # noqa: E402
from paper_2308_14258_b200 import mfp as lib  # noqa: E402

prec = int(sys.argv[1])
w = np.load(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "weights", "sdnet_fit_d128.npy"))
cfg = lib.make_config(128, 128, precision=prec, subsolver=lib.SDNET, check_every=1)
m = lib.Mfp(cfg, lib.make_net(gelu=1 if prec else 0), w)
gb = random_boundaries(500, seed=13)
out = m.sdnet_batch(torch.from_numpy(gb).cuda(), 0).cpu().numpy().astype(np.float64)
ref = oracle.sdnet_forward(w.astype(np.float64), gb.astype(np.float64), oracle.writeset(0, 0)[1])
d = np.abs(out - ref) / np.abs(ref).max()
print(f"precision {prec} poly {os.environ.get('MFP_GELU_POLY', 'default')}: max {d.max():.3e} mean {d.mean():.3e}")
