"""Exact-subsolver MFP per-iteration device time (graph-replayed), C5 and a rank share.
Usage: python tools/exact_probe.py [nx ny] [iters]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2308_14258_b200 as mfp  # noqa: E402
from mfp_inputs import gp_boundary  # noqa: E402

nx = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
ny = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
K = int(sys.argv[3]) if len(sys.argv) > 3 else 512
m = mfp.Mfp(mfp.make_config(nx, ny, subsolver=mfp.EXACT_LAPLACE, check_every=16), mfp.make_net(), None)
g = torch.from_numpy(gp_boundary(nx, ny, 0)).cuda()
m.solve_device(g, 64, 0.0, None)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(m.stream)
m.solve_device(None, K, 0.0, None)
e1.record(m.stream)
e1.synchronize()
print(f"exact {nx}x{ny}: {e0.elapsed_time(e1) * 1e3 / K:.2f} us per iteration (graph-replayed, incl. final phase / {K})",
      flush=True)
m.close()
