"""One rank's share of the C5 domain as a single-rank MFP (bf16, d = MFP_PROBE_D, default 128): K
iterations after a warm-up, for ncu launch lists of the small-batch regime of
strong scaling.  Usage: python tools/share_probe.py NX NY [K]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2308_14258_b200 as mfp  # noqa: E402
from mfp_inputs import gp_boundary, random_weights  # noqa: E402

nx, ny = int(sys.argv[1]), int(sys.argv[2])
K = int(sys.argv[3]) if len(sys.argv) > 3 else 4
d = int(os.environ.get("MFP_PROBE_D", "128"))
m = mfp.Mfp(mfp.make_config(nx, ny, precision=mfp.BF16, subsolver=mfp.SDNET, check_every=16),
            mfp.make_net(d=d, gelu=1), random_weights(0, d=d))
g = torch.from_numpy(gp_boundary(nx, ny, 0)).cuda()
m.solve_device(g, 64, 0.0, None)   # captures the c-block graphs
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(m.stream)
m.solve_device(None, 256, 0.0, None)
e1.record(m.stream)
e1.synchronize()
print(f"d={d} {nx}x{ny}: {e0.elapsed_time(e1) / 256:.4f} ms per iteration (graph-replayed, incl. final phase / 256)", flush=True)
m.solve_device(None, K, 0.0, None)
torch.cuda.synchronize()
