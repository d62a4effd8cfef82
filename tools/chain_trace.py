"""Timeline of the CTA-pair chain kernel (build with MFP_NVCC_EXTRA=-DMFP_TRACE).

Runs one C5-sized phase batch through mfp_sdnet_batch and prints, for CTA 0,
per tile and layer: the four epilogue warps' arrival times, the issuer's a_full
completion and commit, and the warps' d_full wake-ups (clock64 cycles)."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from mfp_inputs import random_weights  # noqa: E402
from paper_2308_14258_b200 import mfp as lib  # noqa: E402

B = 16256
cfg = lib.make_config(4096, 4096, precision=1, subsolver=lib.SDNET)
net = lib.make_net(gelu=1)
w = random_weights(seed=0)
m = lib.Mfp(cfg, net, w)
gb = torch.randn(B, 128, device="cuda")
for _ in range(3):
    m.sdnet_batch(gb, 0)
torch.cuda.synchronize()
buf = np.zeros((2, 18, 32, 8, 4), np.uint64)
f = lib._lib.mfp_debug_trace
f.restype = ctypes.c_int
f.argtypes = [ctypes.c_void_p, ctypes.c_size_t]
assert f(buf.ctypes.data, buf.nbytes) > 0
np.save("gpurun_out/chain_trace.npy", buf)
T = buf[0].astype(np.int64)
t0 = T[T > 0].min()
T = np.where(T > 0, T - t0, -1)
for tile in range(12):
    slot = tile % 4
    warps = [4 * slot + q for q in range(4)]
    line = [f"tile {tile:2d} slot {slot}"]
    for l in range(4):
        arr = [T[w_, tile, l, 0] for w_ in warps]
        wake = [T[w_, tile, l, 1] for w_ in warps]
        iss = T[17, tile, l, 0], T[17, tile, l, 1]
        line.append(f"L{l}: arr {min(arr)}..{max(arr)} iss {iss[0]}/{iss[1]} wake {min(wake)}..{max(wake)}")
    print(" | ".join(line))
