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

B = int(os.environ.get("MFP_TRACE_B", "16256"))   # default: one C5 phase
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
acts, rts, iss, exe, comp, fin, l0, l0s, tails = [], [], [], [], [], [], [], [], []
L = 3   # layers with an MMA (the split layer runs on the CUDA cores)
for tile in range(4, 28):
    slot = tile % 4
    ws = [4 * slot + q for q in range(4)]
    g = lambda l, ev, f: f(T[w, tile, l, ev] for w in ws)
    for l in range(L):
        arr, wake = g(l, 0, max), g(l, 1, max)
        if arr <= 0 or wake <= 0:
            continue
        rts.append(wake - arr)
        iw, ic = T[17, tile, l, 0], T[17, tile, l, 1]
        if iw > 0:
            iss.append(iw - arr)
            exe.append(ic - iw)
        if l < L - 1:
            a2 = g(l + 1, 0, max)
            e2 = g(l, 2, max)
            if a2 > 0 and e2 > 0:
                acts.append(a2 - g(l, 1, min))
                comp.append(e2 - g(l, 1, min))
                fin.append(a2 - e2)
    st, ns, ea = g(0, 3, min), g(2, 3, max), g(1, 3, max)
    if st > 0 and ns > 0 and ea > 0:
        l0s.append(ns - st)
        l0.append(ea - ns)
    if tile + 4 < 32:
        nst = min(T[w, tile + 4, 0, 3] for w in ws)
        if nst > 0:
            tails.append(nst - g(L - 1, 1, max))
mean_ = lambda v: float(np.mean(v)) if v else -1
print(f"layers {L}: act phase {mean_(acts):.0f} (compute {mean_(comp):.0f}, fence+arrive {mean_(fin):.0f}) | round trip {mean_(rts):.0f} "
      f"(issuer wait after CTA0 arrivals {mean_(iss):.0f}, issue->commit {mean_(exe):.0f}) | L0: tile start->z sync {mean_(l0s):.0f}, "
      f"sync->compute end {mean_(l0):.0f} | head+tail {mean_(tails):.0f}")

# per-CTA globaltimer stamps of one more launch: prologue, per-CTA work span, tail
g = lib._lib.mfp_debug_cta_times
g.restype = ctypes.c_int
g.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int]
ct = np.zeros((256, 4), np.uint64)
g(ct.ctypes.data, ct.nbytes, 1)
m.sdnet_batch(gb, 0)
torch.cuda.synchronize()
assert g(ct.ctypes.data, ct.nbytes, 0) > 0
c = ct[:148].astype(np.int64)
t0 = c[:, 0].min()
ent, pro, last, ex = (c[:, 0] - t0) / 1e3, (c[:, 1] - t0) / 1e3, (c[:, 2] - t0) / 1e3, (c[:, 3] - t0) / 1e3
q = lambda v: " ".join(f"{x:.1f}" for x in np.percentile(v, [0, 50, 100]))
print(f"per-CTA us from the first entry (min/median/max): entry {q(ent)} | past prologue {q(pro)} | last head done {q(last)} | exit {q(ex)}")

cc = np.zeros((256, 4), np.uint64)
assert g(cc.ctypes.data, cc.nbytes, 2) > 0
cc = cc[:148].astype(np.int64)
ghz = (cc[:, 2] - cc[:, 1]) / np.maximum(c[:, 2] - c[:, 1], 1)
print(f"SM clock over each CTA's work span (GHz, min/median/max): {q(ghz)}")
