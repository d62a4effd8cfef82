"""NEXT-2 timing: device time of an MFP solve on every rank of a Py x Px grid on
one GPU (MFP_ALL_RANKS), halo through device copies (pack, cudaMemcpyAsync,
unpack) vs the peer-memory kernels (pack+publish, fused pull+unpack) vs the
put transport (halo cells stored into the peers' put buffers by the chain
epilogue, publish, local unpack).  One
device serialises all ranks, so this compares launch counts and per-exchange
overhead of the transports, not NVLink bandwidth.

    python tools/p2p_vs_copy.py [--n 4096] [--grid 2 4] [--iters 64] [--out json]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

import paper_2308_14258_b200 as mfp  # noqa: E402
from mfp_inputs import gp_boundary, random_weights  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=4096)
    ap.add_argument("--grid", type=int, nargs=2, default=[2, 4])
    ap.add_argument("--iters", type=int, default=64)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    g = gp_boundary(a.n, a.n, 1)
    w = random_weights(0)
    res = {"workload": f"{a.n + 1}^2, grid {a.grid[0]}x{a.grid[1]} all ranks on one GPU, bf16 SDNet (W-rand), "
                       f"{a.iters} iterations, check_every 16", "transports": {}}
    for name in ("copy", "p2p", "put"):
        cfg = mfp.make_config(a.n, a.n, tuple(a.grid), precision=1, subsolver=mfp.SDNET, check_every=16)
        m = mfp.Mfp(cfg, mfp.make_net(gelu=1), w, rank=mfp.ALL_RANKS)
        if name in ("p2p", "put"):
            mfp.mfp_p2p_open(m.ctx)
        if name == "put":
            mfp.mfp_p2p_set_mode(m.ctx, mfp.P2P_PUT)
        ms, u_last = [], None
        for _ in range(a.reps + 1):
            u, rep = m.solve(g, a.iters, 0.0)
            ms.append(rep.ms_total - rep.ms_final)
            u_last = u
        ms = sorted(ms[1:])
        prof = m.profile(a.iters)  # per-kernel events, no graphs: the halo span on the side stream
        res["transports"][name] = {"ms_per_iter_median": ms[len(ms) // 2] / a.iters,
                                   "gpu_launches_per_solve": rep.gpu_launches,
                                   "halo_ms_per_iter_profiled": prof.ms_halo,
                                   "halo_bytes_per_iter": rep.halo_bytes_sent / a.iters}
        res["transports"][name]["_u"] = u_last
    u0 = res["transports"]["copy"].pop("_u")
    res["bit_identical"] = {k: bool(np.array_equal(u0, res["transports"][k].pop("_u"))) for k in ("p2p", "put")}
    print(json.dumps(res, indent=1))
    if a.out:
        with open(a.out, "w") as f:
            json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
