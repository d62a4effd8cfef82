#!/usr/bin/env python
"""Fit SDNet weights ("W-fit") — a data-generation / training
tool, NOT part of the hot path and not the paper's Algorithm 1 (no PDE loss, no
DDP): plain data-loss regression of the exact SDNet architecture (reading G7) onto
the exact discrete harmonic extension of its boundary (PAPER §2.1, P:512-519;
the role pyAMG-labelled data plays in §5.1-5.2).

    python tools/fit_sdnet.py --steps 20000 --out weights/sdnet_fit_d128.npy

Labels: H ĝ for the 61 centre-line queries and the 961 interior queries of a
33 x 33 patch, H from the closed-form DST-I expansion of the 5-point Dirichlet
problem (written out here in numpy; shares nothing with the product or the
oracle).  Boundaries: a mixture of (a) SE-kernel GP curves along the perimeter
(the paper's §5.1 recipe), (b) restrictions of random smooth fields (what an MFP
subdomain sees at convergence), (c) edge-wise zeroed versions of both (what it
sees while interior lines still hold the zero initial guess), with random
offsets and scales.  Weights are saved fp32 in SPEC MFCK order.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
M = 32


def perimeter_points(m=M):
    pts = [(i, 0) for i in range(m)] + [(m, i) for i in range(m)] + \
          [(m - i, m) for i in range(m)] + [(0, m - i) for i in range(m)]
    return np.array(pts)


def query_points(kind: str, m=M):
    if kind == "centre":
        pts = [(m // 2, k) for k in range(1, m)] + [(k, m // 2) for k in range(1, m) if k != m // 2]
    else:
        pts = [(i, j) for j in range(1, m) for i in range(1, m)]
    return np.array(pts)


def harmonic_matrix(kind: str, m=M) -> np.ndarray:
    """H[q, k]: value at query q of the discrete harmonic function whose
    boundary is the unit vector e_k (G1 perimeter order)."""
    qs = query_points(kind, m)
    H = np.zeros((len(qs), 4 * m))
    ks = np.arange(1, m)
    th = np.pi * ks / m
    lk = np.arccosh(2.0 - np.cos(th))
    for kb, (bx, by) in enumerate(perimeter_points(m)):
        side, pos = divmod(kb, m)
        if side == 0:
            s_b, along, dist = pos, qs[:, 0], qs[:, 1]
        elif side == 1:
            s_b, along, dist = pos, qs[:, 1], m - qs[:, 0]
        elif side == 2:
            s_b, along, dist = m - pos, qs[:, 0], m - qs[:, 1]
        else:
            s_b, along, dist = m - pos, qs[:, 1], qs[:, 0]
        if s_b == 0 or s_b == m:
            continue
        terms = (2.0 / m) * np.sin(th[None, :] * s_b) * np.sin(th[None, :] * along[:, None]) * \
            np.sinh(lk[None, :] * (m - dist[:, None])) / np.sinh(lk[None, :] * m)
        H[:, kb] = terms.sum(1)
    return H


def sample_boundaries(torch, n, device, gen):
    """Mixture of boundary signals, (n, 128) fp32."""
    nb = 4 * M
    s = torch.linspace(0, 1, nb, device=device)
    out = torch.empty((n, nb), device=device)
    k = n // 3
    # (a) GP curves along the perimeter via random Fourier features of an SE kernel
    var = 0.1 + 0.9 * torch.rand(k, 1, device=device, generator=gen)
    ls = 0.05 + 0.45 * torch.rand(k, 1, device=device, generator=gen)
    F = 64
    w = torch.randn(k, F, device=device, generator=gen) / ls
    b = 2 * math.pi * torch.rand(k, F, device=device, generator=gen)
    a = torch.randn(k, F, device=device, generator=gen)
    out[:k] = torch.sqrt(2 * var / F) * (a[:, :, None] * torch.cos(w[:, :, None] * s[None, None, :] + b[:, :, None])).sum(1)
    # (b) restrictions of random smooth 2-D fields (random low-frequency modes)
    pp = torch.tensor(perimeter_points(), device=device, dtype=torch.float32) / M
    n2 = n - 2 * k
    kx = 2.5 * torch.randn(n2, 6, device=device, generator=gen)
    ky = 2.5 * torch.randn(n2, 6, device=device, generator=gen)
    ph = 2 * math.pi * torch.rand(n2, 6, device=device, generator=gen)
    amp = torch.randn(n2, 6, device=device, generator=gen) / 3
    arg = kx[:, :, None] * pp[None, None, :, 0] + ky[:, :, None] * pp[None, None, :, 1] + ph[:, :, None]
    out[2 * k:] = (amp[:, :, None] * torch.sin(arg)).sum(1)
    # (c) copies of (a)/(b) with whole edges zeroed (interior lines still at the initial 0)
    pick = torch.randint(0, n - k, (k,), device=device, generator=gen)
    src = out[torch.where(pick < k, pick, pick + k)]      # rows of (a) or (b) only
    mask = (torch.rand(k, 4, device=device, generator=gen) < 0.35).float()
    mask = mask.repeat_interleave(M, dim=1)
    out[k:2 * k] = src * (1 - mask)
    if BANK is not None:
        # (e) boundaries the MFP iteration itself feeds the subsolver
        # (tools/collect_mfp_boundaries.py): zero-interior starts to near convergence
        nk = int(n * BANK_FRAC)
        idx = torch.randint(0, BANK.shape[0], (nk,), device=device, generator=gen)
        out[:nk] = BANK[idx]
    if SMOOTH > 0:
        # (d) harmonic polynomials of degree <= 3 with random coefficients: what a
        # subdomain sees near convergence on a large domain, where the MFP's slowly
        # contracting iteration amplifies any systematic error of the subsolver
        ns = int(n * SMOOTH)
        x = pp[None, :, 0] - 0.5
        y = pp[None, :, 1] - 0.5
        basis = torch.stack([torch.ones_like(x[0]), x[0], y[0], x[0] ** 2 - y[0] ** 2, x[0] * y[0],
                             x[0] ** 3 - 3 * x[0] * y[0] ** 2, 3 * x[0] ** 2 * y[0] - y[0] ** 3], 0)   # (7, 128)
        c = torch.randn(ns, 7, device=device, generator=gen) * torch.tensor(
            [0.5, 0.6, 0.6, 0.5, 0.5, 0.3, 0.3], device=device)
        out[n - ns:] = c @ basis
    if not WIDE:
        return out
    # random offsets and scales (harmonic extension commutes with both)
    off = torch.randn(n, 1, device=device, generator=gen) * 0.5
    sc = torch.exp(torch.randn(n, 1, device=device, generator=gen) * 0.3)
    return out * sc + off


WIDE = False  # --wide: add random offsets / scales to the boundary mixture
SMOOTH = 0.0  # --smooth f: fraction of the batch replaced by harmonic polynomials (degree <= 3)
QAT = None    # --qat bf16|fp16: train through the chain's 16-bit operand rounding
BANK = None   # --bank file: boundary vectors collected from MFP runs; BANK_FRAC of each batch
BANK_FRAC = 0.5


def main():
    import torch
    import torch.nn as nn
    import torch.nn.functional as F

    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=20000)
    ap.add_argument("--batch", type=int, default=1024)
    ap.add_argument("--lr", type=float, default=1e-3)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--out", default=os.path.join(ROOT, "weights", "sdnet_fit_d128.npy"))
    ap.add_argument("--wide", action="store_true")
    ap.add_argument("--smooth", type=float, default=0.0)
    ap.add_argument("--bank", default=None)
    ap.add_argument("--qat", default=None, choices=[None, "bf16", "fp16"])
    ap.add_argument("--bank-frac", type=float, default=0.5)
    ap.add_argument("--normalized-loss", action="store_true")
    ap.add_argument("--init", default=None, help="start from these flat weights (MFCK order)")
    ap.add_argument("--eval", action="store_true", help="only evaluate --init")
    args = ap.parse_args()
    global WIDE, SMOOTH, BANK, BANK_FRAC, QAT
    WIDE = args.wide
    SMOOTH = args.smooth
    BANK_FRAC = args.bank_frac
    if args.qat:
        QAT = torch.bfloat16 if args.qat == "bf16" else torch.float16
    dev = torch.device("cuda" if torch.cuda.is_available() else "cpu")
    torch.manual_seed(args.seed)
    if args.bank:
        BANK = torch.tensor(np.load(args.bank), dtype=torch.float32, device=dev)
    gen = torch.Generator(device=dev)
    gen.manual_seed(args.seed)

    Hc = torch.tensor(harmonic_matrix("centre"), dtype=torch.float32, device=dev)
    Hf = torch.tensor(harmonic_matrix("interior"), dtype=torch.float32, device=dev)
    Xc = torch.tensor(query_points("centre") / M, dtype=torch.float32, device=dev)
    Xf = torch.tensor(query_points("interior") / M, dtype=torch.float32, device=dev)

    class SDNet(nn.Module):
        def __init__(s, d=128, nh=3):
            super().__init__()
            s.c0 = nn.Conv1d(1, 8, 5)
            s.c1 = nn.Conv1d(8, 1, 5)
            s.W1 = nn.Linear(4 * M, d)               # boundary half of the split layer (Eq. 5)
            s.W2 = nn.Linear(2, d, bias=False)        # query half
            s.hid = nn.ModuleList([nn.Linear(d, d) for _ in range(nh)])
            s.head = nn.Linear(d, 1)

        def forward(s, g, X):
            x = g[:, None, :]
            x = F.gelu(s.c0(F.pad(x, (2, 2), mode="circular")))
            x = F.gelu(s.c1(F.pad(x, (2, 2), mode="circular")))
            z = s.W1(x.flatten(1))
            h = F.gelu(z[:, None, :] + s.W2(X)[None])
            for lin in s.hid:
                if QAT is not None:
                    # the tensor-core chain's operands: activations h' and weights rounded
                    # to 16 bit (RN), fp32 accumulate; straight-through gradients
                    hq = h + (h.to(QAT).float() - h).detach()
                    wq = lin.weight + (lin.weight.to(QAT).float() - lin.weight).detach()
                    h = F.gelu(F.linear(hq, wq, lin.bias))
                else:
                    h = F.gelu(lin(h))
            return s.head(h)[..., 0]

        def load_flat(s, v):
            v = torch.as_tensor(v, dtype=torch.float32)
            o = 0
            parts = [s.c0.weight, s.c0.bias, s.c1.weight, s.c1.bias, s.W1.weight, s.W2.weight, s.W1.bias]
            for lin in s.hid:
                parts += [lin.weight, lin.bias]
            parts += [s.head.weight, s.head.bias]
            with torch.no_grad():
                for p in parts:
                    p.copy_(v[o:o + p.numel()].reshape(p.shape))
                    o += p.numel()
            assert o == v.numel()

        def flat(s):
            parts = [s.c0.weight, s.c0.bias, s.c1.weight, s.c1.bias, s.W1.weight, s.W2.weight, s.W1.bias]
            for lin in s.hid:
                parts += [lin.weight, lin.bias]
            parts += [s.head.weight[0], s.head.bias]
            return torch.cat([p.detach().reshape(-1).float().cpu() for p in parts]).numpy()

    net = SDNet().to(dev)
    if args.init:
        net.load_flat(np.load(args.init))
    if args.eval:
        args.steps = 0
    opt = torch.optim.AdamW(net.parameters(), lr=args.lr, weight_decay=0.0)
    sched = torch.optim.lr_scheduler.OneCycleLR(opt, max_lr=args.lr, total_steps=max(args.steps, 100),
                                                pct_start=max(0.02, 4.0 / max(args.steps, 4)))
    t0 = time.time()
    log = []
    for step in range(args.steps if not args.eval else 0):
        g = sample_boundaries(torch, args.batch, dev, gen)
        scale = g.abs().amax(1, keepdim=True) + 1e-3
        # centre-line queries every step (the hot path) + a random interior subset (final phase)
        sub = torch.randint(0, Xf.shape[0], (96,), device=dev, generator=gen)
        X = torch.cat([Xc, Xf[sub]])
        Y = torch.cat([g @ Hc.T, g @ Hf[sub].T], 1)
        pred = net(g, X)
        loss = (((pred - Y) / scale) ** 2).mean() if args.normalized_loss else ((pred - Y) ** 2).mean()
        opt.zero_grad(set_to_none=True)
        loss.backward()
        opt.step()
        sched.step()
        if step % 500 == 0 or step == args.steps - 1:
            log.append((step, float(loss)))
            print(f"step {step} loss {float(loss):.3e} ({time.time() - t0:.0f} s)", flush=True)
    # validation on fresh samples, all queries
    with torch.no_grad():
        g = sample_boundaries(torch, 4096, dev, gen)
        g = g[g.abs().amax(1) > 1e-3]          # drop boundaries whose every edge was zeroed
        scale = g.abs().amax(1, keepdim=True)
        ec = ((net(g, Xc) - g @ Hc.T) / scale).abs()
        ef = ((net(g, Xf) - g @ Hf.T) / scale).abs()
    flat = net.flat()
    if args.eval:
        print(json.dumps({"val_centre_max_rel_err": float(ec.max()), "val_centre_mean_rel_err": float(ec.mean()),
                          "val_interior_max_rel_err": float(ef.max()), "val_interior_mean_rel_err": float(ef.mean())}))
        return
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    np.save(args.out, flat.astype(np.float32))
    meta = {"params": int(flat.size), "steps": args.steps, "batch": args.batch, "lr": args.lr, "seed": args.seed,
            "val_centre_max_rel_err": float(ec.max()), "val_centre_mean_rel_err": float(ec.mean()),
            "val_interior_max_rel_err": float(ef.max()), "val_interior_mean_rel_err": float(ef.mean()),
            "train_seconds": time.time() - t0, "loss_log": log}
    json.dump(meta, open(args.out.replace(".npy", ".json"), "w"), indent=1)
    print(json.dumps({k: v for k, v in meta.items() if k != "loss_log"}))


if __name__ == "__main__":
    main()
