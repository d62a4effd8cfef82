"""Algorithm 1 of arXiv 2308.14258: data-parallel training of the SDNet
with a physics-informed loss — SURVEY §8(f) NEXT-3, the paper's second
data-parallel workload.  Not the MFP hot path (that is libmfp); this trains the
weights the hot path consumes (MFCK order, `mfp_init`'s `params`).

One training iteration on every rank:
  1. forward + backward of the DATA loss on the rank's data points — gradients
     accumulate locally, no synchronisation;
  2. forward + backward of the PDE loss on the rank's collocation points —
     accumulated onto the same gradients;
  3. ONE allreduce of the flattened gradient bucket, divided by the world size
     (the global average of  L = L_data + L_pde ), then
  4. the optimizer step, LAMB (You et al.) with per-tensor trust ratios.

Data loss: MSE against the exact discrete harmonic extension of the boundary
(the role of the paper's pyAMG labels), at the 61 centre-line queries and a
random subset of the 961 interior queries.  PDE loss: mean of (N_xx + N_yy)^2 at
random collocation points of the open patch, the second derivatives of the
network output with respect to its query coordinates ("N_xx and N_yy"),
by double reverse-mode autograd.  The query coordinates are per sample
(B, q, 2) so that derivatives stay per point; Eq. 5's broadcasted sum
z[s] + W2 x_p is kept.

PyTorch is the compute here (cuBLAS GEMMs, autograd); torch.distributed (NCCL
on GPUs, gloo on CPU) carries the allreduce.  Launch:
    python -m torch.distributed.run --nproc-per-node N training/algorithm1.py --steps 2000
"""
from __future__ import annotations

import argparse
import json
import math
import os
import sys
import time

import numpy as np
import torch
import torch.nn as nn
import torch.nn.functional as F

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

M = 32


# --------------------------------------------------------------------- model
class SDNet(nn.Module):
    """Reading G7: conv1d 1->8->1 (k = 5, circular) + GELU, split
    layer U = GELU(g W1^T (+) X W2^T) (Eq. 5), n_hidden x (d x d + GELU), linear head."""

    def __init__(self, d: int = 128, n_hidden: int = 3, m: int = M):
        super().__init__()
        self.c0 = nn.Conv1d(1, 8, 5)
        self.c1 = nn.Conv1d(8, 1, 5)
        self.W1 = nn.Linear(4 * m, d)
        self.W2 = nn.Linear(2, d, bias=False)
        self.hid = nn.ModuleList([nn.Linear(d, d) for _ in range(n_hidden)])
        self.head = nn.Linear(d, 1)

    def forward(self, g: torch.Tensor, X: torch.Tensor) -> torch.Tensor:
        """g (B, 4m) boundaries; X (q, 2) shared or (B, q, 2) per-sample queries -> (B, q)."""
        x = g[:, None, :]
        x = F.gelu(self.c0(F.pad(x, (2, 2), mode="circular")))
        x = F.gelu(self.c1(F.pad(x, (2, 2), mode="circular")))
        z = self.W1(x.flatten(1))                                   # (B, d)
        q = self.W2(X)                                              # (q, d) or (B, q, d)
        h = F.gelu(z[:, None, :] + (q[None] if q.dim() == 2 else q))
        for lin in self.hid:
            h = F.gelu(lin(h))
        return self.head(h)[..., 0]

    def parts(self):
        p = [self.c0.weight, self.c0.bias, self.c1.weight, self.c1.bias, self.W1.weight, self.W2.weight, self.W1.bias]
        for lin in self.hid:
            p += [lin.weight, lin.bias]
        return p + [self.head.weight, self.head.bias]

    def flat(self) -> np.ndarray:
        """Parameters in SPEC MFCK order, the layout mfp_init takes."""
        return torch.cat([t.detach().reshape(-1).double().cpu() for t in self.parts()]).numpy()

    def load_flat(self, v) -> None:
        v = torch.as_tensor(np.asarray(v), dtype=torch.float64)
        o = 0
        with torch.no_grad():
            for t in self.parts():
                t.copy_(v[o:o + t.numel()].reshape(t.shape).to(t.dtype))
                o += t.numel()
        assert o == v.numel()


# ------------------------------------------------------------------ data
def perimeter_points(m: int = M) -> np.ndarray:
    return np.array([(i, 0) for i in range(m)] + [(m, i) for i in range(m)] +
                    [(m - i, m) for i in range(m)] + [(0, m - i) for i in range(m)])


def query_points(kind: str, m: int = M) -> np.ndarray:
    if kind == "centre":
        return np.array([(m // 2, k) for k in range(1, m)] + [(k, m // 2) for k in range(1, m) if k != m // 2])
    return np.array([(i, j) for j in range(1, m) for i in range(1, m)])


def harmonic_matrix(qs: np.ndarray, m: int = M) -> np.ndarray:
    """H[q, k]: the 5-point discrete harmonic extension of the unit boundary vector
    e_k (G1 perimeter order) at the grid queries qs — closed-form DST-I expansion of
    the (m+1)^2 Dirichlet problem (the labels of the data loss)."""
    H = np.zeros((len(qs), 4 * m))
    ks = np.arange(1, m)
    th = np.pi * ks / m
    lk = np.arccosh(2.0 - np.cos(th))
    for kb in range(4 * m):
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
        H[:, kb] = ((2.0 / m) * np.sin(th[None, :] * s_b) * np.sin(th[None, :] * along[:, None]) *
                    np.sinh(lk[None, :] * (m - dist[:, None])) / np.sinh(lk[None, :] * m)).sum(1)
    return H


def sample_boundaries(n: int, gen: torch.Generator, device, dtype) -> torch.Tensor:
    """Smooth boundary signals (n, 4m): SE-kernel GP curves along the perimeter by
    random Fourier features (P:19's recipe, SPEC ranges) and restrictions of random
    low-degree harmonic polynomials."""
    nb = 4 * M
    s = torch.linspace(0, 1, nb, device=device, dtype=dtype)
    k = n // 2
    var = 0.1 + 0.9 * torch.rand(k, 1, device=device, dtype=dtype, generator=gen)
    ls = 0.1 + 0.4 * torch.rand(k, 1, device=device, dtype=dtype, generator=gen)
    Fq = 64
    w = torch.randn(k, Fq, device=device, dtype=dtype, generator=gen) / ls
    b = 2 * math.pi * torch.rand(k, Fq, device=device, dtype=dtype, generator=gen)
    a = torch.randn(k, Fq, device=device, dtype=dtype, generator=gen)
    gp = torch.sqrt(2 * var / Fq) * (a[:, :, None] * torch.cos(w[:, :, None] * s[None, None] + b[:, :, None])).sum(1)
    pp = torch.tensor(perimeter_points(), device=device, dtype=dtype) / M - 0.5
    x, y = pp[:, 0], pp[:, 1]
    basis = torch.stack([torch.ones_like(x), x, y, x * x - y * y, x * y, x ** 3 - 3 * x * y * y], 0)
    c = torch.randn(n - k, basis.shape[0], device=device, dtype=dtype, generator=gen) * 0.5
    return torch.cat([gp, c @ basis], 0)


# ------------------------------------------------------------------ losses
def laplacian(net: SDNet, g: torch.Tensor, Xc: torch.Tensor) -> torch.Tensor:
    """N_xx + N_yy at per-sample query points Xc (B, q, 2) in patch coordinates
    (x/m, y/m in [0, 1]); grid-unit second derivatives scale by 1/m^2, irrelevant for
    the residual's zero."""
    Xc = Xc.requires_grad_(True)
    u = net(g, Xc)
    (du,) = torch.autograd.grad(u.sum(), Xc, create_graph=True)
    (uxx,) = torch.autograd.grad(du[..., 0].sum(), Xc, create_graph=True)
    (uyy,) = torch.autograd.grad(du[..., 1].sum(), Xc, create_graph=True)
    return uxx[..., 0] + uyy[..., 1]


class Batch:
    def __init__(self, g, Xd, Yd, Xc):
        self.g, self.Xd, self.Yd, self.Xc = g, Xd, Yd, Xc


class Problem:
    """Exact labels and query sets, on `device` in `dtype`."""

    def __init__(self, device, dtype, n_interior: int = 64, n_colloc: int = 64):
        self.device, self.dtype = device, dtype
        qc, qf = query_points("centre"), query_points("interior")
        self.Xc_data = torch.tensor(qc / M, device=device, dtype=dtype)
        self.Xf_data = torch.tensor(qf / M, device=device, dtype=dtype)
        self.Hc = torch.tensor(harmonic_matrix(qc), device=device, dtype=dtype)
        self.Hf = torch.tensor(harmonic_matrix(qf), device=device, dtype=dtype)
        self.n_interior, self.n_colloc = n_interior, n_colloc

    def batch(self, n: int, gen: torch.Generator) -> Batch:
        g = sample_boundaries(n, gen, self.device, self.dtype)
        sub = torch.randint(0, self.Xf_data.shape[0], (self.n_interior,), device=self.device, generator=gen)
        Xd = torch.cat([self.Xc_data, self.Xf_data[sub]])
        Yd = torch.cat([g @ self.Hc.T, g @ self.Hf[sub].T], 1)
        Xc = 0.02 + 0.96 * torch.rand(n, self.n_colloc, 2, device=self.device, dtype=self.dtype, generator=gen)
        return Batch(g, Xd, Yd, Xc)


# ------------------------------------------------------------------ LAMB
class Lamb(torch.optim.Optimizer):
    """LAMB: Adam moments with bias correction, decoupled weight decay, and a
    per-tensor trust ratio ||w|| / ||update|| (1 when either norm is 0)."""

    def __init__(self, params, lr=1e-3, betas=(0.9, 0.999), eps=1e-6, weight_decay=0.0):
        super().__init__(params, dict(lr=lr, betas=betas, eps=eps, weight_decay=weight_decay))

    @torch.no_grad()
    def step(self):
        for grp in self.param_groups:
            b1, b2 = grp["betas"]
            for p in grp["params"]:
                if p.grad is None:
                    continue
                st = self.state[p]
                if not st:
                    st["t"] = 0
                    st["m"] = torch.zeros_like(p)
                    st["v"] = torch.zeros_like(p)
                st["t"] += 1
                t, m, v = st["t"], st["m"], st["v"]
                m.mul_(b1).add_(p.grad, alpha=1 - b1)
                v.mul_(b2).addcmul_(p.grad, p.grad, value=1 - b2)
                r = (m / (1 - b1 ** t)) / ((v / (1 - b2 ** t)).sqrt() + grp["eps"])
                if grp["weight_decay"] > 0:
                    r = r + grp["weight_decay"] * p
                wn, rn = p.norm(), r.norm()
                trust = (wn / rn) if (wn > 0 and rn > 0) else torch.ones((), device=p.device, dtype=p.dtype)
                p.add_(r, alpha=-grp["lr"] * float(trust))


# ------------------------------------------------------------------ Algorithm 1
# ---- learning-rate rules of §5.2: warmup + polynomial decay, and the
# data-parallel scaling of max_lr (sqrt of the batch growth) and of the warmup
# fraction (linear in the batch growth); SPEC lr_at / scale_for_workers.
def lr_at(max_lr: float, warmup_frac: float, decay: float, it: int, total: int) -> float:
    """Linear ramp 0 -> max_lr over ceil(warmup_frac * total) iterations, then
    max_lr * (1 - progress)^decay down to 0 at it == total ("0.1% of
    iterations for learning rate warmup ... polynomial learning rate decay with
    the exponent set to one")."""
    import math
    w = int(math.ceil(warmup_frac * total))
    if w > 0 and it < w:
        return max_lr * it / w
    span = max(total - w, 1)
    prog = min(max((it - w) / span, 0.0), 1.0)
    return max_lr * (1.0 - prog) ** decay


def scale_for_workers(max_lr: float, warmup_frac: float, p: int) -> tuple[float, float]:
    """"(a) We scale the maximum learning rate by the square root of the
    increase in batch size. (b) The fraction of iterations used for learning rate
    warmup is scaled linearly" (capped at 1/2)."""
    return max_lr * p ** 0.5, min(warmup_frac * p, 0.5)


def train_step(net: SDNet, opt: torch.optim.Optimizer, b: Batch, pde_weight: float = 1.0, world: int = 1):
    """One iteration of Algorithm 1; returns (data loss, pde loss) of this rank."""
    opt.zero_grad(set_to_none=False)
    # step 1: data points — local backward, no gradient synchronisation
    loss_d = F.mse_loss(net(b.g, b.Xd), b.Yd)
    loss_d.backward()
    # step 2: collocation points — PDE loss, gradients accumulated onto step 1's
    loss_p = pde_weight * laplacian(net, b.g, b.Xc).pow(2).mean()
    loss_p.backward()
    # step 3: ONE allreduce of the summed gradients, averaged over the ranks
    if world > 1:
        import torch.distributed as dist
        grads = [p.grad for p in net.parameters()]
        flat = torch.cat([g.reshape(-1) for g in grads])
        dist.all_reduce(flat)
        flat /= world
        o = 0
        for g in grads:
            g.copy_(flat[o:o + g.numel()].view_as(g))
            o += g.numel()
    # step 4: optimizer
    opt.step()
    return float(loss_d.detach()), float(loss_p.detach())


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--batch", type=int, default=256, help="boundaries per rank per step")
    ap.add_argument("--lr", type=float, default=1e-3, help="max_lr at one rank (P:75); scaled by sqrt(world)")
    ap.add_argument("--warmup-frac", type=float, default=1e-3, help="warmup fraction at one rank (P:75)")
    ap.add_argument("--decay", type=float, default=1.0, help="polynomial decay exponent (P:75)")
    ap.add_argument("--pde-weight", type=float, default=1e-3)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--init", default=None)
    ap.add_argument("--out", default=None)
    ap.add_argument("--graph", action="store_true",
                    help="replay each step as one CUDA graph (training/graph_step.py; device-side LAMB state)")
    a = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", "0"))) if torch.cuda.is_available() else torch.device("cpu")
    if world > 1:
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl" if dev.type == "cuda" else "gloo")
    torch.manual_seed(a.seed)                       # identical initial replicas
    net = SDNet().to(dev)
    if a.init:
        net.load_flat(np.load(a.init))
    # each rank keeps its per-rank batch, so the global batch grows with world:
    # the §5.2 scaling rules set the schedule for that global batch
    max_lr, warmup = scale_for_workers(a.lr, a.warmup_frac, world)
    opt = Lamb(net.parameters(), lr=max_lr)
    prob = Problem(dev, torch.float32)
    gen = torch.Generator(device=dev)
    gen.manual_seed(1000 * a.seed + rank)           # each rank draws its own shard
    t0, log = time.time(), []
    if dev.type == "cuda":
        torch.cuda.synchronize()
    gstep = None
    if a.graph and dev.type == "cuda":
        from training.graph_step import DeviceLamb, GraphStep
        opt = DeviceLamb(list(net.parameters()), lr=max_lr)
        gstep = GraphStep(net, opt, prob.batch(a.batch, gen), a.pde_weight, world)
    for step in range(a.steps):
        lr = lr_at(max_lr, warmup, a.decay, step, a.steps)
        if gstep is not None:
            opt.set_lr(lr)
            ld, lp = (float(x) for x in gstep.step(prob.batch(a.batch, gen)))
            if rank == 0 and (step % 100 == 0 or step == a.steps - 1):
                log.append((step, ld, lp))
                print(f"step {step} data {ld:.3e} pde {lp:.3e}", flush=True)
            continue
        for grp in opt.param_groups:
            grp["lr"] = lr
        ld, lp = train_step(net, opt, prob.batch(a.batch, gen), a.pde_weight, world)
        if rank == 0 and (step % 100 == 0 or step == a.steps - 1):
            log.append((step, ld, lp))
            print(f"step {step} data {ld:.3e} pde {lp:.3e}", flush=True)
    if dev.type == "cuda":
        torch.cuda.synchronize()
    dt = time.time() - t0
    if rank == 0:
        res = {"steps": a.steps, "world": world, "batch_per_rank": a.batch,
               "boundaries_per_s": a.steps * a.batch * world / dt, "seconds": dt, "log": log}
        if a.out:
            np.save(a.out, net.flat().astype(np.float32))
        print(json.dumps(res))
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
