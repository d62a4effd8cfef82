"""Algorithm 1's training step replayed as ONE CUDA graph.

The eager step (training/algorithm1.py train_step) launches hundreds of small
kernels — two forwards, a double-backward for the PDE Laplacian, the gradient
flatten / allreduce / unflatten, LAMB per tensor — and syncs the host for the
loss values and LAMB's trust ratios.  Here the step is captured once with static
shapes and replayed with `torch.cuda.CUDAGraph` (the B200-native answer to
launch overhead: streams and graphs, not a tracing compiler):

* `DeviceLamb` is the same LAMB with its step counter, bias corrections,
  trust ratios and learning rate kept in device tensors, so nothing in the step
  syncs the host and every replay advances the state;
* the batch (boundaries, data queries / labels, collocation points) is copied
  into static input buffers before each replay;
* with world > 1 the ONE gradient allreduce (NCCL) is captured too (step 3 of P:289).

`tests/test_gpu_algorithm1.py` checks replayed steps against the eager step.
"""
from __future__ import annotations

import torch
import torch.nn.functional as F

from training.algorithm1 import Batch, SDNet, laplacian


class DeviceLamb:
    """LAMB with device-resident state: m, v per tensor; t, lr as 0-d tensors."""

    def __init__(self, params, lr=1e-3, betas=(0.9, 0.999), eps=1e-6, weight_decay=0.0):
        self.params = [p for p in params]
        dev, dt = self.params[0].device, self.params[0].dtype
        self.b1, self.b2, self.eps, self.wd = betas[0], betas[1], eps, weight_decay
        self.t = torch.zeros((), device=dev, dtype=dt)
        self.lr = torch.full((), lr, device=dev, dtype=dt)
        self.m = [torch.zeros_like(p) for p in self.params]
        self.v = [torch.zeros_like(p) for p in self.params]

    def set_lr(self, lr: float):
        self.lr.fill_(lr)   # outside the graph: a device write the next replay reads

    @torch.no_grad()
    def step(self):
        self.t.add_(1.0)
        c1 = 1.0 - torch.pow(torch.full_like(self.t, self.b1), self.t)
        c2 = 1.0 - torch.pow(torch.full_like(self.t, self.b2), self.t)
        for p, m, v in zip(self.params, self.m, self.v):
            g = p.grad
            m.mul_(self.b1).add_(g, alpha=1 - self.b1)
            v.mul_(self.b2).addcmul_(g, g, value=1 - self.b2)
            r = (m / c1) / ((v / c2).sqrt() + self.eps)
            if self.wd > 0:
                r = r + self.wd * p
            wn, rn = p.norm(), r.norm()
            trust = torch.where((wn > 0) & (rn > 0), wn / rn, torch.ones_like(wn))
            p.sub_(r * (self.lr * trust))


class GraphStep:
    """One Algorithm-1 iteration captured as a CUDA graph; call `step(batch)`."""

    def __init__(self, net: SDNet, opt: DeviceLamb, example: Batch, pde_weight: float = 1.0, world: int = 1,
                 warmup: int = 3):
        self.net, self.opt, self.pde_weight, self.world = net, opt, pde_weight, world
        self.g = example.g.clone()
        self.Xd = example.Xd.clone()
        self.Yd = example.Yd.clone()
        self.Xc = example.Xc.clone()
        for p in net.parameters():
            if p.grad is None:
                p.grad = torch.zeros_like(p)
        # warm up on a side stream (lazy allocations, autograd caches), then capture
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        state = [p.detach().clone() for p in net.parameters()]
        with torch.cuda.stream(s):
            for _ in range(warmup):
                self._body()
        torch.cuda.current_stream().wait_stream(s)
        # undo the warm-up's optimizer updates: the first real step starts from
        # the caller's weights and a fresh LAMB state
        with torch.no_grad():
            for p, w in zip(net.parameters(), state):
                p.copy_(w)
            opt.t.zero_()
            for m, v in zip(opt.m, opt.v):
                m.zero_()
                v.zero_()
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph):
            self.loss_d, self.loss_p = self._body()

    def _body(self):
        for p in self.net.parameters():
            p.grad.zero_()
        loss_d = F.mse_loss(self.net(self.g, self.Xd), self.Yd)
        loss_d.backward()
        loss_p = self.pde_weight * laplacian(self.net, self.g, self.Xc.detach().clone()).pow(2).mean()
        loss_p.backward()
        if self.world > 1:
            import torch.distributed as dist
            grads = [p.grad for p in self.net.parameters()]
            flat = torch.cat([g.reshape(-1) for g in grads])
            dist.all_reduce(flat)
            flat /= self.world
            o = 0
            for g in grads:
                g.copy_(flat[o:o + g.numel()].view_as(g))
                o += g.numel()
        self.opt.step()
        return loss_d.detach(), loss_p.detach()

    def step(self, b: Batch):
        self.g.copy_(b.g)
        self.Xd.copy_(b.Xd)
        self.Yd.copy_(b.Yd)
        self.Xc.copy_(b.Xc)
        self.graph.replay()
        return self.loss_d, self.loss_p   # device tensors (read them when needed)
