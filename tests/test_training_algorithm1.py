"""CPU tests of Algorithm 1 (training/algorithm1.py).

Pins: the training SDNet IS the hot path's network (oracle forward on its MFCK
flat parameters, fp64); its data labels are the oracle's harmonic extension
(LU-built) to 1e-12; the PDE term's autograd Laplacian agrees with central finite
differences; LAMB moves each tensor by exactly lr * ||w|| (trust ratio); and the
data-parallel step — local data + PDE backward, ONE allreduce of the summed
gradients / world — equals the single-process step on the whole batch (gloo,
world size 2)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as tmp

import oracle
from training.algorithm1 import Batch, Lamb, Problem, SDNet, harmonic_matrix, laplacian, query_points, train_step

M = 32


def test_labels_match_oracle_harmonic_matrix():
    Hc = harmonic_matrix(query_points("centre"))
    assert np.max(np.abs(Hc - oracle.harmonic_matrix(0))) < 1e-12
    Hf = harmonic_matrix(query_points("interior"))
    assert np.max(np.abs(Hf - oracle.harmonic_matrix(1))) < 1e-12


def test_training_net_is_the_hot_path_net():
    torch.manual_seed(3)
    net = SDNet().double()
    g = torch.randn(5, 4 * M, dtype=torch.float64)
    X = torch.tensor(oracle.writeset(0, 0)[1], dtype=torch.float64)
    ours = net(g, X).detach().numpy()
    ref = oracle.sdnet_forward(net.flat(), g.numpy(), X.numpy())
    assert np.max(np.abs(ours - ref)) < 1e-12 * max(1.0, np.max(np.abs(ref)))
    net2 = SDNet().double()
    net2.load_flat(net.flat())
    assert np.array_equal(net2.flat(), net.flat())


def test_laplacian_matches_finite_differences():
    torch.manual_seed(4)
    net = SDNet().double()
    g = torch.randn(3, 4 * M, dtype=torch.float64)
    X = 0.1 + 0.8 * torch.rand(3, 7, 2, dtype=torch.float64)
    lap = laplacian(net, g, X.clone()).detach().numpy()
    h = 1e-3
    with torch.no_grad():
        u0 = net(g, X)
        fd = torch.zeros_like(u0)
        for d in range(2):
            e = torch.zeros_like(X)
            e[..., d] = h
            fd += (net(g, X + e) - 2 * u0 + net(g, X - e)) / (h * h)
    assert np.max(np.abs(lap - fd.numpy())) <= 1e-4 * max(1.0, np.max(np.abs(lap)))


def test_lamb_trust_ratio():
    torch.manual_seed(5)
    w = [torch.nn.Parameter(torch.randn(7, 3, dtype=torch.float64)), torch.nn.Parameter(torch.randn(4, dtype=torch.float64))]
    before = [p.detach().clone() for p in w]
    opt = Lamb(w, lr=0.01)
    for p in w:
        p.grad = torch.randn_like(p)
    opt.step()
    for p, b in zip(w, before):
        assert abs(float((p.detach() - b).norm()) - 0.01 * float(b.norm())) < 1e-12


def _ddp_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.manual_seed(0)
    net = SDNet().double()
    opt = Lamb(net.parameters(), lr=1e-3)
    prob = Problem(torch.device("cpu"), torch.float64, n_interior=16, n_colloc=8)
    gen = torch.Generator()
    gen.manual_seed(7)
    full = prob.batch(8, gen)                  # the same global batch on every rank
    sl = slice(4 * rank, 4 * rank + 4)
    b = Batch(full.g[sl], full.Xd, full.Yd[sl], full.Xc[sl])
    train_step(net, opt, b, pde_weight=1e-2, world=world)
    if rank == 0:
        q.put(net.flat())
    dist.destroy_process_group()


def test_data_parallel_step_equals_single_process():
    torch.manual_seed(0)
    net = SDNet().double()
    opt = Lamb(net.parameters(), lr=1e-3)
    prob = Problem(torch.device("cpu"), torch.float64, n_interior=16, n_colloc=8)
    gen = torch.Generator()
    gen.manual_seed(7)
    train_step(net, opt, prob.batch(8, gen), pde_weight=1e-2, world=1)
    ref = net.flat()
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = tmp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_ddp_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = q.get(timeout=300)
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    assert np.max(np.abs(got - ref)) < 1e-12


def test_lr_schedule_and_worker_scaling():
    """§5.2 via SPEC's lr_at / scale_for_workers examples."""
    from training.algorithm1 import lr_at, scale_for_workers
    assert lr_at(1e-3, 0.01, 1.0, 0, 1000) == 0.0                 # ramp start
    assert abs(lr_at(1e-3, 0.01, 1.0, 10, 1000) - 1e-3) < 1e-15   # ramp end (ceil(0.01 * 1000) = 10)
    assert abs(lr_at(1e-3, 0.01, 1.0, 505, 1000) - 5e-4) < 1e-15  # halfway through the decay span
    assert lr_at(1e-3, 0.01, 1.0, 1000, 1000) == 0.0               # 0 at the final iteration
    assert abs(lr_at(1e-3, 0.01, 1.0, 9, 1000) - 9e-4) < 1e-15
    assert abs(scale_for_workers(1e-3, 1e-3, 4)[0] - 2e-3) < 1e-15  # p = 4: sqrt rule
    assert abs(scale_for_workers(1e-3, 1e-3, 16)[1] - 0.016) < 1e-15  # p = 16: linear warmup rule
    assert scale_for_workers(1e-3, 0.1, 16)[1] == 0.5


def test_device_lamb_equals_lamb():
    """training/graph_step.py DeviceLamb (device-resident t, lr, trust ratio; the
    CUDA-graph-capturable form) makes the same LAMB updates as Lamb."""
    from training.graph_step import DeviceLamb
    torch.manual_seed(11)
    a, b = SDNet().double(), SDNet().double()
    b.load_flat(a.flat())
    oa, ob = Lamb(a.parameters(), lr=2e-3, weight_decay=1e-4), DeviceLamb(list(b.parameters()), lr=2e-3,
                                                                          weight_decay=1e-4)
    for it in range(5):
        g = torch.Generator().manual_seed(it)
        for pa, pb in zip(a.parameters(), b.parameters()):
            grad = torch.randn(pa.shape, dtype=torch.float64, generator=g)
            pa.grad = grad.clone()
            pb.grad = grad.clone()
        oa.step()
        ob.step()
    assert np.max(np.abs(a.flat() - b.flat())) < 1e-12
