"""Algorithm 1 on the B200: the data-parallel
SDNet training step runs on the GPU, and the weights it produces drive the hot
path's kernels.

* the training step (data loss + PDE loss with the autograd Laplacian, one
  gradient allreduce, LAMB) runs on cuda and reduces the data loss;
* the GPU step equals the same step in fp64 on the CPU (the CPU suite pins that
  step against the single-process whole-batch step on gloo, world size 2);
* the trained network, exported in MFCK order, IS the network libmfp evaluates:
  mfp_sdnet_batch (fp32 SIMT chain and the FP16X tensor-core chain) against the
  training module's own forward on the same boundaries and queries.
"""
import numpy as np
import pytest
import torch

import oracle
from training.algorithm1 import Lamb, Problem, SDNet, train_step

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def lib():
    assert torch.cuda.is_available()
    import paper_2308_14258_b200 as mfp
    return mfp


def _trained(steps=30, batch=64):
    torch.manual_seed(0)
    net = SDNet().cuda()
    opt = Lamb(net.parameters(), lr=2e-3)
    prob = Problem(torch.device("cuda"), torch.float32, n_interior=32, n_colloc=16)
    gen = torch.Generator(device="cuda")
    gen.manual_seed(7)
    losses = []
    for _ in range(steps):
        ld, _ = train_step(net, opt, prob.batch(batch, gen), pde_weight=1e-3)
        losses.append(ld)
    return net, losses


def test_training_step_on_gpu_reduces_data_loss():
    net, losses = _trained(steps=150)
    assert all(np.isfinite(losses))
    assert np.mean(losses[-20:]) < 0.8 * np.mean(losses[:20])


def test_gpu_step_matches_cpu_fp64_step():
    """Same weights, same batch: the GPU step's losses and accumulated gradient
    (data + PDE, before the optimizer; lr = 0 keeps the weights) agree with the
    fp64 CPU step to fp32 accuracy."""
    torch.manual_seed(1)
    net_g = SDNet().cuda()
    net_c = SDNet().double()
    net_c.load_flat(net_g.flat())
    prob_c = Problem(torch.device("cpu"), torch.float64, n_interior=16, n_colloc=8)
    b = prob_c.batch(16, torch.Generator().manual_seed(3))
    bg = type(b)(b.g.float().cuda(), b.Xd.float().cuda(), b.Yd.float().cuda(), b.Xc.float().cuda())
    opt_g, opt_c = Lamb(net_g.parameters(), lr=0.0), Lamb(net_c.parameters(), lr=0.0)
    ld_g, lp_g = train_step(net_g, opt_g, bg, pde_weight=1e-3)
    ld_c, lp_c = train_step(net_c, opt_c, b, pde_weight=1e-3)
    assert abs(ld_g - ld_c) <= 1e-4 * abs(ld_c)
    assert abs(lp_g - lp_c) <= 1e-2 * abs(lp_c) + 1e-12
    gg = torch.cat([p.grad.reshape(-1).double().cpu() for p in net_g.parameters()]).numpy()
    gc = torch.cat([p.grad.reshape(-1) for p in net_c.parameters()]).numpy()
    assert np.max(np.abs(gg - gc)) <= 1e-3 * np.max(np.abs(gc))


@pytest.mark.parametrize("precision,tol", [(0, 1e-5), (3, 3e-3)])
def test_trained_weights_drive_the_hot_path(lib, precision, tol):
    net, _ = _trained(steps=10)
    w = net.flat().astype(np.float32)
    g = torch.randn(300, 128, device="cuda") * 0.5
    X = torch.tensor(oracle.writeset(0, 0)[1], dtype=torch.float32, device="cuda")
    with torch.no_grad():
        ref = net.double()(g.double(), X.double()).cpu().numpy()
    cfg = lib.make_config(128, 128, precision=precision, subsolver=lib.SDNET, check_every=1)
    m = lib.Mfp(cfg, lib.make_net(gelu=0 if precision == 0 else 2), w)
    out = m.sdnet_batch(g, 0).cpu().numpy()
    assert np.max(np.abs(out - ref)) <= tol * np.max(np.abs(ref))
    m.close()


def test_graph_step_matches_eager():
    """training/graph_step.py: the step replayed as one CUDA graph (device-side
    LAMB state) reproduces the eager step's weights over 8 steps on the same
    batches, to fp32 rounding."""
    from training.graph_step import DeviceLamb, GraphStep
    torch.manual_seed(2)
    net_e = SDNet().cuda()
    net_g = SDNet().cuda()
    net_g.load_flat(net_e.flat())
    prob = Problem(torch.device("cuda"), torch.float32, n_interior=32, n_colloc=16)
    gen = torch.Generator(device="cuda")
    gen.manual_seed(5)
    batches = [prob.batch(64, gen) for _ in range(8)]
    opt_e = Lamb(net_e.parameters(), lr=2e-3)
    opt_g = DeviceLamb(list(net_g.parameters()), lr=2e-3)
    gs = GraphStep(net_g, opt_g, batches[0], pde_weight=1e-3)
    for b in batches:
        ld_e, _ = train_step(net_e, opt_e, b, pde_weight=1e-3)
        ld_g, _ = gs.step(b)
        assert abs(float(ld_g) - ld_e) <= 1e-4 * abs(ld_e) + 1e-7
    we, wg = net_e.flat(), net_g.flat()
    assert np.max(np.abs(we - wg)) <= 1e-4 * np.max(np.abs(we))
