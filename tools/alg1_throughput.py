"""Algorithm 1 step throughput on one GPU (boundaries / s), eager and replayed as one
CUDA graph (training/graph_step.py): python tools/alg1_throughput.py [batch] [steps]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from training.algorithm1 import Lamb, Problem, SDNet, train_step  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 256
K = int(sys.argv[2]) if len(sys.argv) > 2 else 50
torch.manual_seed(0)
net = SDNet().cuda()
opt = Lamb(net.parameters(), lr=1e-3)
prob = Problem(torch.device("cuda"), torch.float32)
gen = torch.Generator(device="cuda")
gen.manual_seed(0)
batches = [prob.batch(B, gen) for _ in range(4)]
for i in range(5):
    train_step(net, opt, batches[i % 4], 1e-3)
torch.cuda.synchronize()
t0 = time.perf_counter()
for i in range(K):
    train_step(net, opt, batches[i % 4], 1e-3)
torch.cuda.synchronize()
dt = time.perf_counter() - t0
eager = {"ms_per_step": 1000 * dt / K, "boundaries_per_s": K * B / dt}
from training.graph_step import DeviceLamb, GraphStep  # noqa: E402
net2 = SDNet().cuda()
gs = GraphStep(net2, DeviceLamb(list(net2.parameters()), lr=1e-3), batches[0], 1e-3)
for i in range(5):
    gs.step(batches[i % 4])
torch.cuda.synchronize()
t0 = time.perf_counter()
for i in range(K):
    gs.step(batches[i % 4])
torch.cuda.synchronize()
dg = time.perf_counter() - t0
print(json.dumps({"experiment": "Algorithm 1 step (P:289) on 1 B200, fp32: eager PyTorch vs the step replayed "
                                "as one CUDA graph (training/graph_step.py)",
                  "batch_per_rank": B, "data_queries": 61 + prob.n_interior, "collocation_points": prob.n_colloc,
                  "steps": K, "eager": eager,
                  "graph": {"ms_per_step": 1000 * dg / K, "boundaries_per_s": K * B / dg}}))
