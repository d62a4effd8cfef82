"""Multi-process (gloo, CPU) test of the distributed MFP protocol.

Each rank builds its plan through libmfp's host-only C ABI (compute sets =
mfp_plan_anchors, halo cells = mfp_plan_halo) and runs Algorithm 2 on a
numpy copy of its read region with the exact subsolver (H_c from the oracle,
test-side), exchanging the packed halo values with torch.distributed
send/recv once per iteration.  The owner view after t iterations must equal
the oracle's single-process D1 emulation — which pins the plan's compute
sets, the send/recv lists and their canonical order across real processes.
"""
import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

M = 32


def _worker(rank, world, grid, nx, ny, t, port, out_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    import paper_2308_14258_b200 as mfp
    from mfp_inputs import boundary_points, gp_boundary

    cfg = mfp.make_config(nx, ny, grid, subsolver=mfp.EXACT_LAPLACE)
    info = mfp.mfp_plan_query(cfg, rank)
    H = oracle.harmonic_matrix(0)
    g = gp_boundary(nx, ny, 5).astype(np.float64)
    U = np.zeros((ny + 1, nx + 1))
    bp = boundary_points(nx, ny)
    U[bp[:, 1], bp[:, 0]] = g
    peers = list(info.peers[: info.n_peers])
    sends = [mfp.mfp_plan_halo(cfg, rank, i, 0) for i in range(len(peers))]
    recvs = [mfp.mfp_plan_halo(cfg, rank, i, 1) for i in range(len(peers))]
    anchors = [mfp.mfp_plan_anchors(cfg, rank, ph) for ph in range(4)]
    for _ in range(t):
        for ph in range(4):
            anc = anchors[ph]
            if len(anc) == 0:
                continue
            gb = np.stack([U[oracle.perimeter(ax, ay)[:, 1], oracle.perimeter(ax, ay)[:, 0]] for ax, ay in anc])
            yb = gb @ H.T
            for (ax, ay), y in zip(anc, yb):
                wr, _ = oracle.writeset(ax, ay)
                U[wr[:, 1], wr[:, 0]] = y
        # communicate_new_boundaries: one packed message per neighbour
        reqs, bufs = [], []
        for s, snd, rcv in zip(peers, sends, recvs):
            buf = torch.from_numpy(np.ascontiguousarray(U[snd[:, 2], snd[:, 1]]))
            reqs.append(dist.isend(buf, s))
            rb = torch.empty(len(rcv), dtype=torch.float64)
            reqs.append(dist.irecv(rb, s))
            bufs.append((rcv, rb))
        for r_ in reqs:
            r_.wait()
        for rcv, rb in bufs:
            U[rcv[:, 2], rcv[:, 1]] = rb.numpy()
    # owned line points -> rank 0
    X0, Y0 = info.X0, info.Y0
    X1 = nx + 1 if info.rx == grid[1] - 1 else info.X1
    Y1 = ny + 1 if info.ry == grid[0] - 1 else info.Y1
    block = torch.from_numpy(np.ascontiguousarray(U[Y0:Y1, X0:X1]))
    meta = torch.tensor([X0, X1, Y0, Y1], dtype=torch.int64)
    if rank == 0:
        full = np.zeros((ny + 1, nx + 1))
        full[Y0:Y1, X0:X1] = block.numpy()
        for src in range(1, world):
            m = torch.empty(4, dtype=torch.int64)
            dist.recv(m, src)
            a, b, c, d = m.tolist()
            blk = torch.empty((d - c, b - a), dtype=torch.float64)
            dist.recv(blk, src)
            full[c:d, a:b] = blk.numpy()
        np.save(out_path, full)
    else:
        dist.send(meta, 0)
        dist.send(block, 0)
    dist.destroy_process_group()


@pytest.mark.parametrize("grid,kx,ky,t", [((1, 2), 4, 4, 6), ((2, 2), 4, 4, 5)])
def test_gloo_protocol_matches_oracle_emulation(tmp_path, grid, kx, ky, t):
    import oracle
    from mfp_inputs import gp_boundary
    nx, ny = kx * M, ky * M
    world = grid[0] * grid[1]
    out = str(tmp_path / "u.npy")
    port = 29500 + (os.getpid() % 1000)
    mp.start_processes(_worker, args=(world, grid, nx, ny, t, port, out), nprocs=world, join=True,
                       start_method="spawn")
    got = np.load(out)
    ref = oracle.mfp_run(oracle.MfpConfig(nx, ny, Py=grid[0], Px=grid[1], subsolver="exact"),
                         gp_boundary(nx, ny, 5).astype(np.float64), t, final=False)
    X, Y = np.meshgrid(np.arange(nx + 1), np.arange(ny + 1))
    lines = (X % 16 == 0) | (Y % 16 == 0)
    assert np.max(np.abs(got[lines] - ref.lines[lines])) < 1e-12
