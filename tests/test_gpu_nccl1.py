"""The NCCL code paths on one GPU through a 1-rank communicator (mfp_nccl_comm_init
with nranks = 1 passed to a 1x1 context): the collective config / weight digest
of mfp_init, the delta allreduce-MAX inside the captured CUDA-graph blocks (P:43
"convergence threshold"; with a communicator the stop rule stays host-checked),
the watchdog's stream polling, the non-finite agreement.  Results must be
bit-identical to the same solve without a communicator.  (Multi-rank NCCL needs
more than one GPU: NCCL refuses two ranks on one device.)
"""
import numpy as np
import pytest

from mfp_inputs import gp_boundary, random_weights

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def lib():
    import torch
    assert torch.cuda.is_available()
    import paper_2308_14258_b200 as mfp
    return mfp


@pytest.mark.parametrize("subsolver,precision,tol", [("exact", 0, 1e-5), ("sdnet", 1, 0.0), ("sdnet", 1, 1e-4)])
def test_one_rank_communicator_bit_identical(lib, subsolver, precision, tol):
    nx = ny = 256
    g = gp_boundary(nx, ny, 6)
    sub = lib.EXACT_LAPLACE if subsolver == "exact" else lib.SDNET
    w = None if subsolver == "exact" else random_weights(0)
    cfg = lib.make_config(nx, ny, precision=precision, subsolver=sub, check_every=4)
    net = lib.make_net(gelu=0 if precision == 0 else 1)
    comm = lib.mfp_nccl_comm_init(1, lib.mfp_nccl_get_unique_id(), 0)
    try:
        a = lib.Mfp(cfg, net, w, rank=0, nccl_comm=comm)
        b = lib.Mfp(cfg, net, w, rank=0)
        t = 2000 if tol > 0 else 11
        ua, ra = a.solve(g, t, tol * float(np.max(np.abs(g))))
        ub, rb = b.solve(g, t, tol * float(np.max(np.abs(g))))
        assert ra.iterations == rb.iterations and ra.converged == rb.converged
        assert ra.last_delta == rb.last_delta
        assert np.array_equal(ua, ub)
        a.close()
        b.close()
    finally:
        lib.mfp_nccl_comm_destroy(comm)


def test_one_rank_communicator_rejects_all_ranks(lib):
    comm = lib.mfp_nccl_comm_init(1, lib.mfp_nccl_get_unique_id(), 0)
    try:
        cfg = lib.make_config(64, 64, (1, 2), subsolver=lib.EXACT_LAPLACE)
        with pytest.raises(lib.MfpError) as e:
            lib.Mfp(cfg, lib.make_net(), None, rank=lib.ALL_RANKS, nccl_comm=comm)
        assert e.value.status == 1
        with pytest.raises(lib.MfpError) as e:      # communicator size != grid size
            lib.Mfp(lib.make_config(64, 64, (1, 2), subsolver=lib.EXACT_LAPLACE), lib.make_net(), None, rank=0,
                    nccl_comm=comm)
        assert e.value.status == 1
    finally:
        lib.mfp_nccl_comm_destroy(comm)
