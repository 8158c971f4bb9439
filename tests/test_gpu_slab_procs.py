"""The slab decomposition as REAL separate processes (one per rank, torch.distributed): two
processes share the one GPU of the test box and exchange through gloo with host staging
(`DistComm` on a non-NCCL backend; NCCL refuses two ranks on one device).  Each process waits
for the other on the HOST only.  Results against the oracle's global box mesh."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import synth
from tests.gpu_common import rel_l2

pytestmark = pytest.mark.gpu

N, K, ITERS = 16, 2, 5


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _inputs(world):
    parts = [synth.make_inputs("C2", 10 + r, N=N) for r in range(world)]
    rng = np.random.default_rng(5)
    n_nodes_g = (K * N + 1) ** 2 * (K * N * world + 1)
    n_p_g = parts[0]["sizes"]["n_p"] * world
    return parts, rng.standard_normal(3 * n_nodes_g), rng.standard_normal(n_p_g)


def _worker(rank, world, port, out):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1607_03936_b200 import DistComm, SlabContext
        parts, u, p = _inputs(world)
        comm = DistComm(SlabContext.plane_cap(N, K), "cuda")
        assert comm.staged
        ctx = SlabContext(N, K, comm)
        d = lambda a: torch.as_tensor(np.ascontiguousarray(a), dtype=torch.float64, device="cuda")  # noqa: E731
        ctx.set_viscosity(d(parts[rank]["mu_q"]), 1.0, 2.0)
        npl, nl = (K * N + 1) ** 2, ctx.n_nodes
        ng = npl * (K * N * world + 1)
        g0 = rank * K * N * npl
        ul = np.concatenate([u[c * ng + g0:c * ng + g0 + nl] for c in range(3)])
        pl = p[rank * ctx.n_p:(rank + 1) * ctx.n_p]
        yA = ctx.apply_A(d(ul), torch.empty(ctx.n_v, dtype=torch.float64, device="cuda"))
        z = ctx.apply_wbfbt(d(pl), torch.empty(ctx.n_p, dtype=torch.float64, device="cuda"), ITERS)
        ctx.sync()
        out[rank] = (yA.cpu().numpy(), z.cpu().numpy(), comm.n_exchange, comm.n_allreduce)
        ctx.close()
    finally:
        dist.destroy_process_group()


def test_two_processes_one_gpu_gloo():
    from oracle import Oracle
    world = 2
    mp_ctx = mp.get_context("spawn")
    with mp_ctx.Manager() as m:
        out = m.dict()
        port = _free_port()
        procs = [mp_ctx.Process(target=_worker, args=(r, world, port, out)) for r in range(world)]
        for pr in procs:
            pr.start()
        for pr in procs:
            pr.join(600)
            assert pr.exitcode == 0
        res = [out[r] for r in range(world)]
    parts, u, p = _inputs(world)
    o = Oracle(N, K, Nz=world * N)
    mu = np.concatenate([q["mu_q"] for q in parts])
    o.setup(mu, 1.0, 2.0)
    yA, z = o.apply_A(mu, u), o.wbfbt(p, ITERS)
    npl, nl, ng = (K * N + 1) ** 2, (K * N + 1) ** 3, o.n_nodes
    for r in range(world):
        g0 = r * K * N * npl
        ref = np.concatenate([yA[c * ng + g0:c * ng + g0 + nl] for c in range(3)])
        assert rel_l2(res[r][0], ref) <= 1e-11
        assert res[r][2] > 0 and res[r][3] > 0
    assert rel_l2(np.concatenate([res[0][1], res[1][1]]), z) <= 1e-9
    # the shared plane of A u: both owners hold the same bits
    a0, a1 = res[0][0].reshape(3, nl), res[1][0].reshape(3, nl)
    assert np.array_equal(a0[:, nl - npl:], a1[:, :npl])
