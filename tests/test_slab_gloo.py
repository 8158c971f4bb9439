"""CPU (gloo) tests of the slab decomposition's host logic (DESIGN.md
Sec. 9): `DistComm` moves the shared planes between rank-1 / rank+1 in the directions
include/wbfbt.h states and all-reduces the scalar slots, with world sizes 2 and 3 (a middle
rank has both neighbours).  The decomposition identity the library implements -- global
operator = sum over ranks of UNMASKED cube operators, plane partials summed, global mask --
is checked here with the oracle's cube as the local operator against the oracle's box
(tests/test_oracle_box.py pins the box), so the exchange directions are tested end to end
without a GPU."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _plane_sum(comm, fields, n_nodes, npl):
    """The library's dd_plane_sum on numpy fields through the communicator's buffers."""
    nf = len(fields)
    for i, f in enumerate(fields):
        comm.send_lo[i * npl:(i + 1) * npl] = torch.from_numpy(f[:npl].copy())
        comm.send_hi[i * npl:(i + 1) * npl] = torch.from_numpy(f[n_nodes - npl:].copy())
    comm.exchange(nf * npl)
    for i, f in enumerate(fields):
        if comm.has_lo:
            f[:npl] += comm.recv_lo[i * npl:(i + 1) * npl].numpy()
        if comm.has_hi:
            f[n_nodes - npl:] += comm.recv_hi[i * npl:(i + 1) * npl].numpy()


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import Oracle
        from paper_1607_03936_b200.slab import DistComm
        N, k = 3, 2
        nn1 = k * N + 1
        npl = nn1 * nn1
        loc, glob = Oracle(N, k), Oracle(N, k, Nz=world * N)
        comm = DistComm(3 * npl, "cpu")
        assert (comm.rank, comm.nranks, comm.has_lo, comm.has_hi) == (rank, world, rank > 0, rank < world - 1)
        rng = np.random.default_rng(7)  # the same global data on every rank
        mu = rng.uniform(0.1, 10.0, glob.n_el * glob.n_q)
        u, p = rng.standard_normal(glob.n_v), rng.standard_normal(glob.n_p)
        gmask = 1.0 - glob.boundary_mask().astype(np.float64)  # n_v, 1 interior
        g0 = rank * k * N * npl

        def loc_v(v):
            return np.concatenate([v[c * glob.n_nodes + g0:c * glob.n_nodes + g0 + loc.n_nodes] for c in range(3)])
        # B^T: unmasked cube apply, plane sum, global mask
        y = loc.apply_BT(p[rank * loc.n_p:(rank + 1) * loc.n_p], nomask=True)
        f = [y[c * loc.n_nodes:(c + 1) * loc.n_nodes] for c in range(3)]
        _plane_sum(comm, f, loc.n_nodes, npl)
        y *= loc_v(gmask)
        ref = loc_v(glob.apply_BT(p))
        e_bt = float(np.abs(y - ref).max() / np.abs(ref).max())
        # A: global-masked input, unmasked cube apply, plane sum, mask
        mu_l = mu[rank * loc.n_el * loc.n_q:(rank + 1) * loc.n_el * loc.n_q]
        ya = loc.apply_A(mu_l, loc_v(u) * loc_v(gmask), nomask=True)
        f = [ya[c * loc.n_nodes:(c + 1) * loc.n_nodes] for c in range(3)]
        _plane_sum(comm, f, loc.n_nodes, npl)
        ya *= loc_v(gmask)
        ref = loc_v(glob.apply_A(mu, u))
        e_a = float(np.abs(ya - ref).max() / np.abs(ref).max())
        # scalar slots: sum and max, a slot range with an offset, identical bits on every rank
        comm.scal[:] = torch.arange(8, dtype=torch.float64) * (rank + 1)
        comm.allreduce(1, 2, 0)
        comm.allreduce(5, 1, 1)
        sc = comm.scal.numpy().copy()
        out[rank] = (e_bt, e_a, sc.tolist(), comm.n_exchange)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_slab_exchange_and_identity_gloo(world):
    mp_ctx = mp.get_context("spawn")
    with mp_ctx.Manager() as m:
        out = m.dict()
        port = _free_port()
        procs = [mp_ctx.Process(target=_worker, args=(r, world, port, out)) for r in range(world)]
        for p in procs:
            p.start()
        for p in procs:
            p.join(240)
            assert p.exitcode == 0
        res = [out[r] for r in range(world)]
    tri = world * (world + 1) // 2
    for r, (e_bt, e_a, sc, _) in enumerate(res):
        assert e_bt <= 1e-13 and e_a <= 1e-13, (r, e_bt, e_a)
        exp = [float(i * (r + 1)) for i in range(8)]
        exp[1], exp[2] = 1.0 * tri, 2.0 * tri  # summed slots 1, 2
        exp[5] = 5.0 * world                   # max slot 5
        assert sc == exp, (r, sc)
