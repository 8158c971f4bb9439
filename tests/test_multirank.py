"""World-size-2 CPU (gloo) test of bench.py's multi-GPU host logic (DESIGN.md
Sec. 9, replicas only): each rank gets its own seeded problem, the reported time
is the max over ranks, and the job throughput counts every rank's steps."""
import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import bench
        import synth
        seed = bench.replica_seed(rank)
        inp = synth.make_inputs("C1", seed)
        t_local = 10.0 + rank  # rank 1 is slower
        t_max = bench.max_over_ranks(t_local, world)
        out[rank] = (seed, float(inp["mu_q"].sum()), t_max, bench.job_throughput(world, 4, t_max))
        bench.barrier(world)
    finally:
        dist.destroy_process_group()


def test_two_rank_replicas_gloo():
    mp_ctx = mp.get_context("spawn")
    with mp_ctx.Manager() as m:
        out = m.dict()
        port = _free_port()
        procs = [mp_ctx.Process(target=_worker, args=(r, 2, port, out)) for r in range(2)]
        for p in procs:
            p.start()
        for p in procs:
            p.join(120)
            assert p.exitcode == 0
        r0, r1 = out[0], out[1]
    assert r0[0] == 0 and r1[0] == 1            # distinct problems per rank
    assert r0[1] != r1[1]                        # different sinker centres -> different mu
    assert r0[2] == r1[2] == 11.0                # max over ranks, seen by both
    assert r0[3] == pytest.approx(2 * 4 / 11e-3)  # all ranks' steps over the slowest time
