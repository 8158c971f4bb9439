"""Slab-decomposition record: GPU (ranks as host threads on one GPU) against
the oracle's box mesh, with the errors written out, plus the one-rank cost of the slab code path
against the fused single-GPU path.  Writes gpurun_out/slab_r02.json.
usage: python tools/slab_report.py [--full]"""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tests.gpu_common import dev, empty, host, rel_l2  # noqa: E402
from tests.test_gpu_slab import SlabCase, run_ranks  # noqa: E402


def one(N, k, R, seed, cfg=None, iters=(1, 5, 10), wb_iters=4):
    c = SlabCase(N, k, R, a_l=2.0, a_r=3.0, seed=seed, cfg=cfg)
    rec = {"N": N, "k": k, "ranks": R, "seed": seed, "box": [N, N, N * R],
           "nonpos": [c.ost["n_nonpos_Cw"], c.ost["n_nonpos_Dw"]]}
    us = [dev(c.loc_v(c.u, r)) for r in range(R)]
    ps = [dev(c.loc_p(c.p, r)) for r in range(R)]

    def f(r):
        x = c.ctx[r]
        return (host(x.apply_A(us[r], empty(x.n_v))), host(x.apply_B(us[r], empty(x.n_p))),
                host(x.apply_BT(ps[r], empty(x.n_v))), host(x.apply_K(0, ps[r], empty(x.n_p))),
                host(x.apply_K(1, ps[r], empty(x.n_p))))
    res = run_ranks(R, f, c.comms)
    yA, pB, yBT = c.o.apply_A(c.mu, c.u), c.o.apply_B(c.u), c.o.apply_BT(c.p)
    qL, qR = c.o.apply_K(c.ost["Cinv"], c.p), c.o.apply_K(c.ost["Dinv"], c.p)
    rec["A"] = max(rel_l2(res[r][0], c.loc_v(yA, r)) for r in range(R))
    rec["B"] = max(rel_l2(res[r][1], c.loc_p(pB, r)) for r in range(R))
    rec["BT"] = max(rel_l2(res[r][2], c.loc_v(yBT, r)) for r in range(R))
    rec["K_l"] = max(rel_l2(res[r][3], c.loc_p(qL, r)) for r in range(R))
    rec["K_r"] = max(rel_l2(res[r][4], c.loc_p(qR, r)) for r in range(R))
    if rec["nonpos"] == [0, 0]:
        rec["pcg_prefix"] = {}
        for it in iters:
            got = np.concatenate(run_ranks(R, lambda r: host(c.ctx[r].poisson_pcg(1, ps[r], empty(c.nl_p), it)),
                                           c.comms))
            rec["pcg_prefix"][str(it)] = rel_l2(got, c.o.poisson(c.ost["Dinv"], c.ost["diagKr"], c.p, it))
        got = np.concatenate(run_ranks(R, lambda r: host(c.ctx[r].apply_wbfbt(ps[r], empty(c.nl_p), wb_iters)),
                                       c.comms))
        rec[f"wbfbt_{wb_iters}"] = rel_l2(got, c.o.wbfbt(c.p, wb_iters))
    c.close()
    return rec


def cost_C5():
    """One rank at C5: slab code path (unfused K_w, launch-by-launch PCG) vs the fused path."""
    import synth
    from paper_1607_03936_b200 import Context, SlabContext, ThreadComm
    inp = synth.make_inputs("C5", 0)
    mu, p = dev(inp["mu_q"]), dev(inp["p"])
    a = Context(64, 2)
    b = SlabContext(64, 2, ThreadComm.group(1, SlabContext.plane_cap(64, 2), "cuda")[0])
    a.set_viscosity(mu)
    b.set_viscosity(mu)
    z = empty(a.n_p)

    def t(fn, reps=5):
        fn()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(reps):
            fn()
        torch.cuda.synchronize()
        return (time.perf_counter() - t0) / reps * 1e3
    out = {"fused_wbfbt_ms": t(lambda: a.apply_wbfbt(p, z, 100)), "slab1_wbfbt_ms": t(lambda: b.apply_wbfbt(p, z, 100)),
           "fused_K_ms": t(lambda: a.apply_K(1, p, z), 20), "slab1_K_ms": t(lambda: b.apply_K(1, p, z), 20)}
    out["slab1_pcg_iter_us"] = (t(lambda: b.poisson_pcg(1, p, z, 60), 3) - t(lambda: b.poisson_pcg(1, p, z, 20), 3)) / 40 * 1e3
    za, zb = host(a.apply_wbfbt(p, empty(a.n_p), 20)), host(b.apply_wbfbt(p, empty(b.n_p), 20))
    out["slab1_vs_fused_wbfbt20_rel_l2"] = rel_l2(zb, za)
    a.close(); b.close()
    return out


def main():
    cases = [(8, 2, 2), (16, 2, 2), (16, 2, 3), (13, 2, 3), (32, 2, 2), (8, 4, 2), (12, 4, 3), (6, 3, 2)]
    recs = []
    for N, k, R in cases:
        for seed in (0, 1):
            recs.append(one(N, k, R, seed))
            print(json.dumps(recs[-1]), flush=True)
    if "--full" in sys.argv:
        recs.append(one(64, 2, 2, 0, cfg="C5", iters=(1, 5, 10, 20), wb_iters=10))
        print(json.dumps(recs[-1]), flush=True)
    out = {"parity": recs, "cost_C5_one_rank": cost_C5()}
    print(json.dumps(out["cost_C5_one_rank"]))
    os.makedirs("gpurun_out", exist_ok=True)
    json.dump(out, open("gpurun_out/slab_r02.json", "w"), indent=1)


if __name__ == "__main__":
    main()
