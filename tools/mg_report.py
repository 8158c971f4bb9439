"""Record of the round-2 rows at full size: pressure / velocity multigrid
parity against the oracle, mesh-independent MG-PCG convergence, and the multi-sinker Stokes
solve with the three Schur approximations.
    python tools/mg_report.py [--seeds 0,1,2] [--out profiles/mg_stokes_r02.json]"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seeds", default="0,1,2")
    ap.add_argument("--configs", default="C2,C3,C5")
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "mg_stokes_r02.json"))
    a = ap.parse_args()
    import torch
    import synth
    from oracle import mg as omg
    from tests.gpu_common import Pair, dev, empty, host, rel_l2
    recs = []
    for cfg in a.configs.split(","):
        for seed in [int(s) for s in a.seeds.split(",")]:
            t0 = time.time()
            P = Pair(cfg, seed=seed)
            c, o, st = P.ctx, P.o, P.ost
            rec = dict(cfg=cfg, seed=seed, N=P.N)
            c.setup_mg(3, P.mu)
            mg_r = omg.MG(P.N, st["Dw"])
            b = P.inp["p"]
            bp = o.project(b)
            rec["levels"] = int(c.query("mg_levels"))
            rec["vcycle"] = rel_l2(host(c.mg_vcycle(1, dev(bp), empty(c.n_p))), mg_r.vcycle(bp))
            rec["mgcg_prefix"] = {str(it): rel_l2(host(c.poisson_mgcg(1, dev(b), empty(c.n_p), it)), mg_r.pcg(b, it))
                                  for it in (1, 3, 8)}
            got = None
            for it in range(4, 60, 2):
                x = host(c.poisson_mgcg(1, dev(bp), empty(c.n_p), it))
                if o.poisson_relres(st["Dinv"], bp, x) < 1e-6:
                    got = it
                    break
            rec["mgcg_iters_to_1e-6"] = got
            V = omg.VMG(P.N, P.inp["mu_q"])
            mask = o.boundary_mask().astype(bool)
            ub = np.where(mask, 0.0, P.inp["u"])
            rec["velocity_vcycle"] = rel_l2(host(c.velocity_vcycle(dev(ub), empty(c.n_v))), V.vcycle(ub))
            fq = dev(synth.forcing_at_quadrature(P.N, P.k, P.inp["centers"], P.cfg.delta, P.cfg.omega))
            rec["stokes"] = {}
            for name, kind in (("wBFBT", 0), ("M_p(1/mu)", 2), ("diag(A)-BFBT", 1)):
                c.set_schur(kind)
                c.set_viscosity(P.mu)
                c.setup_mg(3, P.mu)
                c.set_velocity_mg(2)
                c.set_inner_mg(8 if kind == 0 else 0)
                f = c.load_vector(fq, empty(c.n_v))
                g = empty(c.n_p).zero_()
                u, p = empty(c.n_v), empty(c.n_p)
                torch.cuda.synchronize()
                ts = time.perf_counter()
                _, _, it, rr = c.stokes_fgmres(f, g, u, p, 200, 300, 1e-6, 20, 6, 1.0, 2.0)
                torch.cuda.synchronize()
                rec["stokes"][name] = dict(iterations=it, relres=rr, seconds=time.perf_counter() - ts)
            c.set_schur(0)
            rec["wall_s"] = round(time.time() - t0, 1)
            print(json.dumps(rec), flush=True)
            recs.append(rec)
            del P
    with open(a.out, "w") as fo:
        json.dump(dict(what="round-2 multigrid / Stokes record at full size (tools/mg_report.py)", records=recs), fo,
                  indent=1)


if __name__ == "__main__":
    main()
