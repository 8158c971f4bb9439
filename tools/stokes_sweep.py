"""Stokes FGMRES iterations / time to 1e-6 with both multigrids, over preconditioner knobs.
usage: python tools/stokes_sweep.py C5"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
from paper_1607_03936_b200 import Context  # noqa: E402

cfg = synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C5"]
inp = synth.make_inputs(cfg, 0)
d = lambda a: torch.as_tensor(a, dtype=torch.float64, device="cuda")  # noqa: E731
mu = d(inp["mu_q"])
fq = d(synth.forcing_at_quadrature(cfg.N, cfg.k, inp["centers"], cfg.delta, cfg.omega))
for schur, nu, cyc, inner, restart in ((0, 3, 1, 4, 100), (0, 3, 2, 4, 100), (0, 5, 1, 4, 100), (0, 3, 1, 8, 100),
                                       (0, 3, 2, 8, 200), (2, 3, 2, 0, 200), (1, 3, 2, 0, 200)):
    c = Context(cfg.N, cfg.k)
    c.set_schur(schur)
    c.set_viscosity(mu)
    c.setup_mg(nu, mu)
    c.set_velocity_mg(cyc)
    if inner:
        c.set_inner_mg(inner)
    f = c.load_vector(fq, torch.empty(c.n_v, dtype=torch.float64, device="cuda"))
    g = torch.zeros(c.n_p, dtype=torch.float64, device="cuda")
    u, p = torch.empty_like(f), torch.empty_like(g)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    _, _, it, rr = c.stokes_fgmres(f, g, u, p, restart, 600, 1e-6, 20, 6, 1.0, 2.0)
    torch.cuda.synchronize()
    print(f"{cfg.name} schur={schur} nu={nu} vcycles={cyc} inner_mg={inner} restart={restart}: {it} it, "
          f"relres {rr:.2e}, {time.perf_counter() - t0:.1f} s", flush=True)
    del c
