"""FGMRES Stokes solve with the multi-sinker forcing: iterations to the
paper's 1e-6 residual reduction for inner-solve choices.
usage: python tools/stokes_exp.py C2 [smooth_iters ...]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_1607_03936_b200 import Context  # noqa: E402

cfg = synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C2"]
sms = [int(a) for a in sys.argv[2:]] or [6, 20]
inp = synth.make_inputs(cfg, 0)
c = Context(inp["N"], inp["k"])
d = lambda a: torch.as_tensor(a, dtype=torch.float64, device="cuda")  # noqa: E731
c.set_viscosity(d(inp["mu_q"]))
fq = d(synth.forcing_at_quadrature(cfg.N, cfg.k, inp["centers"], cfg.delta, cfg.omega))
f = c.load_vector(fq, torch.empty(c.n_v, dtype=torch.float64, device="cuda"))
g = torch.zeros(c.n_p, dtype=torch.float64, device="cuda")
v0 = d(np.random.default_rng(8).standard_normal(c.n_v))
lam = c.velocity_eigmax(v0, 20)
c.setup_mg(3)
u = torch.empty(c.n_v, dtype=torch.float64, device="cuda")
p = torch.empty(c.n_p, dtype=torch.float64, device="cuda")
for inner in ("pcg", "mg2", "mg5"):
    if inner.startswith("mg"):
        c.set_inner_mg(int(inner[2:]))
    else:
        c.set_inner_mg(0)
    for sm in sms:
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        _, _, it, rr = c.stokes_fgmres(f, g, u, p, 100, 400, 1e-6, cfg.iters, sm, 0.1 * lam, 1.1 * lam)
        torch.cuda.synchronize()
        print(f"{cfg.name} inner={inner} smooth={sm}: {it} iterations, relres {rr:.2e}, {time.perf_counter() - t0:.2f} s",
              flush=True)
