"""Small invocations of every product kernel family, for compute-sanitizer (SURVEY.md Sec. 5:
race / memory checking).  usage: python tools/san_case.py [small|tma]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_1607_03936_b200 import Context  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "small"
cases = [("C1", None), ("C2", 8), ("C4", 3)] if which == "small" else [("C5", 44)]
d = lambda a: torch.as_tensor(a, dtype=torch.float64, device="cuda")  # noqa: E731
for cfg, N in cases:
    inp = synth.make_inputs(cfg, 0, N=N)
    c = Context(inp["N"], inp["k"])
    mu, u, p = d(inp["mu_q"]), d(inp["u"]), d(inp["p"])
    f64 = dict(dtype=torch.float64, device="cuda")
    yA, pB, yBT, z = (torch.empty(n, **f64) for n in (c.n_v, c.n_p, c.n_v, c.n_p))
    c.hotpath(mu, u, p, 3, yA, pB, yBT, z)
    c.apply_K(1, p, z)
    if which == "tma":
        c.set_option("k_zm", 1)
        c.poisson_pcg(1, p, z, 3)
        c.set_option("k_zm", 0)
        c.set_option("kz", 1)
        c.poisson_pcg(1, p, z, 3)
    lam = c.poisson_eigmax(1, p, 3)
    c.poisson_cheb(1, p, z, 3, 0.1 * lam, 1.1 * lam)
    if inp["k"] == 2:
        c.setup_mg(2, mu)
        c.poisson_mgcg(1, p, z, 2)
        c.velocity_vcycle(u, yA)
        c.set_inner_mg(1)
        c.set_velocity_mg(1)
    c.apply_dabfbt(p, z, 2)
    fq = d(synth.forcing_at_quadrature(inp["N"], inp["k"], inp["centers"], 200.0, 0.1))
    F = c.load_vector(fq, torch.empty(c.n_v, **f64))
    c.stokes_fgmres(F, torch.zeros(c.n_p, **f64), yA, z, 3, 2, 0.0, 2, 2, 1.0, 2.0)
    c.set_schur(2)
    c.set_viscosity(mu)
    c.apply_mpinv(p, z)
    c.sync()
    torch.cuda.synchronize()
    print(cfg, N, "ok", float(z.abs().sum()), flush=True)
print("done")
