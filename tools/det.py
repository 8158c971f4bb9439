"""Run-to-run determinism probe of each op on one config."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
from paper_1607_03936_b200 import Context  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C5"
inp = synth.make_inputs(cfg, 0)
c = Context(inp["N"], inp["k"])
d = lambda a: torch.as_tensor(a, dtype=torch.float64, device="cuda")  # noqa: E731
mu, u, p = d(inp["mu_q"]), d(inp["u"]), d(inp["p"])
c.set_viscosity(mu)
f64 = dict(dtype=torch.float64, device="cuda")


def rep(name, fn, n, k=6):
    outs = []
    for _ in range(k):
        o = torch.empty(n, **f64)
        fn(o)
        outs.append(o)
    torch.cuda.synchronize()
    bad = [i for i in range(1, k) if not torch.equal(outs[0], outs[i])]
    md = max((float((outs[0] - outs[i]).abs().max()) for i in bad), default=0.0)
    print(f"{name}: {'DETERMINISTIC' if not bad else f'NONDET runs {bad} maxdiff {md:.3e}'}")


rep("A", lambda o: c.apply_A(u, o), c.n_v)
rep("B", lambda o: c.apply_B(u, o), c.n_p)
rep("BT", lambda o: c.apply_BT(p, o), c.n_v)
for kv in (0, 1):
    c.set_option("k_variant", kv)
    rep(f"K kvar={kv}", lambda o: c.apply_K(1, p, o), c.n_p)
    rep(f"pcg1 kvar={kv}", lambda o: c.poisson_pcg(1, p, o, 1), c.n_p)
    rep(f"pcg3 kvar={kv}", lambda o: c.poisson_pcg(1, p, o, 3), c.n_p)
    for g in (0, 1):
        c.set_option("graph", g)
        rep(f"pcg30 kvar={kv} graph={g}", lambda o: c.poisson_pcg(1, p, o, 30), c.n_p)
    c.set_option("graph", 1)
rep("wbfbt", lambda o: c.apply_wbfbt(p, o, 100), c.n_p, k=3)
