"""Run each hot-path op once on a config (default C5) -- the command profiled by ncu.
usage: python tools/prof_ops.py [C5] [ops...]   ops: A B BT K pcg1 wbfbt2"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
from paper_1607_03936_b200 import Context  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C5"
ops = sys.argv[2:] or ["A", "B", "BT", "K", "pcg1"]
inp = synth.make_inputs(cfg, 0)
c = Context(inp["N"], inp["k"])
d = lambda a: torch.as_tensor(a, dtype=torch.float64, device="cuda")  # noqa: E731
mu, u, p = d(inp["mu_q"]), d(inp["u"]), d(inp["p"])
yv, pv = torch.empty(c.n_v, dtype=torch.float64, device="cuda"), torch.empty(c.n_p, dtype=torch.float64, device="cuda")
c.set_viscosity(mu)
for op in ops:
    if op == "A": c.apply_A(u, yv)
    elif op == "B": c.apply_B(u, pv)
    elif op == "BT": c.apply_BT(p, yv)
    elif op == "K": c.apply_K(1, p, pv)
    elif op == "pcg1": c.poisson_pcg(1, p, pv, 1)
    elif op == "wbfbt2": c.apply_wbfbt(p, pv, 2)
torch.cuda.synchronize()
print("ok", ops)
