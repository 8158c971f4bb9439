"""A few C4 A(mu)u applies (the k = 4 slice kernel + gather), for ncu captures."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
from paper_1607_03936_b200 import Context  # noqa: E402

inp = synth.make_inputs(sys.argv[1] if len(sys.argv) > 1 else "C4", 0)
c = Context(inp["N"], inp["k"])
d = lambda a: torch.as_tensor(a, dtype=torch.float64, device="cuda")  # noqa: E731
c.set_viscosity(d(inp["mu_q"]))
u = d(inp["u"])
y = torch.empty_like(u)
for _ in range(3):
    c.apply_A(u, y)
torch.cuda.synchronize()
