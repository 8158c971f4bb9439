"""A few C5 B / B^T applies through the z-marching column kernels (bbt_zc argv[1]), for ncu."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
from paper_1607_03936_b200 import Context  # noqa: E402

inp = synth.make_inputs("C5", 0)
c = Context(inp["N"], inp["k"])
d = lambda a: torch.as_tensor(a, dtype=torch.float64, device="cuda")  # noqa: E731
c.set_viscosity(d(inp["mu_q"]))
c.set_option("bbt_zc", int(sys.argv[1]) if len(sys.argv) > 1 else 4)
u, p = d(inp["u"]), d(inp["p"])
y, q = torch.empty_like(u), torch.empty_like(p)
for _ in range(2):
    c.apply_B(u, q)
    c.apply_BT(p, y)
torch.cuda.synchronize()
