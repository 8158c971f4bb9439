"""Run the C5 Poisson PCG a few times with the given library options (for ncu captures).
usage: python tools/k_once.py key=value ...   e.g. k_zm=1 zm_zc=8"""
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
for kv in sys.argv[1:]:
    k, v = kv.split("=")
    c.set_option(k, float(v))
c.set_option("graph", 0)
p = d(inp["p"])
out = torch.empty(c.n_p, dtype=torch.float64, device="cuda")
for _ in range(3):
    c.poisson_pcg(1, p, out, 10)
torch.cuda.synchronize()
print("ok", c.query("k_zm"))
