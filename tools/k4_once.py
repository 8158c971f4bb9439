"""One C4 Jacobi-PCG solve (10 iterations, no graph) through the fused k = 4 Poisson kernel
variant argv[1] (-1: the unfused kernels), for ncu captures of k_K4_fused."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
from paper_1607_03936_b200 import Context  # noqa: E402

var = int(sys.argv[1]) if len(sys.argv) > 1 else 0
inp = synth.make_inputs("C4", 0)
c = Context(inp["N"], inp["k"])
d = lambda a: torch.as_tensor(a, dtype=torch.float64, device="cuda")  # noqa: E731
c.set_viscosity(d(inp["mu_q"]))
c.set_option("graph", 0)
if var < 0:
    c.set_option("k4f", 0)
else:
    c.set_option("k4_var", var)
p = d(inp["p"])
x = torch.empty_like(p)
c.poisson_pcg(1, p, x, 10)
torch.cuda.synchronize()
