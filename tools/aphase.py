"""Phase timeline of the k = 2 A tile kernel (thread 0 of each CTA, clock64 cycles per CTA).
Rebuilds the library with -DWB_KPROF in place (rebuild normally afterwards)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "paper_1607_03936_b200"))
import build  # noqa: E402

build.FLAGS += ["-DWB_KPROF"]
build.build(force=True)
import torch  # noqa: E402

import synth  # noqa: E402
from paper_1607_03936_b200 import Context  # noqa: E402

inp = synth.make_inputs(sys.argv[1] if len(sys.argv) > 1 else "C5", 0)
c = Context(inp["N"], inp["k"])
d = lambda a: torch.as_tensor(a, dtype=torch.float64, device="cuda")  # noqa: E731
c.set_viscosity(d(inp["mu_q"]))
u = d(inp["u"])
y = torch.empty(c.n_v, dtype=torch.float64, device="cuda")
c.apply_A(u, y)
c.query("aprof7")
for _ in range(5):
    c.apply_A(u, y)
v = [c.query(f"aprof{k}") for k in range(8)]
names = ["staging issue", "staging wait+bar", "U load+interp", "Gauss levels", "interp^T", "slots+bar",
         "node sums/out"]
tot = sum(v[:7])
print(f"CTAs {v[7]:.0f}; cycles per CTA (thread 0)")
for k, n in enumerate(names):
    print(f"  {n:18s} {v[k] / v[7]:8.1f}  {100 * v[k] / tot:5.1f} %")
print(f"  total {tot / v[7]:8.1f} cycles per CTA")
