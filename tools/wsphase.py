"""Role timeline of the warp-specialised Poisson kernel k_K2_ws (k_dbg 0x4000):
clock64 cycles per tile of consumer thread 0 and producer thread 0, summed over all
CTAs of a 50-iteration PCG at C5.  Rebuilds the library with -DWB_KPROF in place
(rebuild normally afterwards)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "paper_1607_03936_b200"))
import torch  # noqa: E402

import build  # noqa: E402

build.FLAGS += ["-DWB_KPROF"] + [f for f in os.environ.get("WS_FLAGS", "").split() if f]
build.build(force=True)
import synth  # noqa: E402
from paper_1607_03936_b200 import Context  # noqa: E402

inp = synth.make_inputs("C5", 0)
c = Context(inp["N"], inp["k"])
d = lambda a: torch.as_tensor(a, dtype=torch.float64, device="cuda")  # noqa: E731
mu, p = d(inp["mu_q"]), d(inp["p"])
pv = torch.empty(c.n_p, dtype=torch.float64, device="cuda")
c.set_viscosity(mu)
c.set_option("k_ws", 1)
iters = 50
c.set_option("k_dbg", 0x4000 | 0x2000 | int(os.environ.get("WS_DBG", "0"), 0))
c.poisson_pcg(1, p, pv, iters)
c.query("kprof7")  # clear
c.poisson_pcg(1, p, pv, iters)
v = [c.query(f"kprof{k}") for k in range(8)]
c.set_option("k_dbg", 0)
tiles = v[7]
print(f"k_K2_ws: {tiles:.0f} tiles over {iters} launches; cycles per tile")
for k, n in enumerate(["consumer wait full", "consumer wait X", "consumer step 1 + bar", "consumer step 2 + bar",
                       "producer wait empty", "producer wait raw", "producer step 0 + bar"]):
    print(f"  {n:24s} {v[k] / tiles:9.1f}")
print(f"  consumer total {sum(v[:4]) / tiles:9.1f}   producer total {sum(v[4:7]) / tiles:9.1f}")
