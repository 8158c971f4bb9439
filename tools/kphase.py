"""Phase timeline of the TMA Poisson kernel (k_dbg 0x4000, thread 0 of each CTA,
clock64 cycles): per tile and per launch, from a 50-iteration PCG at C5.
Needs the library built with -DWB_KPROF (this script rebuilds it so, in place;
rebuild normally afterwards)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_1607_03936_b200"))
import build  # noqa: E402

build.FLAGS += ["-DWB_KPROF"]
build.build(force=True)
import synth  # noqa: E402
from paper_1607_03936_b200 import Context  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C5"
extra = int(sys.argv[2], 0) if len(sys.argv) > 2 else 0
inp = synth.make_inputs(cfg, 0)
c = Context(inp["N"], inp["k"])
d = lambda a: torch.as_tensor(a, dtype=torch.float64, device="cuda")  # noqa: E731
mu, p = d(inp["mu_q"]), d(inp["p"])
pv = torch.empty(c.n_p, dtype=torch.float64, device="cuda")
c.set_viscosity(mu)
iters = 50
c.set_option("k_dbg", 0x4000 | 0x2000 | extra)
c.poisson_pcg(1, p, pv, iters)
c.query("kprof7")  # clear
c.poisson_pcg(1, p, pv, iters)
v = [c.query(f"kprof{k}") for k in range(8)]
c.set_option("k_dbg", 0)
tiles = v[6]
launches = iters
ctas = tiles / launches / ((inp["N"] // 4) * (inp["N"] // 8) * (inp["N"] // 8)) * 148 if tiles else 0
names = ["prologue/control", "wait p/r/Minv", "step 0 (+bar)", "wait X", "step 1 (+bar)", "step 2 (+bar)", "",
         "TMA issue (thr 0)"]
tot = sum(v[:6]) + v[7]
print(f"tiles {tiles:.0f} over {launches} launches; cycles per tile (thread 0 of each CTA), clock 1.965 GHz")
for k, n in enumerate(names):
    if not n:
        continue
    print(f"  {n:18s} {v[k] / tiles:9.1f} cyc/tile  {100 * v[k] / tot:5.1f} %")
print(f"  per launch per CTA: {tot / (launches * 148):9.0f} cyc = {tot / (launches * 148) / 1965:6.2f} us")
# launch timeline of one PCG iteration (it = 5): %globaltimer per CTA
c.set_option("k_dbg", 0x4000 | 0x2000 | extra)
c.poisson_pcg(1, p, pv, iters)
t = [c.query(f"ktl{k}") for k in range(6)]
c.set_option("k_dbg", 0)
print(f"launch it=5 (ns): span {t[0]:.0f}, CTA entry spread {t[1]:.0f}, mean entry->loop {t[2]:.0f}, "
      f"mean loop {t[3]:.0f}, mean loop end->exit {t[4]:.0f}, exit spread {t[5]:.0f}")
