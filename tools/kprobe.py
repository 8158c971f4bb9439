"""Phase timing probe of the fused K kernel (option k_dbg; results invalid):
per-iteration time of the graph-replayed PCG loop, (t(50) - t(10)) / 40."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
from paper_1607_03936_b200 import Context  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C5"
inp = synth.make_inputs(cfg, 0)
c = Context(inp["N"], inp["k"])
d = lambda a: torch.as_tensor(a, dtype=torch.float64, device="cuda")  # noqa: E731
mu, p = d(inp["mu_q"]), d(inp["p"])
pv = torch.empty(c.n_p, dtype=torch.float64, device="cuda")
c.set_viscosity(mu)
st = torch.cuda.current_stream()


def t_us(it, reps=7):
    c.poisson_pcg(1, p, pv, it)
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st); c.poisson_pcg(1, p, pv, it); b.record(st); b.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts) * 1e3


probes = [("full", 0), ("no step1", 0x100), ("no step2", 0x200), ("no halo loads", 0x400), ("no step1+2", 0x300),
          ("only control+Xs+store", 0x700), ("no q+pnew store", 0x1800), ("empty (no Xs, no ctl)", 0xc700),
          ("full - Xs", 0x4000)]
if len(sys.argv) > 2:
    probes = probes[:1]
for kv in ((0, 1) if len(sys.argv) <= 2 else (0,)):
    c.set_option("k_variant", kv)
    for name, dbg in probes:
        c.set_option("k_dbg", dbg | 0x2000)  # 0x2000: never stop (probe)
        per = (t_us(50) - t_us(10)) / 40
        print(f"kvar={kv} {name:24s}: per PCG iteration {per:7.2f} us")
c.set_option("k_dbg", 0)
print("occupancy CTAs/SM: K2", c.query("occ_k2"), "A", c.query("occ_a2"))
