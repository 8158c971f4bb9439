"""TMA Poisson kernel: its two box variants (kz = 1: z box, kz = 0: r + Minv boxes),
bitwise equality and per-iteration time.  (Contexts of the TMA kernel store the PCG
vectors y fastest; the pointer kernel serves the other contexts.)"""
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
c.set_viscosity(mu)
st = torch.cuda.current_stream()
res = {}
for tma in (0, 1):  # here: the kz option
    c.set_option("kz", tma)
    out = torch.empty(c.n_p, dtype=torch.float64, device="cuda")
    c.apply_K(1, p, out)
    k = out.clone()
    c.poisson_pcg(1, p, out, 20)
    torch.cuda.synchronize()
    res[tma] = (k, out.clone())

    def t_us(it, reps=7):
        c.poisson_pcg(1, p, out, it)
        ts = []
        for _ in range(reps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(st); c.poisson_pcg(1, p, out, it); b.record(st); b.synchronize()
            ts.append(a.elapsed_time(b))
        return statistics.median(ts) * 1e3
    per = (t_us(50) - t_us(10)) / 40
    print(f"kz={tma}: per PCG iteration {per:.2f} us", flush=True)
print("K bitwise equal (expected):", torch.equal(res[0][0], res[1][0]),
      "max rel diff", float(((res[0][0] - res[1][0]).abs().max() / res[0][0].abs().max())))
print("PCG20 bitwise equal:", torch.equal(res[0][1], res[1][1]),
      "max rel diff", float(((res[0][1] - res[1][1]).abs().max() / res[0][1].abs().max())))
