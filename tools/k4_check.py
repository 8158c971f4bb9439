"""Fused k = 3, 4 Poisson kernel (k4_fused.cuh) against the B^T / gather / B kernels it
replaces: K_w applies and PCG prefixes on small, ragged and full C4 meshes (relative l2),
then per-iteration PCG time and wBFBT applies/s at C4 for every tile variant."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_1607_03936_b200 import Context  # noqa: E402

K3 = synth.Config("K3", 6, 3, 4, 200.0, 0.1, 1e-2, 1e2, 20)
d = lambda a: torch.as_tensor(a, dtype=torch.float64, device="cuda")  # noqa: E731
rel = lambda a, b: float(torch.linalg.norm(a - b) / torch.linalg.norm(b))  # noqa: E731
st = torch.cuda.current_stream()

for cfg, N in [("C4", 1), ("C4", 2), ("C4", 3), ("C4", 5), ("C4", 8), ("C4", 12), ("C4", None), (K3, None), (K3, 3),
               (K3, 7)]:
    inp = synth.make_inputs(synth.CONFIGS[cfg] if isinstance(cfg, str) else cfg, 0, N=N)
    c = Context(inp["N"], inp["k"])
    c.set_viscosity(d(inp["mu_q"]))
    p = d(inp["p"])
    out = {}
    for var in ([None, 0, 1, 2, 3, 4, 5, 6, 7, 8, 9] if inp["k"] == 4 else [None, 0, 1]):
        if var is None:
            c.set_option("k4f", 0)
        else:
            c.set_option("k4f", 1)
            c.set_option("k4_var", var)
        q0, q1 = torch.empty_like(p), torch.empty_like(p)
        c.apply_K(0, p, q0)
        c.apply_K(1, p, q1)
        x = torch.empty_like(p)
        c.poisson_pcg(1, p, x, 5)
        torch.cuda.synchronize()
        out[var] = (q0.clone(), q1.clone(), x.clone())
    ref = out[None]
    errs = {v: max(rel(o[0], ref[0]), rel(o[1], ref[1]), rel(o[2], ref[2])) for v, o in out.items() if v is not None}
    print(f"{getattr(cfg, 'name', cfg)} N={inp['N']} k={inp['k']}: max rel vs unfused (K_l, K_r, PCG5) "
          + " ".join(f"v{v}={e:.2e}" for v, e in errs.items()), flush=True)

inp = synth.make_inputs("C4", 0)
c = Context(inp["N"], inp["k"])
c.set_viscosity(d(inp["mu_q"]))
p = d(inp["p"])
x = torch.empty_like(p)


def t_us(fn, reps=9):
    fn()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st); fn(); b.record(st); b.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts) * 1e3


for var in [None, 0, 1, 2, 3, 4, 5, 6, 7, 8, 9]:
    if var is None:
        c.set_option("k4f", 0)
    else:
        c.set_option("k4f", 1)
        c.set_option("k4_var", var)
    it = (t_us(lambda: c.poisson_pcg(1, p, x, 50)) - t_us(lambda: c.poisson_pcg(1, p, x, 10))) / 40
    k = t_us(lambda: c.apply_K(1, p, x))
    z = torch.empty_like(p)
    w = t_us(lambda: c.apply_wbfbt(p, z, 50))
    print(f"C4 variant {var}: PCG iteration {it:.2f} us, K apply (with transposes) {k:.2f} us, "
          f"wBFBT(50) {w:.1f} us = {1e6 / w:.0f} applies/s", flush=True)
