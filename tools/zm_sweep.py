"""Per-iteration PCG time at C5 for the z-march kernel variants and chunk lengths
(graph replays, (t(50) - t(10)) / 40), against the TMA kernel."""
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
c.set_viscosity(d(inp["mu_q"]))
p = d(inp["p"])
pv = torch.empty(c.n_p, dtype=torch.float64, device="cuda")
st = torch.cuda.current_stream()


def timed(fn, reps=7):
    fn()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st); fn(); b.record(st); b.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts) * 1e3


def per_iter():
    t10 = timed(lambda: c.poisson_pcg(1, p, pv, 10))
    t50 = timed(lambda: c.poisson_pcg(1, p, pv, 50))
    return (t50 - t10) / 40


c.set_option("k_zm", 0)
print(f"tma: {per_iter():.2f} us/iter", flush=True)
c.set_option("k_zm", 1)
ref = None
vs = [int(a) for a in sys.argv[2:]] or list(range(5))
for v in vs:
    c.set_option("zm_var", v)
    for zc in (4, 6, 8, 16):
        c.set_option("zm_zc", zc)
        x = c.poisson_pcg(1, p, pv, 10).clone()
        if ref is None:
            ref = x
        err = float((x - ref).norm() / ref.norm())
        print(f"var {v} zc {zc}: {per_iter():.2f} us/iter (vs var0 {err:.1e})", flush=True)
