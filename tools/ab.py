"""Quick A/B timing of kernel variants on one config (CUDA events, L2 flushed).
usage: python tools/ab.py [C5]"""
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
mu, u, p = d(inp["mu_q"]), d(inp["u"]), d(inp["p"])
f64 = dict(dtype=torch.float64, device="cuda")
yv, pv = torch.empty(c.n_v, **f64), torch.empty(c.n_p, **f64)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
c.set_viscosity(mu)
st = torch.cuda.current_stream()


def timed(fn, reps=20, cold=True):
    fn()
    ts = []
    for _ in range(reps):
        if cold:
            flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st); fn(); b.record(st); b.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts) * 1e3  # us


n_v = c.n_v
tA = timed(lambda: c.apply_A(u, yv))
print(f"A (cold L2): {tA:.1f} us  {n_v / tA / 1e3:.1f} GDOF/s")
print(f"B: {timed(lambda: c.apply_B(u, pv)):.1f} us")
print(f"BT: {timed(lambda: c.apply_BT(p, yv)):.1f} us")
print(f"K (cold): {timed(lambda: c.apply_K(1, p, pv)):.1f} us  K (warm): {timed(lambda: c.apply_K(1, p, pv), cold=False):.1f} us")
for g in (1, 0):
    c.set_option("graph", g)
    t10 = timed(lambda: c.poisson_pcg(1, p, pv, 10), reps=10, cold=False)
    t50 = timed(lambda: c.poisson_pcg(1, p, pv, 50), reps=10, cold=False)
    print(f"graph={g}: pcg10 {t10:.1f} us, pcg50 {t50:.1f} us, per-iter {(t50 - t10) / 40:.2f} us")
c.set_option("graph", 1)
it = synth.CONFIGS[cfg].iters
print(f"wBFBT({it}): {timed(lambda: c.apply_wbfbt(p, pv, it), reps=5, cold=False):.1f} us")
print(f"setup: {timed(lambda: c.set_viscosity(mu), reps=5):.1f} us")
for kv in (0, 1):
    c.set_option("k_variant", kv)
    t10 = timed(lambda: c.poisson_pcg(1, p, pv, 10), reps=10, cold=False)
    t50 = timed(lambda: c.poisson_pcg(1, p, pv, 50), reps=10, cold=False)
    c.set_option("profile", 1)
    c.poisson_pcg(1, p, pv, 20)
    kms = c.query("prof_k_ms") / c.query("prof_k_count")
    c.set_option("profile", 0)
    print(f"k_variant={kv}: per-iter {(t50 - t10) / 40:.2f} us, K kernel {kms*1e3:.2f} us")
