"""Per PCG iteration time (graph replay, (t(50) - t(10)) / 40) at C5 over option settings.
usage: python tools/opt_ab.py C5 "kz=0,l2win=0" "kz=1,l2win=1" ...   (each argument one setting)"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
from paper_1607_03936_b200 import Context  # noqa: E402

inp = synth.make_inputs(sys.argv[1], 0, N=int(os.environ["AB_N"]) if os.environ.get("AB_N") else None)
c = Context(inp["N"], inp["k"])
d = lambda a: torch.as_tensor(a, dtype=torch.float64, device="cuda")  # noqa: E731
mu, p = d(inp["mu_q"]), d(inp["p"])
pv = torch.empty(c.n_p, dtype=torch.float64, device="cuda")
c.set_viscosity(mu)
st = torch.cuda.current_stream()
reps = int(os.environ.get("AB_REPS", "7"))


def t_us(it):
    c.poisson_pcg(1, p, pv, it)
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st); c.poisson_pcg(1, p, pv, it); b.record(st); b.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts) * 1e3


ref = None
for setting in sys.argv[2:]:
    for kv in setting.split(","):
        k, v = kv.split("=")
        c.set_option(k, float(v))
    per = (t_us(50) - t_us(10)) / 40
    out = pv.clone()
    ref = out if ref is None else ref
    print(f"N={inp['N']} {setting:24s}: per PCG iteration {per:7.2f} us = {per * 1e3 / inp['N'] ** 3:.3f} ns/element"
          f"  (max rel diff vs first {float((out - ref).abs().max() / ref.abs().max()):.1e})")
