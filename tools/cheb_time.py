"""Chebyshev-Jacobi inner solve at C5: power-iteration interval,
then per-iteration time from graph replays ((t(50) - t(10)) / 40) and one 30-iteration
solve for an ncu launch list (run under ncu with --metrics gpu__time_duration.sum)."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_1607_03936_b200 import Context  # noqa: E402

inp = synth.make_inputs("C5", 0)
c = Context(inp["N"], inp["k"])
d = lambda a: torch.as_tensor(a, dtype=torch.float64, device="cuda")  # noqa: E731
c.set_viscosity(d(inp["mu_q"]))
p = d(inp["p"])
x = torch.empty(c.n_p, dtype=torch.float64, device="cuda")
v0 = d(np.random.default_rng(7).standard_normal(c.n_p))
lam = c.poisson_eigmax(1, v0, 20)
st = torch.cuda.current_stream()
if os.environ.get("CHEB_ONCE"):
    c.set_option("graph", 0)
    c.poisson_cheb(1, p, x, 30, 0.1 * lam, 1.1 * lam)
    torch.cuda.synchronize()
    sys.exit(0)


def t_us(it, reps=7):
    c.poisson_cheb(1, p, x, it, 0.1 * lam, 1.1 * lam)
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st); c.poisson_cheb(1, p, x, it, 0.1 * lam, 1.1 * lam); b.record(st); b.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts) * 1e3


print(f"lambda_max estimate (20 steps) {lam:.6g}; Chebyshev per iteration {(t_us(50) - t_us(10)) / 40:.2f} us")
