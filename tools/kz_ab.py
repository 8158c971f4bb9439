"""Per PCG iteration time (graph replay, (t(50) - t(10)) / 40) for kz = 0, 1 at C5."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
from paper_1607_03936_b200 import Context  # noqa: E402

inp = synth.make_inputs(sys.argv[1] if len(sys.argv) > 1 else "C5", 0)
c = Context(inp["N"], inp["k"])
d = lambda a: torch.as_tensor(a, dtype=torch.float64, device="cuda")  # noqa: E731
mu, p = d(inp["mu_q"]), d(inp["p"])
pv = torch.empty(c.n_p, dtype=torch.float64, device="cuda")
c.set_viscosity(mu)
st = torch.cuda.current_stream()
reps = int(os.environ.get("KZ_REPS", "7"))


def t_us(it):
    c.poisson_pcg(1, p, pv, it)
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st); c.poisson_pcg(1, p, pv, it); b.record(st); b.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts) * 1e3


res = {}
for kz in (0, 1):
    c.set_option("kz", kz)
    per = (t_us(50) - t_us(10)) / 40
    res[kz] = pv.clone()
    print(f"kz={kz}: per PCG iteration {per:7.2f} us")
print("max rel diff kz0 vs kz1:", float((res[0] - res[1]).abs().max() / res[0].abs().max()))
