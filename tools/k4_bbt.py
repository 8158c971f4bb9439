"""C4 B / B^T: the tile kernels (option k4bt 2) against the element kernels + gather (0):
relative l2 of the outputs, and the median time of each apply."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
from paper_1607_03936_b200 import Context  # noqa: E402

d = lambda a: torch.as_tensor(a, dtype=torch.float64, device="cuda")  # noqa: E731
st = torch.cuda.current_stream()
for cfg in ["C4"] + sys.argv[1:]:
    inp = synth.make_inputs(cfg, 0)
    c = Context(inp["N"], inp["k"])
    c.set_viscosity(d(inp["mu_q"]))
    u, p = d(inp["u"]), d(inp["p"])
    res = {}
    for v in (0, 2):
        c.set_option("k4bt", v)
        y, q = torch.empty_like(u), torch.empty_like(p)
        ts = {}
        for name, fn in (("B", lambda: c.apply_B(u, q)), ("BT", lambda: c.apply_BT(p, y))):
            fn()
            tt = []
            for _ in range(21):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(st); fn(); b.record(st); b.synchronize()
                tt.append(a.elapsed_time(b) * 1e3)
            ts[name] = statistics.median(tt)
        res[v] = (y.clone(), q.clone(), ts)
    rel = lambda a, b: float(torch.linalg.norm(a - b) / torch.linalg.norm(b))  # noqa: E731
    print(cfg, "rel BT", rel(res[2][0], res[0][0]), "rel B", rel(res[2][1], res[0][1]),
          "| element+gather", res[0][2], "| tile", res[2][2], "us; n_v", c.n_v, flush=True)
