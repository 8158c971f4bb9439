"""C5 (and argv configs) B / B^T cold times: tile / box kernels (bbt_zc 0) against the
z-marching column kernels (bbt_zc 2, 4, 8), with the relative difference of the outputs."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
from paper_1607_03936_b200 import Context  # noqa: E402

d = lambda a: torch.as_tensor(a, dtype=torch.float64, device="cuda")  # noqa: E731
st = torch.cuda.current_stream()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
rel = lambda a, b: float(torch.linalg.norm(a - b) / torch.linalg.norm(b))  # noqa: E731
for cfg in sys.argv[1:] or ["C5", "C3"]:
    inp = synth.make_inputs(cfg, 0)
    c = Context(inp["N"], inp["k"])
    c.set_viscosity(d(inp["mu_q"]))
    u, p = d(inp["u"]), d(inp["p"])
    ref = None
    for cz in (0, 2, 4, 8):
        c.set_option("bbt_zc", cz)
        y, q = torch.empty_like(u), torch.empty_like(p)
        ts = {}
        for name, fn in (("B", lambda: c.apply_B(u, q)), ("BT", lambda: c.apply_BT(p, y))):
            fn()
            tt = []
            for _ in range(21):
                flush.zero_()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(st); fn(); b.record(st); b.synchronize()
                tt.append(a.elapsed_time(b) * 1e3)
            ts[name] = round(statistics.median(tt), 2)
        if ref is None:
            ref = (y.clone(), q.clone())
        print(cfg, "bbt_zc", cz, ts, "us; rel BT", rel(y, ref[0]), "rel B", rel(q, ref[1]), flush=True)
