"""Per-config throughput on one GPU (BASELINE.json configs C1-C5): A, B, B^T GDOF/s
(n_v / apply time, L2 flushed before each rep, median of 30) with the HBM fraction of
their algorithmic bytes, and wBFBT applies/s at the config's PCG
count.  Writes one JSON object per config to stdout."""
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import synth  # noqa: E402
from paper_1607_03936_b200 import Context  # noqa: E402

hbm = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device="cuda")
st = torch.cuda.current_stream()


def timed(fn, reps=30):
    fn()
    ts = []
    for _ in range(reps):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st); fn(); b.record(st); b.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts) * 1e-3  # s


for cfg in sys.argv[1:] or ["C1", "C2", "C3", "C4", "C5"]:
    inp = synth.make_inputs(cfg, 0)
    c = Context(inp["N"], inp["k"])
    d = lambda a: torch.as_tensor(a, dtype=torch.float64, device="cuda")  # noqa: E731
    mu, u, p = d(inp["mu_q"]), d(inp["u"]), d(inp["p"])
    c.set_viscosity(mu)
    yv = torch.empty(c.n_v, dtype=torch.float64, device="cuda")
    pv = torch.empty(c.n_p, dtype=torch.float64, device="cuda")
    iters = synth.CONFIGS[cfg].iters
    tA = timed(lambda: c.apply_A(u, yv))
    tB = timed(lambda: c.apply_B(u, pv))
    tBT = timed(lambda: c.apply_BT(p, yv))
    tW = timed(lambda: c.apply_wbfbt(p, pv, iters), reps=5)
    bA = 8 * (c.n_el * c.n_q + 2 * c.n_v)
    bB = 8 * (c.n_v + c.n_p)
    print(json.dumps({"config": cfg, "N": inp["N"], "k": inp["k"], "n_v": c.n_v, "pcg_iters": iters,
                      "A_gdofs": c.n_v / tA / 1e9, "A_us": tA * 1e6, "A_hbm_frac": bA / tA / 1e9 / hbm,
                      "B_gdofs": c.n_v / tB / 1e9, "B_hbm_frac": bB / tB / 1e9 / hbm,
                      "BT_gdofs": c.n_v / tBT / 1e9, "BT_hbm_frac": bB / tBT / 1e9 / hbm,
                      "wbfbt_applies_per_s": 1.0 / tW, "wbfbt_ms": tW * 1e3}), flush=True)
    c.close()
