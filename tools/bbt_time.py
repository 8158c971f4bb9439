"""Cold B / B^T timings and bitwise self-consistency (for kernel A/B builds)."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from tests.gpu_common import Pair, dev, empty, host, rel_l2  # noqa: E402

st = torch.cuda.current_stream()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")


def timed(fn, reps=30):
    fn()
    ts = []
    for _ in range(reps):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st); fn(); b.record(st); b.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts) * 1e3


for cfg, N in (("C2", 7), ("C5", 45), ("C5", None)):
    P = Pair(cfg, N)
    c = P.ctx
    u, p = dev(P.inp["u"]), dev(P.inp["p"])
    yb, pb = empty(c.n_v), empty(c.n_p)
    eB = rel_l2(host(c.apply_B(u, pb)), P.o.apply_B(P.inp["u"]))
    eBT = rel_l2(host(c.apply_BT(p, yb)), P.o.apply_BT(P.inp["p"]))
    tB = timed(lambda: c.apply_B(u, pb))
    tBT = timed(lambda: c.apply_BT(p, yb))
    nbytes = 8 * (c.n_v + c.n_p)
    print(f"{cfg} N={P.N}: B {tB:.1f} us ({nbytes / tB / 1e3:.0f} GB/s, err {eB:.1e}), "
          f"BT {tBT:.1f} us ({nbytes / tBT / 1e3:.0f} GB/s, err {eBT:.1e})", flush=True)
