"""Parity + timing of the node-owner z-march Poisson kernel (k_zm) against the TMA kernel.
usage: python tools/zm_check.py [N ...]"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from tests.gpu_common import Pair, dev, empty, host, rel_l2  # noqa: E402

Ns = [int(a) for a in sys.argv[1:]] or [44, 46, 64]
st = torch.cuda.current_stream()


def timed(fn, reps=10):
    fn()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st); fn(); b.record(st); b.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts) * 1e3


for N in Ns:
    P = Pair("C5", N=N)
    c, o, s = P.ctx, P.o, P.ost
    b = P.inp["p"]
    print(f"N={N} k_zm available: {c.query('k_zm')}", flush=True)
    for zm in (1, 0):
        c.set_option("k_zm", zm)
        for side, X in ((0, s["Cinv"]), (1, s["Dinv"])):
            q = host(c.apply_K(side, dev(b), empty(c.n_p)))
            print(f"  zm={zm} side={side} apply_K rel {rel_l2(q, o.apply_K(X, b)):.2e}")
        for it in (1, 5, 20):
            x = host(c.poisson_pcg(1, dev(b), empty(c.n_p), it))
            print(f"  zm={zm} pcg{it} rel {rel_l2(x, o.poisson(s['Dinv'], s['diagKr'], b, it)):.2e}", flush=True)
    pv = empty(c.n_p)
    bd = dev(b)
    for zm, zc in ((0, 4), (1, 2), (1, 3), (1, 4), (1, 6), (1, 8)):
        c.set_option("k_zm", zm)
        c.set_option("zm_zc", zc)
        t10 = timed(lambda: c.poisson_pcg(1, bd, pv, 10))
        t50 = timed(lambda: c.poisson_pcg(1, bd, pv, 50))
        c.set_option("profile", 1)
        c.poisson_pcg(1, bd, pv, 20)
        kms = c.query("prof_k_ms") / c.query("prof_k_count")
        c.set_option("profile", 0)
        print(f"  zm={zm} zc={zc}: per-iter {(t50 - t10) / 40:.2f} us, K kernel (event pair) {kms * 1e3:.2f} us",
              flush=True)
    c.set_option("k_zm", 1)
    c.set_option("zm_zc", 4)
    x1 = host(c.poisson_pcg(1, bd, pv, 10))
    for _ in range(3):
        assert np.array_equal(host(c.poisson_pcg(1, bd, pv, 10)), x1)
    print("  bitwise repeat ok")
