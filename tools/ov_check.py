"""k_K2_ov (overlapped element step) vs k_K2_tma: bitwise equality of PCG results and of
apply_K at C5 and ragged N, and the per-iteration time of each (tools/opt_ab.py method)."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
from paper_1607_03936_b200 import Context  # noqa: E402

d = lambda a: torch.as_tensor(a, dtype=torch.float64, device="cuda")  # noqa: E731
for N in (44, 46, 64):
    inp = synth.make_inputs("C5", 0, N=N)
    c = Context(inp["N"], inp["k"])
    c.set_viscosity(d(inp["mu_q"]))
    p = d(inp["p"])
    outs = {}
    for kov in (0, 1):
        c.set_option("k_ov", kov)
        assert c.query("k_ov") == kov
        x = torch.empty(c.n_p, dtype=torch.float64, device="cuda")
        c.poisson_pcg(1, p, x, 30)
        qk = torch.empty_like(x)
        c.apply_K(0, p, qk)
        outs[kov] = (x.clone(), qk.clone())
    same = all(torch.equal(a, b) for a, b in zip(outs[0], outs[1]))
    print(f"N={N}: bitwise equal (PCG 30 its, apply_K): {same}  max|dx|={float((outs[0][0]-outs[1][0]).abs().max()):.2e}")
    st = torch.cuda.current_stream()

    def t_us(it):
        ts = []
        for _ in range(7):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(st); c.poisson_pcg(1, p, x, it); b.record(st); b.synchronize()
            ts.append(a.elapsed_time(b))
        return statistics.median(ts) * 1e3
    for setting in ((0, 0), (1, 0), (0, 1)):
        c.set_option("kz", setting[0]); c.set_option("k_ov", setting[1])
        t_us(10)
        print(f"  kz={setting[0]} k_ov={setting[1]}: {(t_us(50) - t_us(10)) / 40:.2f} us/iter")
    c.set_option("kz", 0); c.set_option("k_ov", 0)
