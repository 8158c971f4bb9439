"""Shared helpers of the -m gpu parity tests: run the CUDA path (through the
C ABI via the thin binding) and the CPU oracle on the same seeded inputs."""
from __future__ import annotations

import numpy as np

import synth


def rel_l2(a, b) -> float:
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    nb = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (nb if nb > 0 else 1.0))


def dev(x):
    import torch
    return torch.as_tensor(np.ascontiguousarray(x), dtype=torch.float64, device="cuda")


def host(t) -> np.ndarray:
    return t.detach().cpu().numpy()


def empty(n, dtype=None):
    import torch
    return torch.empty(n, dtype=dtype or torch.float64, device="cuda")


# k = 3 (accepted by wb_create; not a BASELINE config): the C1 recipe with Q3 x P2disc.
K3 = synth.Config("K3", 6, 3, 4, 200.0, 0.1, 1e-2, 1e2, 20)


class Pair:
    """One (config, N, seed) case: inputs, a GPU context and an oracle."""

    def __init__(self, cfg: str, N: int | None = None, seed: int = 0, a_l=1.0, a_r=1.0, flags=0, setup=True):
        from oracle import Oracle
        from paper_1607_03936_b200 import Context
        self.cfg = synth.CONFIGS[cfg] if isinstance(cfg, str) else cfg
        self.inp = synth.make_inputs(self.cfg, seed, N=N)
        self.N, self.k = self.inp["N"], self.inp["k"]
        self.ctx = Context(self.N, self.k, flags=flags)
        self.o = Oracle(self.N, self.k)
        self.a_l, self.a_r = a_l, a_r
        self.mu = dev(self.inp["mu_q"])
        if setup:
            self.ctx.set_viscosity(self.mu, a_l, a_r)
            self.ost = self.o.setup(self.inp["mu_q"], a_l, a_r)

    def gpu(self, name, *args):
        return getattr(self.ctx, name)(*args)
