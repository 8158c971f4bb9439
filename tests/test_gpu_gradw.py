"""GPU parity of the viscosity-gradient wBFBT weights (rmk:wbfbt-visc-grad,
PAPER.md:2132-2150; reading R17) against the oracle
(tests/test_oracle_gradw.py pins it): option "weights" 1 before wb_set_viscosity."""
import numpy as np
import pytest

from tests.gpu_common import Pair, dev, empty, host, rel_l2

pytestmark = pytest.mark.gpu


def _grad_pair(cfg, N=None, a_l=1.0, a_r=1.0):
    p = Pair(cfg, N=N, setup=False)
    p.ctx.set_option("weights", 1)
    assert p.ctx.query("weights") == 1
    p.ctx.set_viscosity(p.mu, a_l, a_r)
    p.ost = p.o.setup(p.inp["mu_q"], a_l, a_r, weights="grad")
    return p


@pytest.mark.parametrize("cfg,N,a_l,a_r", [("C1", None, 1.0, 1.0), ("C2", None, 2.0, 1.0), ("C3", 12, 1.0, 3.0),
                                           ("C4", 5, 1.0, 1.0), ("C5", 44, 1.0, 1.0)])
def test_grad_weights_lumped_and_jacobi(cfg, N, a_l, a_r):
    p = _grad_pair(cfg, N, a_l, a_r)
    ctx, st = p.ctx, p.ost
    Cw, Dw, Ci, Di = (empty(ctx.n_nodes) for _ in range(4))
    ctx.get_lumped(Cw, Dw, Ci, Di)
    # same bar as the eq:wbfbt weights (test_gpu_parity.test_lumped_and_jacobi)
    for g, o in ((Cw, st["Cw"]), (Dw, st["Dw"])):
        assert np.max(np.abs(host(g) - o)) <= 1e-13 * np.max(np.abs(o))
    # nonpositive counts: a sign is an integer decided by floating point, so compare the
    # signs that are unique -- entries above the rounding band of the lumped sums (on the
    # coarse high-contrast meshes the gradient weights cancel to ~1e-14 of the maximum)
    mask = p.o.boundary_mask()[:ctx.n_nodes] == 0
    for g, o, key in ((Cw, st["Cw"], "n_nonpos_Cw"), (Dw, st["Dw"], "n_nonpos_Dw")):
        gh = host(g)
        band = np.abs(o) <= 1e-12 * np.max(np.abs(o))
        assert np.array_equal((gh <= 0)[mask & ~band], (o <= 0)[mask & ~band])
        lo = int(np.sum((o <= 0) & mask & ~band))
        assert lo <= ctx.query(key) <= lo + int(np.sum(band & mask)), key
        if not np.any(band & mask):
            assert ctx.query(key) == st[key]
    dl, dr = empty(ctx.n_p), empty(ctx.n_p)
    ctx.get_jacobi(dl, dr)
    if st["n_nonpos_Cw"] == 0:
        assert rel_l2(host(dl), st["diagKl"]) <= 1e-12
        assert rel_l2(host(dr), st["diagKr"]) <= 1e-12
    # the weights differ from eq:wbfbt's on a heterogeneous viscosity
    sq = p.o.lumped(p.inp["mu_q"], a_l, a_r)
    assert not np.allclose(st["Cw"], sq["Cw"])


def test_grad_weights_wbfbt_and_A_unchanged():
    """wBFBT with the gradient weights (C2, 20 PCG iterations: prefix-parity range, R15),
    and A still applies mu (its output equals the eq:wbfbt context's bit for bit)."""
    p = _grad_pair("C2")
    b = p.inp["p"]
    z = host(p.ctx.apply_wbfbt(dev(b), empty(p.ctx.n_p), 20))
    assert rel_l2(z, p.o.wbfbt(b, 20)) <= 1e-8
    q = Pair("C2")
    u = dev(p.inp["u"])
    ya, yb = empty(p.ctx.n_v), empty(q.ctx.n_v)
    p.ctx.apply_A(u, ya)
    q.ctx.apply_A(u, yb)
    assert np.array_equal(host(ya), host(yb))
    # back to the default weights on the same context
    p.ctx.set_option("weights", 0)
    p.ctx.set_viscosity(p.mu)
    Cw = empty(p.ctx.n_nodes)
    p.ctx.get_lumped(Cw)
    Cq = empty(q.ctx.n_nodes)
    q.ctx.get_lumped(Cq)
    assert np.array_equal(host(Cw), host(Cq))


def test_weights_option_rejects_bad_values():
    from paper_1607_03936_b200 import WBError
    p = Pair("C1", setup=False)
    for v in (2, -1, 0.5):
        with pytest.raises(WBError):
            p.ctx.set_option("weights", v)
