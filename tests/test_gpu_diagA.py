"""GPU parity of diag(A) and the Chebyshev-Jacobi smoother on A (reading R18; the
paper's smoother for the viscous block) against the oracle
(tests/test_oracle_diagA.py pins it)."""
import numpy as np
import pytest

from tests.gpu_common import Pair, dev, empty, host, rel_l2

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("cfg,N", [("C1", None), ("C2", 8), ("C4", 4), ("C5", 20)])
def test_diagA_matches_oracle(cfg, N):
    p = Pair(cfg, N=N)
    got = host(p.ctx.get_diagA(empty(p.ctx.n_v)))
    ref = p.o.diag_A(p.inp["mu_q"])
    # a sum of positive element terms: the single-apply bar of north_star, entrywise
    assert np.max(np.abs(got - ref) / np.maximum(np.abs(ref), 1e-300)) <= 1e-12
    assert np.array_equal(got == 0.0, ref == 0.0)


@pytest.mark.parametrize("cfg,N,iters", [("C1", None, 5), ("C2", 8, 8), ("C4", 4, 4)])
def test_velocity_cheb_and_eigmax_match_oracle(cfg, N, iters):
    p = Pair(cfg, N=N)
    mu = p.inp["mu_q"]
    v0 = np.random.default_rng(3).standard_normal(p.ctx.n_v)
    for steps in (1, 6):
        ref = p.o.velocity_eigmax(mu, v0, steps)
        got = p.ctx.velocity_eigmax(dev(v0), steps)
        assert abs(got - ref) <= 1e-11 * ref   # each step one A apply (1e-11 bar)
    lam = p.o.velocity_eigmax(mu, v0, 15)
    b = np.random.default_rng(4).uniform(-1, 1, p.ctx.n_v)
    ref = p.o.velocity_cheb(mu, b, iters, 0.1 * lam, 1.1 * lam)
    got = host(p.ctx.velocity_cheb(dev(b), empty(p.ctx.n_v), iters, 0.1 * lam, 1.1 * lam))
    assert rel_l2(got, ref) <= 1e-11
    # Dirichlet dofs stay 0
    assert np.all(got[ref == 0.0] == 0.0)


def test_velocity_cheb_reduces_residual_and_rejects_bad_input():
    from paper_1607_03936_b200 import WBError
    p = Pair("C2")
    mu = p.inp["mu_q"]
    v0 = np.random.default_rng(5).standard_normal(p.ctx.n_v)
    lam = p.ctx.velocity_eigmax(dev(v0), 50)
    mask = p.o.boundary_mask().astype(bool)
    b = np.where(mask, 0.0, np.random.default_rng(6).uniform(-1, 1, p.ctx.n_v))
    res = []
    for it in (2, 8, 24):
        x = host(p.ctx.velocity_cheb(dev(b), empty(p.ctx.n_v), it, 0.1 * lam, 1.1 * lam))
        res.append(np.linalg.norm(b - p.o.apply_A(mu, x)) / np.linalg.norm(b))
    assert res[0] > res[1] > res[2]
    for lo, hi in ((0.0, 1.0), (2.0, 1.0)):
        with pytest.raises(WBError):
            p.ctx.velocity_cheb(dev(b), empty(p.ctx.n_v), 2, lo, hi)
    bb = dev(b)
    with pytest.raises(WBError):
        p.ctx.velocity_cheb(bb, bb, 2, 0.1, 1.0)
