"""GPU parity of the Chebyshev-accelerated Jacobi solve and its power iteration
(reading R16) against the oracle (tests/test_oracle_cheb.py pins
it), through the C ABI.  Chebyshev is a fixed polynomial filter, so the two sides
agree to rounding at every iteration count (unlike CG, R15)."""
import numpy as np
import pytest

from tests.gpu_common import Pair, dev, empty, host, rel_l2

pytestmark = pytest.mark.gpu


def _interval(p, side, steps=30):
    """PETSc-style smoother interval [0.1, 1.1] x the oracle's power-iteration estimate (R16)."""
    X, d = (p.ost["Cinv"], p.ost["diagKl"]) if side == 0 else (p.ost["Dinv"], p.ost["diagKr"])
    v0 = np.random.default_rng(11).standard_normal(p.o.n_p)
    lam = p.o.poisson_eigmax(X, d, v0, steps)
    return 0.1 * lam, 1.1 * lam, X, d, v0


@pytest.mark.parametrize("cfg,N,iters", [("C1", None, 6), ("C2", 8, 12), ("C2", None, 20), ("C3", 12, 15),
                                         ("C4", 4, 10), ("C5", 44, 10)])
def test_cheb_matches_oracle(cfg, N, iters):
    p = Pair(cfg, N=N)
    b = p.inp["p"]
    for side in (0, 1):
        lmin, lmax, X, d, _ = _interval(p, side)
        ref = p.o.poisson_cheb(X, d, b, iters, lmin, lmax)
        got = host(p.ctx.poisson_cheb(side, dev(b), empty(p.ctx.n_p), iters, lmin, lmax))
        assert np.all(np.isfinite(got))
        # indefinite K_w (nonpositive lumped entries, C1) lies partly outside the interval,
        # where the filter grows: there the bar is rounding relative to that growth
        tol = 1e-11 if (p.ost["n_nonpos_Cw"] == 0 and p.ost["n_nonpos_Dw"] == 0) else 1e-9
        assert rel_l2(got, ref) <= tol, (side, rel_l2(got, ref))
        assert abs(got[::p.ctx.n_p // p.ctx.n_el].sum()) <= 1e-10 * np.abs(got).max() * p.ctx.n_el  # projected


@pytest.mark.parametrize("cfg,N", [("C1", None), ("C2", 8), ("C4", 4), ("C5", 44)])
def test_eigmax_matches_oracle(cfg, N):
    p = Pair(cfg, N=N)
    for side in (0, 1):
        X, d = (p.ost["Cinv"], p.ost["diagKl"]) if side == 0 else (p.ost["Dinv"], p.ost["diagKr"])
        v0 = np.random.default_rng(side).standard_normal(p.o.n_p)
        for steps in (1, 7, 25):
            ref = p.o.poisson_eigmax(X, d, v0, steps)
            got = p.ctx.poisson_eigmax(side, dev(v0), steps)
            # each step is one K_w apply, whose bar is north_star's single-apply 1e-11
            assert abs(got - ref) <= 1e-11 * abs(ref), (side, steps, got, ref)


def test_cheb_zero_iters_and_edge_cases():
    p = Pair("C2", N=6)
    b = p.inp["p"]
    lmin, lmax, X, d, v0 = _interval(p, 1)
    # 0 steps: x = P 0 = 0 (as the oracle)
    got = host(p.ctx.poisson_cheb(1, dev(b), empty(p.ctx.n_p), 0, lmin, lmax))
    assert np.array_equal(got, np.zeros(p.ctx.n_p))
    assert p.ctx.poisson_eigmax(1, dev(v0), 0) == 0.0
    assert p.ctx.poisson_eigmax(1, dev(np.zeros(p.ctx.n_p)), 5) == 0.0
    # constant b: projected to 0, so x = 0
    got = host(p.ctx.poisson_cheb(1, dev(np.tile([1.0, 0, 0, 0], p.ctx.n_el)), empty(p.ctx.n_p), 5, lmin, lmax))
    assert np.abs(got).max() <= 1e-13
    # linear in b (a fixed filter) on the GPU as well
    rng = np.random.default_rng(4)
    b1, b2 = rng.uniform(-1, 1, p.ctx.n_p), rng.uniform(-1, 1, p.ctx.n_p)
    f = lambda v: host(p.ctx.poisson_cheb(1, dev(v), empty(p.ctx.n_p), 8, lmin, lmax))  # noqa: E731
    lhs, rhs = f(2 * b1 - 3 * b2), 2 * f(b1) - 3 * f(b2)
    assert rel_l2(lhs, rhs) <= 1e-12
    # bad intervals and arguments are rejected
    from paper_1607_03936_b200 import WBError
    for lo, hi in ((0.0, 1.0), (-1.0, 1.0), (2.0, 1.0), (1.0, 1.0), (1.0, float("inf")), (float("nan"), 1.0)):
        with pytest.raises(WBError):
            p.ctx.poisson_cheb(1, dev(b), empty(p.ctx.n_p), 3, lo, hi)
    with pytest.raises(WBError):
        p.ctx.poisson_cheb(2, dev(b), empty(p.ctx.n_p), 3, lmin, lmax)
    with pytest.raises(WBError):
        p.ctx.poisson_eigmax(0, dev(v0), -1)
    bb = dev(b)
    with pytest.raises(WBError):
        p.ctx.poisson_cheb(1, bb, bb, 3, lmin, lmax)


def test_cheb_residual_decreases_with_exact_interval():
    """Quality check: with the interval from a converged power iteration the relative
    residual of the projected solve falls with the iteration count (C2 at its N = 16:
    positive D_w, so K_r is semi-definite; coarser C2 meshes have nonpositive lumped
    entries and an indefinite K_r, where a Chebyshev interval cannot hold the spectrum)."""
    p = Pair("C2")
    assert p.ost["n_nonpos_Dw"] == 0
    b = p.o.project(p.inp["p"])
    X, d = p.ost["Dinv"], p.ost["diagKr"]
    v0 = np.random.default_rng(2).standard_normal(p.o.n_p)
    lam = p.ctx.poisson_eigmax(1, dev(v0), 300)
    assert abs(lam - p.o.poisson_eigmax(X, d, v0, 300)) <= 1e-11 * lam
    res = []
    for it in (5, 20, 60):
        x = host(p.ctx.poisson_cheb(1, dev(b), empty(p.ctx.n_p), it, 0.1 * lam, 1.1 * lam))
        res.append(p.o.poisson_relres(X, b, x))
    assert res[0] > res[1] > res[2]


@pytest.mark.parametrize("cfg,N,iters", [("C1", None, 6), ("C2", 8, 10), ("C3", 12, 10), ("C4", 4, 8), ("C5", 44, 10)])
def test_wbfbt_with_cheb_inner_matches_oracle(cfg, N, iters):
    """wBFBT with Chebyshev-Jacobi inner solves (wb_set_inner_cheb, R16): a linear map, so
    parity is rounding-level (1e-10; 1e-8 where K_w is indefinite)."""
    p = Pair(cfg, N=N)
    lo_l, hi_l, _, _, _ = _interval(p, 0)
    lo_r, hi_r, _, _, _ = _interval(p, 1)
    p.ctx.set_inner_cheb(lo_l, hi_l, lo_r, hi_r)
    assert p.ctx.query("inner") == 1
    b = p.inp["p"]
    ref = p.o.wbfbt_cheb(b, iters, lo_l, hi_l, lo_r, hi_r)
    got = host(p.ctx.apply_wbfbt(dev(b), empty(p.ctx.n_p), iters))
    definite = p.ost["n_nonpos_Cw"] == 0 and p.ost["n_nonpos_Dw"] == 0
    assert rel_l2(got, ref) <= (1e-10 if definite else 1e-8), rel_l2(got, ref)
    # the hot-path entry uses the same inner solves
    yA, pB = empty(p.ctx.n_v), empty(p.ctx.n_p)
    yBT, z = empty(p.ctx.n_v), empty(p.ctx.n_p)
    p.ctx.hotpath(p.mu, dev(p.inp["u"]), dev(b), iters, yA, pB, yBT, z)
    assert np.array_equal(host(z), got)
    p.ctx.set_inner_cheb()
    assert p.ctx.query("inner") == 0
    from paper_1607_03936_b200 import WBError
    with pytest.raises(WBError):
        p.ctx.set_inner_cheb(1.0, 0.5, 0.1, 1.0)
