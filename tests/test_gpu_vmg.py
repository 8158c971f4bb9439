"""GPU velocity multigrid (R22) and the full Stokes solve with both multigrids against the
oracle (oracle/mg.VMG, oracle/stokes.StokesOracle), and the paper's comparison of Schur
approximations on a multi-sinker problem (Sec. 3.2, Tables 1-2)."""
import numpy as np
import pytest

import synth
from tests.gpu_common import Pair, dev, empty, host, rel_l2

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", params=[("C2", None), ("C3", None), ("C4", 4)], ids=lambda c: c[0])
def vpair(request):
    from oracle import mg as omg
    cfg, N = request.param
    P = Pair(cfg, N)
    P.ctx.setup_mg(3, P.mu)
    P.vmg = omg.VMG(P.N, P.inp["mu_q"], k=P.k)
    assert P.ctx.query("mg_levels") == len(P.vmg.lev)
    return P


def test_velocity_levels_and_vcycle(vpair):
    P = vpair
    for l, L in enumerate(P.vmg.lev):
        assert abs(P.ctx.query(f"mg_vlambda_{l}") - L["lam"]) <= 1e-10 * L["lam"]
    mask = P.o.boundary_mask().astype(bool)
    b = np.where(mask, 0.0, P.inp["u"])
    x = host(P.ctx.velocity_vcycle(dev(b), empty(P.ctx.n_v)))
    assert rel_l2(x, P.vmg.vcycle(b)) <= 1e-10
    assert np.all(x[mask] == 0.0)


def _forcing(P):
    c = P.cfg
    return synth.forcing_at_quadrature(P.N, P.k, P.inp["centers"], c.delta, c.omega)


@pytest.mark.parametrize("cfg,N", [("C2", None), ("C4", 4)])
def test_stokes_full_mg_matches_oracle(cfg, N):
    """FGMRES, 4 iterations, At^-1 = one velocity V-cycle, wBFBT with MG-PCG(3) inner solves:
    GPU vs oracle <= 1e-8 (C4: both hierarchies start with the spectral level)."""
    from oracle import mg as omg
    from oracle import stokes as ost
    P = Pair(cfg, N)
    c = P.ctx
    c.setup_mg(3, P.mu)
    c.set_inner_mg(3)
    c.set_velocity_mg(1)
    f = host(c.load_vector(dev(_forcing(P)), empty(c.n_v)))
    g = np.zeros(c.n_p)
    u, p = empty(c.n_v), empty(c.n_p)
    _, _, it, rr = c.stokes_fgmres(dev(f), dev(g), u, p, 10, 4, 0.0, 10, 6, 1.0, 2.0)
    mu = P.inp["mu_q"]
    ml, mr = omg.MG(P.N, P.ost["Cw"], k=P.k), omg.MG(P.N, P.ost["Dw"], k=P.k)
    V = omg.VMG(P.N, mu, k=P.k)
    so = ost.StokesOracle(P.o, mu, lambda b: omg.wbfbt_mg(P.o, mu, P.ost, ml, mr, b, 3), 6, 1.0, 2.0,
                          ainv=lambda a: V.cycles(a, 1))
    uo, po, ito, rro = so.solve(f, g, 10, 4, 0.0)
    assert it == ito == 4
    assert rel_l2(host(u), uo) <= 1e-8 and rel_l2(host(p), po) <= 1e-8
    assert abs(rr - rro) <= 1e-8 * rro


def _solve(cfg, schur, inner_mg=8, cycles=2, max_iters=300, N=None, restart=200):
    P = Pair(cfg, N, setup=False)
    c = P.ctx
    c.set_schur(schur)
    c.set_viscosity(P.mu)
    c.setup_mg(3, P.mu)
    c.set_velocity_mg(cycles)
    if schur == 0:
        c.set_inner_mg(inner_mg)
    f = c.load_vector(dev(_forcing(P)), empty(c.n_v))
    g = empty(c.n_p).zero_()
    u, p = empty(c.n_v), empty(c.n_p)
    _, _, it, rr = c.stokes_fgmres(f, g, u, p, restart, max_iters, 1e-6, 10, 6, 1.0, 2.0)
    return it, rr


def test_stokes_converges_and_wbfbt_beats_mp():
    """C2 (16^3, 8 sinkers, DR 1e6) with the multi-sinker forcing: with both multigrids the
    solve reaches the paper's 1e-6 reduction, and wBFBT needs fewer
    FGMRES iterations than M_p(1/mu) (Sec. 3.2: M_p degrades with many sinkers and
    high dynamic ratio, wBFBT stays robust)."""
    res = {k: _solve("C2", k) for k in (0, 2)}
    print("C2 FGMRES iterations to 1e-6: wBFBT", res[0], " M_p(1/mu)", res[2])
    assert res[0][1] <= 1e-6
    assert res[0][0] < res[2][0]


def test_stokes_c5_converges_and_wbfbt_beats_mp():
    """The headline mesh C5 (64^3, 24 sinkers, DR 1e10) reaches the 1e-6 reduction with wBFBT
    (2 velocity V-cycles as At^-1, MG-PCG(8) inner Poisson solves; measured 63 iterations)
    well before M_p(1/mu), which has not reached it after the same number of iterations."""
    it, rr = _solve("C5", 0, max_iters=300)
    print("C5 FGMRES iterations to 1e-6 (wBFBT, MG inner, 2 velocity V-cycles):", it, rr)
    assert rr <= 1e-6
    it_mp, rr_mp = _solve("C5", 2, max_iters=it)
    print("C5 M_p(1/mu) after", it_mp, "iterations: relres", rr_mp)
    assert rr_mp > 10 * rr


def test_stokes_c4_converges_with_spectral_levels():
    """C4 (24^3, Q4 x P3disc, DR 1e6): with the spectral level in both multigrids the solve
    reaches the 1e-6 reduction."""
    it, rr = _solve("C4", 0, max_iters=300)
    print("C4 FGMRES iterations to 1e-6 (wBFBT, MG inner, 2 velocity V-cycles):", it, rr)
    assert rr <= 1e-6


def test_stokes_restart_growth():
    """A later solve with a longer restart than an earlier one (the FGMRES work arrays grow)."""
    P = Pair("C2", N=6)
    c = P.ctx
    f = dev(np.where(P.o.boundary_mask().astype(bool), 0.0, P.inp["u"]))
    g = empty(c.n_p).zero_()
    u, p = empty(c.n_v), empty(c.n_p)
    for m in (3, 40):
        _, _, it, rr = c.stokes_fgmres(f, g, u, p, m, 45, 0.0, 5, 2, 1.0, 2.0)
        assert it == 45 and np.isfinite(rr)
