"""GPU pressure multigrid (R20) against the oracle (oracle/mg.py):
level weights, Chebyshev intervals, one V-cycle, MG-PCG prefixes and wBFBT with MG inner
solves, plus the mesh-independent convergence the paper claims."""
import numpy as np
import pytest

from tests.gpu_common import Pair, dev, empty, host, rel_l2

pytestmark = pytest.mark.gpu

CASES = [("C2", None), ("C3", None), ("C1", None), ("C2", 8), ("C4", 8), ("C4", None)]


@pytest.fixture(scope="module", params=CASES, ids=lambda c: f"{c[0]}-N{c[1]}")
def mgpair(request):
    from oracle import mg as omg
    cfg, N = request.param
    P = Pair(cfg, N)
    P.ctx.setup_mg(3)
    P.mg_l = omg.MG(P.N, P.ost["Cw"], k=P.k)
    P.mg_r = omg.MG(P.N, P.ost["Dw"], k=P.k)
    return P


def test_levels_weights_and_intervals(mgpair):
    P = mgpair
    c = P.ctx
    assert int(c.query("mg_levels")) == len(P.mg_r.levels)
    for l, (Ll, Lr) in enumerate(zip(P.mg_l.levels, P.mg_r.levels)):
        assert int(c.query(f"mg_N_{l}")) == Lr.N and int(c.query(f"mg_k_{l}")) == Lr.o.k
        n = (Lr.o.k * Lr.N + 1) ** 3
        Cg, Dg = empty(n), empty(n)
        c.mg_get_lumped(l, Cg, Dg)
        for g, o in ((Cg, Ll.C), (Dg, Lr.C)):
            assert np.max(np.abs(host(g) - o)) <= 1e-14 * np.max(np.abs(o))
        assert int(c.query(f"mg_nonpos_0_{l}")) == Ll.n_nonpos
        assert int(c.query(f"mg_nonpos_1_{l}")) == Lr.n_nonpos
        if l < len(P.mg_r.levels) - 1 and Lr.n_nonpos == 0:
            assert abs(c.query(f"mg_lambda_1_{l}") - Lr.lam) <= 1e-10 * Lr.lam
            assert abs(c.query(f"mg_lambda_0_{l}") - Ll.lam) <= 1e-10 * Ll.lam


def test_vcycle(mgpair):
    P = mgpair
    if any(L.n_nonpos for L in P.mg_r.levels):
        pytest.skip("indefinite level operator (R9): Chebyshev smoothing is not a contraction there")
    b = P.o.project(P.inp["p"])
    x = host(P.ctx.mg_vcycle(1, dev(b), empty(P.ctx.n_p)))
    assert rel_l2(x, P.mg_r.vcycle(b)) <= 1e-10


@pytest.mark.parametrize("iters", [1, 3, 8])
def test_mgcg_prefix(mgpair, iters):
    P = mgpair
    if any(L.n_nonpos for L in P.mg_r.levels):
        pytest.skip("indefinite level operator (R9)")
    b = P.inp["p"]
    x = host(P.ctx.poisson_mgcg(1, dev(b), empty(P.ctx.n_p), iters))
    assert rel_l2(x, P.mg_r.pcg(b, iters)) <= 1e-10


def test_wbfbt_mg_inner(mgpair):
    from oracle import mg as omg
    P = mgpair
    if any(L.n_nonpos for L in P.mg_r.levels + P.mg_l.levels):
        pytest.skip("indefinite level operator (R9)")
    P.ctx.set_inner_mg(4)
    try:
        z = host(P.ctx.apply_wbfbt(dev(P.inp["p"]), empty(P.ctx.n_p), 1))
    finally:
        P.ctx.set_inner_mg(0)
    zo = omg.wbfbt_mg(P.o, P.inp["mu_q"], P.ost, P.mg_l, P.mg_r, P.inp["p"], 4)
    assert rel_l2(z, zo) <= 1e-9


def test_mesh_independent_convergence():
    """MG-PCG reaches a 1e-6 residual reduction in the same iteration count (+-2) at N = 16
    and N = 32 (C2's recipe), while Jacobi-PCG needs several times more and grows."""
    its, its_j = [], []
    for N in (16, 32):
        P = Pair("C2", N)
        P.ctx.setup_mg(3)
        st = P.ost
        b = P.o.project(P.inp["p"])
        bd = dev(b)
        got = None
        for it in range(2, 40):
            x = host(P.ctx.poisson_mgcg(1, bd, empty(P.ctx.n_p), it))
            if P.o.poisson_relres(st["Dinv"], b, x) < 1e-6:
                got = it
                break
        assert got is not None
        its.append(got)
        for it in range(50, 2000, 50):
            x = host(P.ctx.poisson_pcg(1, bd, empty(P.ctx.n_p), it))
            if P.o.poisson_relres(st["Dinv"], b, x) < 1e-6:
                break
        its_j.append(it)
    print("MG-PCG iterations", its, "Jacobi-PCG", its_j)
    assert abs(its[1] - its[0]) <= 2 and its_j[1] > 4 * its[1] and its_j[1] > its_j[0]


def test_full_size_c5_mgcg():
    """C5 (64^3, DR 1e10): 8 MG-PCG iterations against the oracle, and 30 iterations reach
    the 1e-6 reduction the paper's solver targets."""
    from oracle import mg as omg
    P = Pair("C5")
    P.ctx.setup_mg(3)
    mgr = omg.MG(P.N, P.ost["Dw"])
    b = P.inp["p"]
    x = host(P.ctx.poisson_mgcg(1, dev(b), empty(P.ctx.n_p), 8))
    assert rel_l2(x, mgr.pcg(b, 8)) <= 1e-9
    bp = P.o.project(b)
    x = host(P.ctx.poisson_mgcg(1, dev(bp), empty(P.ctx.n_p), 30))
    assert P.o.poisson_relres(P.ost["Dinv"], bp, x) < 1e-6


def test_k4_pmg_convergence():
    """C4 (24^3, Q4 x P3disc, DR 1e6): the p/h multigrid (spectral level, then h-levels) as
    PCG preconditioner reaches a 1e-6 reduction in far fewer iterations than Jacobi-PCG."""
    P = Pair("C4")
    P.ctx.setup_mg(3)
    assert [int(P.ctx.query(f"mg_k_{l}")) for l in range(int(P.ctx.query("mg_levels")))] == [4, 2, 2, 2, 2]
    st = P.ost
    b = P.o.project(P.inp["p"])
    bd = dev(b)
    got = None
    for it in range(10, 80, 5):
        x = host(P.ctx.poisson_mgcg(1, bd, empty(P.ctx.n_p), it))
        if P.o.poisson_relres(st["Dinv"], b, x) < 1e-6:
            got = it
            break
    x = host(P.ctx.poisson_pcg(1, bd, empty(P.ctx.n_p), 4 * (got or 80)))
    rr_j = P.o.poisson_relres(st["Dinv"], b, x)
    print("C4 p/h-MG-PCG iterations to 1e-6:", got, "; Jacobi-PCG relres after 4x as many:", rr_j)
    assert got is not None and rr_j > 1e-6
