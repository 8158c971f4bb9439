"""Pins of the pressure-multigrid oracle (oracle/mg.py; R20).

* splitmix64 start vector: the generator's published first output from state 0;
* prolongation = exact embedding: a coarse P1disc field evaluated at points of the fine
  children equals the prolongated fine field there; P^T P = 8 I (orthonormal reference
  bases, child volume 1/8);
* restriction = L2 adjoint on dual vectors: (P^T r_f)_i = int f q_i^c for r_f[j] = int f q_j^f;
* coarse weights: constant density injects exactly (C_l = c M_l), and stay positive;
* MG-PCG converged equals the pseudo-inverse solution K^+ b (dense, constant deflated);
* the V-cycle is a symmetric operator (symmetric smoother, converged coarse solve);
* mesh independence ("iteration numbers are independent of mesh
  size"): iterations to a 1e-6 residual reduction at N = 4, 8, 16 differ by <= 2, while
  Jacobi-PCG's grow.
"""
from math import sqrt

import numpy as np
import pytest

import synth
from oracle import Oracle
from oracle import mg as omg
from tests.test_oracle_B import _dense_B


def test_splitmix_published_value():
    M64 = (1 << 64) - 1
    # first splitmix64 output from state 0 is 0xE220A8397B1DCDAF (Steele, Lea & Flood 2014)
    v = omg.splitmix_vector(2, seed=0)
    assert v[0] == 2.0 * ((0xE220A8397B1DCDAF >> 11) / 2.0 ** 53) - 1.0
    assert np.all(np.abs(omg.splitmix_vector(1000)) <= 1.0)
    del M64


def _eval_p1(coef, xi):
    """P1 field of one element (orthonormal modes 1, x, y, z on the reference cube) at xi."""
    l0 = 1 / sqrt(2)
    l1 = lambda t: sqrt(1.5) * t  # noqa: E731
    return l0 ** 3 * coef[0] + l1(xi[0]) * l0 ** 2 * coef[1] + l1(xi[1]) * l0 ** 2 * coef[2] + l1(xi[2]) * l0 ** 2 * coef[3]


def test_prolongation_is_exact_embedding():
    o = Oracle(2, 2)
    T = omg.prolongation_tables(o)
    rng = np.random.default_rng(0)
    Nc = 2
    xc = rng.uniform(-1, 1, 4 * Nc ** 3)
    xf = omg.prolong(T, xc, Nc, 4)
    ch = omg.child_index(Nc)
    for ec in range(Nc ** 3):
        for s in range(8):
            sh = np.array([s & 1, (s >> 1) & 1, (s >> 2) & 1]) * 2 - 1
            for xi in rng.uniform(-1, 1, (3, 3)):
                vf = _eval_p1(xf[4 * ch[ec, s]: 4 * ch[ec, s] + 4], xi)
                vc = _eval_p1(xc[4 * ec: 4 * ec + 4], (xi + sh) / 2)
                assert vf == pytest.approx(vc, abs=1e-14)
    # P^T P = 8 I
    PtP = sum(T[s].T @ T[s] for s in range(8))
    assert np.allclose(PtP, 8 * np.eye(4), atol=1e-14)


def test_restriction_is_l2_adjoint():
    """r_f[j] = int_{fine e} f q_j for f = a coarse-elementwise P1 function g: then
    P^T r_f = int_{coarse e} g q_i^c = (h_c/2)^3 g_c (orthonormal reference modes)."""
    o = Oracle(2, 2)
    T = omg.prolongation_tables(o)
    Nc = 1
    g = np.array([0.3, -1.2, 0.7, 2.0])
    hf = 1.0 / (2 * Nc)
    gf = omg.prolong(T, g, Nc, 4)
    rf = (hf / 2) ** 3 * gf  # int_{fine e} g q_j = (h_f/2)^3 g_f[j] (g is P1 on the child)
    rc = omg.restrict(T, rf, Nc, 4)
    assert np.allclose(rc, (2 * hf / 2) ** 3 * g, atol=1e-15)


def test_coarse_weights_inject_density():
    N = 8
    o = Oracle(N, 2)
    M = o.lumped(np.ones(o.n_el * o.n_q))["Cw"]
    m = omg.MG(N, 3.5 * M)
    for L in m.levels:
        Ml = L.o.lumped(np.ones(L.o.n_el * L.o.n_q))["Cw"]
        assert np.allclose(L.C, 3.5 * Ml, rtol=1e-14)
    inp = synth.make_inputs("C2", 0, N=16)
    o = Oracle(16, 2)
    st = o.setup(inp["mu_q"])
    m = omg.MG(16, st["Cw"])
    assert [L.N for L in m.levels] == [16, 8, 4, 2, 1]
    assert all(L.n_nonpos == 0 for L in m.levels)


def _pinv_deflated(K, nm=4):
    n = K.shape[0]
    z = np.zeros(n)
    z[::nm] = 1.0
    z /= np.linalg.norm(z)
    Pm = np.eye(n) - np.outer(z, z)
    ev, V = np.linalg.eigh(Pm @ K @ Pm)
    keep = np.abs(ev) > 1e-10 * np.abs(ev).max()
    return (V[:, keep] / ev[keep]) @ V[:, keep].T


def _mild(o, seed=0):
    return np.random.default_rng(seed).uniform(0.5, 2.0, o.n_el * o.n_q)


def test_mgpcg_converges_to_pseudoinverse():
    N = 4
    o = Oracle(N, 2)
    st = o.setup(_mild(o))
    m = omg.MG(N, st["Dw"])
    B = _dense_B(o)
    K = B @ (np.tile(m.levels[0].X, 3)[:, None] * B.T)
    b = o.project(np.random.default_rng(1).uniform(-1, 1, o.n_p))
    x = m.pcg(b, 25)
    xe = _pinv_deflated(K) @ b
    assert np.linalg.norm(x - xe) <= 1e-9 * np.linalg.norm(xe)


def test_vcycle_symmetric():
    N = 4
    o = Oracle(N, 2)
    st = o.setup(_mild(o, 3))
    m = omg.MG(N, st["Dw"])
    rng = np.random.default_rng(4)
    a, b = (o.project(rng.uniform(-1, 1, o.n_p)) for _ in range(2))
    lhs, rhs = m.vcycle(a) @ b, a @ m.vcycle(b)
    assert abs(lhs - rhs) <= 1e-10 * abs(lhs)


def _iters_to(o, K_apply, prec, b, tol=1e-6, cap=400):
    x = np.zeros_like(b)
    r = o.project(b)
    z = prec(r)
    p = z.copy()
    rz = r @ z
    r0 = np.linalg.norm(r)
    for it in range(1, cap + 1):
        q = K_apply(p)
        a = rz / (p @ q)
        x += a * p
        r -= a * q
        if np.linalg.norm(r) < tol * r0:
            return it
        z = prec(r)
        rz1 = r @ z
        p = z + rz1 / rz * p
        rz = rz1
    return cap


def test_mesh_independent_iterations():
    """multigrid iteration numbers are independent of the mesh size.
    Two smooth wide sinkers (delta = 20, omega = 0.3, viscosity ratio 10), N = 4, 8, 16."""
    its, its_j = [], []
    cen = np.array([[0.3, 0.4, 0.5], [0.7, 0.6, 0.4]])
    for N in (4, 8, 16):
        o = Oracle(N, 2)
        mu = synth.viscosity_at_quadrature(N, 2, cen, 20.0, 0.3, 1.0, 10.0)
        st = o.setup(mu)
        assert st["n_nonpos_Dw"] == 0
        m = omg.MG(N, st["Dw"])
        L0 = m.levels[0]
        b = o.project(np.random.default_rng(5).uniform(-1, 1, o.n_p))
        its.append(_iters_to(o, L0.K, m.vcycle, b))
        minv = np.where(np.abs(L0.diagK) > 1e-13 * np.abs(L0.diagK).max(), 1 / L0.diagK, 0.0)
        its_j.append(_iters_to(o, L0.K, lambda r: minv * r, b))
    assert max(its) - min(its) <= 2, its
    assert its_j[-1] > 2 * its[-1] and its_j[-1] > its_j[0], (its, its_j)


# ---------------------------------------------------------------- velocity multigrid (R22)
def test_q2_prolongation_interpolates_quadratics_exactly():
    """Coarse nodal values of u = x^2 y (1 - z), a Q2 function on every coarse element,
    prolongate to its exact values at the fine nodes; restriction is the transpose."""
    Nc = 2
    o = Oracle(Nc, 2)
    xn = o.tables()["xn"]
    P1 = omg.q2_prolongation_1d(Nc, xn)

    def nodes(N):
        line = np.concatenate([[(e + (xn[a] + 1) / 2) / N for a in range(2)] for e in range(N)] + [[1.0]])
        Z, Y, X = np.meshgrid(line, line, line, indexing="ij")
        return X.ravel(), Y.ravel(), Z.ravel()

    u = lambda x, y, z: x * x * y * (1 - z)  # noqa: E731
    xc = np.concatenate([u(*nodes(Nc)), np.zeros((2 * Nc + 1) ** 3), -u(*nodes(Nc))])
    xf = omg.vprolong(P1, xc)
    ref = np.concatenate([u(*nodes(2 * Nc)), np.zeros((4 * Nc + 1) ** 3), -u(*nodes(2 * Nc))])
    assert np.allclose(xf, ref, atol=1e-15)
    rng = np.random.default_rng(0)
    a, b = rng.standard_normal(xc.size), rng.standard_normal(xf.size)
    assert omg.vprolong(P1, a) @ b == pytest.approx(a @ omg.vrestrict(P1, b), rel=1e-13)


def test_mu_coarsening_constants_and_positivity():
    o = Oracle(4, 2)
    wg = o.tables()["wg"]
    assert np.allclose(omg.coarsen_mu(np.full(4 ** 3 * 27, 2.5), 2, wg), 2.5, rtol=1e-15)
    mu = np.random.default_rng(1).uniform(1e-3, 1e3, 4 ** 3 * 27)
    mc = omg.coarsen_mu(mu, 2, wg)
    assert np.all(mc > 0) and mc.max() <= mu.max() and mc.min() >= mu.min()


def test_velocity_vcycle_symmetric_and_mesh_independent():
    """The velocity V-cycle is a symmetric linear map (Chebyshev smoothing and coarse solve
    are fixed polynomials); MG-PCG on A needs about the same iterations at N = 4, 8, 16 for a
    smooth viscosity while Jacobi-PCG's grow."""
    cen = np.array([[0.3, 0.4, 0.5], [0.7, 0.6, 0.4]])
    o = Oracle(4, 2)
    mu = synth.viscosity_at_quadrature(4, 2, cen, 20.0, 0.3, 1.0, 10.0)
    V = omg.VMG(4, mu)
    mask = o.boundary_mask().astype(bool)
    rng = np.random.default_rng(2)
    a, b = (np.where(mask, 0.0, rng.standard_normal(o.n_v)) for _ in range(2))
    assert V.vcycle(a) @ b == pytest.approx(a @ V.vcycle(b), rel=1e-10)
    its, its_j = [], []
    for N in (4, 8, 16):
        o = Oracle(N, 2)
        mu = synth.viscosity_at_quadrature(N, 2, cen, 20.0, 0.3, 1.0, 10.0)
        V = omg.VMG(N, mu)
        mask = o.boundary_mask().astype(bool)
        rhs = np.where(mask, 0.0, np.random.default_rng(3).uniform(-1, 1, o.n_v))
        A = lambda v: o.apply_A(mu, v)  # noqa: E731
        dA = o.diag_A(mu)
        dinv = np.where(mask, 0.0, 1.0 / np.where(dA != 0, dA, 1.0))
        its.append(_cg_its(A, V.vcycle, rhs))
        its_j.append(_cg_its(A, lambda r: dinv * r, rhs))
    assert max(its) - min(its) <= 3, its
    assert its_j[-1] > 2 * its[-1] and its_j[-1] > its_j[0], (its, its_j)


def _cg_its(A, prec, b, tol=1e-6, cap=400):
    x = np.zeros_like(b)
    r = b.copy()
    z = prec(r)
    p = z.copy()
    rz = r @ z
    r0 = np.linalg.norm(r)
    for it in range(1, cap + 1):
        q = A(p)
        a = rz / (p @ q)
        x += a * p
        r -= a * q
        if np.linalg.norm(r) < tol * r0:
            return it
        z = prec(r)
        rz1 = r @ z
        p = z + rz1 / rz * p
        rz = rz1
    return cap


# ---------------------------------------------------------------- spectral (p) level, k = 4
def test_p_transfer_is_mode_embedding():
    """P1disc modes are the first four P3disc modes (R2 ordering, orthonormal on the same
    element): the spectral transfer is [I_4; 0] (closed form)."""
    T = omg.p_transfer_table(Oracle(1, 4), Oracle(1, 2))
    ref = np.zeros((20, 4))
    ref[:4, :4] = np.eye(4)
    assert np.allclose(T, ref, atol=1e-14)


def test_k4_hierarchy_weights_and_converged_mgpcg():
    N = 2
    o = Oracle(N, 4)
    M = o.lumped(np.ones(o.n_el * o.n_q))["Cw"]
    m = omg.MG(N, 2.5 * M, k=4)
    assert [(L.N, L.o.k) for L in m.levels] == [(2, 4), (2, 2), (1, 2)]
    for L in m.levels:
        Ml = L.o.lumped(np.ones(L.o.n_el * L.o.n_q))["Cw"]
        assert np.allclose(L.C, 2.5 * Ml, rtol=1e-13)
    st = o.setup(_mild(o, 5))
    m = omg.MG(N, st["Dw"], k=4)
    B = _dense_B(o)
    K = B @ (np.tile(m.levels[0].X, 3)[:, None] * B.T)
    b = o.project(np.random.default_rng(6).uniform(-1, 1, o.n_p))
    xe = _pinv_deflated(K, nm=o.n_m) @ b
    x = m.pcg(b, 30)
    assert np.linalg.norm(x - xe) <= 1e-8 * np.linalg.norm(xe)


def test_k4_mg_beats_jacobi():
    """C4's recipe (Q4 x P3disc, 8 sinkers, DR 1e6) on 8^3: p/h-MG-PCG reaches a 1e-6 reduction
    in far fewer iterations than Jacobi-PCG (52 vs 317)."""
    inp = synth.make_inputs("C4", 0, N=8)
    o = Oracle(8, 4)
    st = o.setup(inp["mu_q"])
    m = omg.MG(8, st["Dw"], k=4)
    L0 = m.levels[0]
    b = o.project(inp["p"])
    its = _iters_to(o, L0.K, m.vcycle, b)
    minv = np.where(np.abs(L0.diagK) > 1e-13 * np.abs(L0.diagK).max(), 1 / L0.diagK, 0.0)
    its_j = _iters_to(o, L0.K, lambda r: minv * r, b)
    assert its < 60 and its_j > 4 * its, (its, its_j)  # measured 52 vs 317


def test_velocity_p_level():
    """k = 4 velocity hierarchy: the Q2-in-Q4 prolongation reproduces a Q2 field exactly at the
    Q4 nodes; the spectral mu coarsening is exact on constants; the V-cycle stays symmetric."""
    N = 2
    o4, o2 = Oracle(N, 4), Oracle(N, 2)
    P1 = omg.p_prolongation_1d(N, o2.tables()["xn"], o4.tables()["xn"])

    def nodes(o):
        xn = o.tables()["xn"]
        k = o.k
        line = np.concatenate([[(e + (xn[a] + 1) / 2) / N for a in range(k)] for e in range(N)] + [[1.0]])
        Z, Y, X = np.meshgrid(line, line, line, indexing="ij")
        return X.ravel(), Y.ravel(), Z.ravel()

    u = lambda x, y, z: (x * x - y) * z * (1 - z)  # noqa: E731
    zc = np.zeros((2 * N + 1) ** 3)
    xf = omg.vprolong(P1, np.concatenate([u(*nodes(o2)), zc, zc]))
    assert np.allclose(xf[:(4 * N + 1) ** 3], u(*nodes(o4)), atol=1e-14)
    assert np.allclose(omg.coarsen_mu_p(np.full(o4.n_el * 125, 3.0), o4.n_el, o4.tables()["wg"]), 3.0, rtol=1e-15)
    mu = np.random.default_rng(0).uniform(0.5, 2.0, o4.n_el * 125)
    V = omg.VMG(N, mu, k=4)
    assert [(L["N"], L["o"].k) for L in V.lev] == [(2, 4), (2, 2), (1, 2)]
    mask = o4.boundary_mask().astype(bool)
    rng = np.random.default_rng(1)
    a, b = (np.where(mask, 0.0, rng.standard_normal(o4.n_v)) for _ in range(2))
    assert V.vcycle(a) @ b == pytest.approx(a @ V.vcycle(b), rel=1e-10)
