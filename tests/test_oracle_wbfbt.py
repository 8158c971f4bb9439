"""Pins for the oracle's Jacobi-PCG and wBFBT apply.

* converged PCG (iters >> n_p, positive D_w) equals the pseudo-inverse
  solution K^+ b (numpy eigh, constant mode deflated);
* PCG with 1 iteration equals the closed form (r.z / z.Kz) z;
* wBFBT with converged inner solves equals eq:wbfbt
  evaluated densely with exact pseudo-inverses;
* wBFBT(16 mu) = 16 wBFBT(mu) bit-exactly (scaling invariance of the weights,
  PAPER.md:1382-1385);
* a_l = a_r -> K_l = K_r: the converged operator is symmetric.
The fixed-iteration VALUES have no closed form: parity unpinned beyond these
(DESIGN.md Sec. 6).
"""
from math import sqrt

import numpy as np
import pytest

import synth
from oracle import Oracle
from tests.test_oracle_B import _dense_B


def _mild_mu(o, seed=0):
    return np.random.default_rng(seed).uniform(0.5, 2.0, o.n_el * o.n_q)


def _z0(o):
    z = np.zeros(o.n_p)
    z[::o.n_m] = 2 * sqrt(2)
    return z / np.linalg.norm(z)


def _pinv_deflated(K, z):
    """Pseudo-inverse of symmetric K restricted to the complement of unit vector z."""
    Pm = np.eye(len(z)) - np.outer(z, z)
    ev, V = np.linalg.eigh(Pm @ K @ Pm)
    keep = np.abs(ev) > 1e-10 * np.abs(ev).max()
    return (V[:, keep] / ev[keep]) @ V[:, keep].T


def converged_iters(o, Xinv, diagK, b, tol=1e-13, step=5, cap=2000):
    """Smallest multiple of `step` at which the projected PCG residual is below tol.
    (CG keeps iterating past convergence under the fixed-count rule and then drifts,
    so 'many iterations' is not a converged regime -- stop at the residual floor.)"""
    for it in range(step, cap, step):
        if o.poisson_relres(Xinv, b, o.poisson(Xinv, diagK, b, it)) < tol:
            return it
    raise AssertionError("PCG did not converge")


@pytest.mark.parametrize("N,k", [(2, 2), (3, 2), (2, 4), (1, 2), (1, 4)])
def test_pcg_converges_to_pseudoinverse(N, k):
    """N = 1 pins the pseudo-inverse Jacobi threshold of R11 (jacobi_minv): on one element
    every velocity node but the interior ones is Dirichlet, the constant-mode row of K vanishes
    (the interior bubbles' derivatives integrate to zero), its diagonal is rounding-level, and
    only Minv = 0 there (not 1 / diag) lets PCG converge to the deflated K^+ b."""
    o = Oracle(N, k)
    st = o.setup(_mild_mu(o))
    assert st["n_nonpos_Dw"] == 0
    B = _dense_B(o)
    K = B @ (np.tile(st["Dinv"], 3)[:, None] * B.T)
    z = _z0(o)
    b = o.project(np.random.default_rng(1).uniform(-1, 1, o.n_p))
    it = converged_iters(o, st["Dinv"], st["diagKr"], b)
    x = o.poisson(st["Dinv"], st["diagKr"], b, iters=it)
    ref = _pinv_deflated(K, z) @ b
    assert np.linalg.norm(x - ref) <= 1e-10 * np.linalg.norm(ref)


@pytest.mark.parametrize("N,k", [(2, 2), (2, 4)])
def test_poisson_relres_closed_forms(N, k):
    """or_poisson_relres = ||b - K x|| / ||b||: exactly 1 at x = 0, and |1 - t| at
    x = t K^+ b for b in the range of K (b projected off the constant pressure)."""
    o = Oracle(N, k)
    st = o.setup(_mild_mu(o, 3))
    B = _dense_B(o)
    K = B @ (np.tile(st["Dinv"], 3)[:, None] * B.T)
    b = o.project(np.random.default_rng(5).uniform(-1, 1, o.n_p))
    assert o.poisson_relres(st["Dinv"], b, np.zeros(o.n_p)) == 1.0
    xs = _pinv_deflated(K, _z0(o)) @ b
    for t, want in ((1.0, 0.0), (0.5, 0.5), (-1.0, 2.0)):
        assert abs(o.poisson_relres(st["Dinv"], b, t * xs) - want) <= 1e-11


def test_pcg_one_iteration_closed_form():
    o = Oracle(3, 2)
    st = o.setup(_mild_mu(o, 4))
    B = _dense_B(o)
    K = B @ (np.tile(st["Dinv"], 3)[:, None] * B.T)
    b = np.random.default_rng(2).uniform(-1, 1, o.n_p)
    zz = b / st["diagKr"]
    x1 = o.pcg(st["Dinv"], st["diagKr"], b, 1)
    np.testing.assert_allclose(x1, (b @ zz) / (zz @ K @ zz) * zz, rtol=1e-12)
    np.testing.assert_array_equal(o.pcg(st["Dinv"], st["diagKr"], b, 0), 0)


def test_pcg_step_matches_pcg():
    o = Oracle(3, 2)
    st = o.setup(synth.make_inputs("C2", 0, N=3)["mu_q"])
    b = o.project(np.random.default_rng(3).uniform(-1, 1, o.n_p))
    Minv = 1.0 / st["diagKr"]
    x, r = np.zeros(o.n_p), b.copy()
    p = Minv * r
    rz = float(np.cumsum(r * p)[-1])   # sequential, as the oracle's dot (py3.12 sum() is compensated)
    for _ in range(7):
        x, r, p, rz = o.pcg_step(st["Dinv"], st["diagKr"], x, r, p, rz)
    np.testing.assert_array_equal(x, o.pcg(st["Dinv"], st["diagKr"], b, 7))


def test_pcg_scalars_match_dense_textbook_pcg():
    """The recorded alpha_i, beta_i (O9) equal those of a textbook PCG written here in
    numpy on the dense K (assembled from the dense B) with the same Jacobi Minv; the
    solution equals o.pcg's bit-exactly (recording does not change the arithmetic)."""
    o = Oracle(3, 2)
    st = o.setup(_mild_mu(o, 5))
    B = _dense_B(o)
    K = B @ (np.tile(st["Dinv"], 3)[:, None] * B.T)
    b = o.project(np.random.default_rng(4).uniform(-1, 1, o.n_p))
    iters = 6
    x, al, be, run = o.pcg_scalars(st["Dinv"], st["diagKr"], b, iters)
    assert run == iters
    np.testing.assert_array_equal(x, o.pcg(st["Dinv"], st["diagKr"], b, iters))
    Minv = 1.0 / st["diagKr"]
    r = b.copy(); z = Minv * r; p = z.copy(); rz = r @ z
    for i in range(iters):
        q = K @ p
        a = rz / (p @ q)
        r = r - a * q
        z = Minv * r
        rz2 = r @ z
        bt = rz2 / rz
        p = z + bt * p
        rz = rz2
        assert abs(al[i] - a) <= 1e-9 * abs(a), (i, al[i], a)
        assert abs(be[i] - bt) <= 1e-7 * abs(bt), (i, be[i], bt)
        assert al[i] > 0 and be[i] > 0  # SPD on the complement of the constants
    # zero iterations: nothing recorded
    _, al0, be0, run0 = o.pcg_scalars(st["Dinv"], st["diagKr"], b, 0)
    assert run0 == 0 and al0.size == 0


@pytest.mark.parametrize("a_l,a_r", [(1.0, 1.0), (1.0, 2.0), (3.0, 1.0)])
def test_wbfbt_converged_equals_dense_formula(a_l, a_r):
    N, k = 2, 2
    o = Oracle(N, k)
    mu = _mild_mu(o, 9)
    st = o.setup(mu, a_l, a_r)
    B = _dense_B(o)
    mask = o.boundary_mask().astype(bool)
    m = o.dofmap().reshape(o.n_el, o.n_q)
    A = np.zeros((o.n_v, o.n_v))
    for e in range(o.n_el):
        idx = np.concatenate([c * o.n_nodes + m[e] for c in range(3)])
        A[np.ix_(idx, idx)] += o.element_A_matrix(mu[e * o.n_q:(e + 1) * o.n_q])
    A[mask, :] = 0
    A[:, mask] = 0
    Ci, Di = np.tile(st["Cinv"], 3), np.tile(st["Dinv"], 3)
    Kl = B @ (Ci[:, None] * B.T)
    Kr = B @ (Di[:, None] * B.T)
    z = _z0(o)
    S = _pinv_deflated(Kl, z) @ (B @ (Ci[:, None] * (A @ (Di[:, None] * B.T)))) @ _pinv_deflated(Kr, z)
    r = np.random.default_rng(4).uniform(-1, 1, o.n_p)
    Pm = np.eye(o.n_p) - np.outer(z, z)
    ref = Pm @ S @ Pm @ r
    rp = o.project(r)
    it = max(converged_iters(o, st["Dinv"], st["diagKr"], rp), converged_iters(o, st["Cinv"], st["diagKl"], rp))
    got = o.wbfbt(r, iters=it)
    assert np.linalg.norm(got - ref) <= 1e-8 * np.linalg.norm(ref)
    if a_l == a_r:
        assert np.allclose(S, S.T, rtol=0, atol=1e-8 * np.abs(S).max())


@pytest.mark.parametrize("cfg,N", [("C1", 4), ("C2", 5)])
def test_wbfbt_scale_invariance_bitexact(cfg, N):
    inp = synth.make_inputs(cfg, 0, N=N)
    o = Oracle(N, 2)
    o.setup(inp["mu_q"], 1.0, 2.0)
    z1 = o.wbfbt(inp["p"], iters=synth.CONFIGS[cfg].iters)
    o.setup(16 * inp["mu_q"], 1.0, 2.0)
    z16 = o.wbfbt(inp["p"], iters=synth.CONFIGS[cfg].iters)
    np.testing.assert_array_equal(z16, 16 * z1)


def test_wbfbt_output_projected():
    inp = synth.make_inputs("C2", 0, N=4)
    o = Oracle(4, 2)
    o.setup(inp["mu_q"])
    z = o.wbfbt(inp["p"], 10)
    assert abs(_z0(o) @ z) <= 1e-14 * np.linalg.norm(z) * 10


def test_jacobi_pseudoinverse_threshold_only_removes_the_null_row():
    """DESIGN.md R11: Minv is 1/diag K except where |d| <= 1e-13 max|d|.  On the N = 1
    mesh every velocity node is Dirichlet, so B^T of ANY mode vanishes... except the
    interior GLL node at k = 2: the constant mode still has B^T z0 = 0 by the divergence
    theorem, so diag(K)_{mode 0} = sum (B_e[0,:])^2 X = 0 up to rounding -- the one row the
    threshold removes.  On N >= 2 with positive lumped masses no entry is near the
    threshold, so the pseudo-inverse is the plain inverse there."""
    B1 = None
    o = Oracle(1, 2)
    st = o.setup(_mild_mu(o))
    d = st["diagKr"]
    assert abs(d[0]) <= 1e-13 * np.abs(d).max()          # the constant-mode row vanishes
    assert np.all(np.abs(d[1:]) > 1e-3 * np.abs(d).max())  # the others are O(1)
    B1 = _dense_B(o)
    assert np.linalg.norm(B1[0]) <= 1e-14 * np.linalg.norm(B1)  # B^T z0 = 0 on N = 1
    for N, k in ((2, 2), (3, 2), (2, 4)):
        o = Oracle(N, k)
        st = o.setup(_mild_mu(o))
        d = st["diagKr"]
        assert np.abs(d).min() > 1e-6 * np.abs(d).max()
    # and on N = 1 the converged PCG is still the pseudo-inverse solution (mode 0 is z0)
    o = Oracle(1, 2)
    st = o.setup(_mild_mu(o))
    K = B1 @ (np.tile(st["Dinv"], 3)[:, None] * B1.T)
    b = o.project(np.random.default_rng(2).uniform(-1, 1, o.n_p))
    x = o.poisson(st["Dinv"], st["diagKr"], b, 3)
    assert np.allclose(x, _pinv_deflated(K, _z0(o)) @ b, rtol=0, atol=1e-12 * np.linalg.norm(x))
