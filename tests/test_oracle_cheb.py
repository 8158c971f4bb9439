"""Pins for the oracle's Chebyshev-accelerated Jacobi solve and its power iteration
(PAPER.md:2531-2546 names the smoother; recurrence and bounds:
reading R16).

* The recurrence (Saad 2003, Alg. 12.1) is a fixed polynomial filter: after k steps
  from x0 = 0, x_k = s_k(M^-1 K) M^-1 b with residual polynomial
  1 - lambda s_k(lambda) = T_k((theta - lambda)/delta) / T_k(theta/delta).  The pins
  evaluate that closed form by eigendecomposition (numpy eigh on the symmetric
  M^-1/2 K M^-1/2) and numpy's Chebyshev polynomials, and compare the iterates:
  diagonal, dense SPD with a Jacobi preconditioner, and the assembled (dense,
  brute force) K_w of tiny meshes with the constant mode projected out.
* The power iteration equals ||(M^-1 K)^k v0|| / ||(M^-1 K)^(k-1) v0|| (matrix powers).
"""
import numpy as np
import pytest
from numpy.polynomial import Chebyshev

import oracle
from oracle import Oracle
from tests.test_oracle_B import _dense_B
from tests.test_oracle_wbfbt import _mild_mu


def _s_of(lam, k, lmin, lmax):
    """s_k(lambda) with 1 - lambda s_k(lambda) = T_k((theta - lambda)/delta) / T_k(theta/delta),
    evaluated stably: T_k by numpy's Chebyshev series (Clenshaw); at lambda ~ 0 the limit
    s_k(0) = -r_k'(0) = T_k'(sigma1) / (delta T_k(sigma1))."""
    theta, delta = 0.5 * (lmax + lmin), 0.5 * (lmax - lmin)
    Tk = Chebyshev.basis(k)
    r = Tk((theta - lam) / delta) / Tk(theta / delta)
    small = np.abs(lam) < 1e-9 * lmax
    s0 = Tk.deriv()(theta / delta) / (delta * Tk(theta / delta))
    return np.where(small, s0, (1.0 - r) / np.where(small, 1.0, lam))


def _closed_form(K, Minv, b, k, lmin, lmax):
    """x_k = s_k(M^-1 K) M^-1 b = M^-1/2 V s_k(L) V^T M^-1/2 b, M^-1/2 K M^-1/2 = V L V^T."""
    m = np.sqrt(Minv)
    L, V = np.linalg.eigh(m[:, None] * K * m[None, :])
    s = _s_of(L, k, lmin, lmax)
    return m * (V @ (s * (V.T @ (m * b))))


@pytest.mark.parametrize("k", [1, 2, 5, 12])
def test_cheb_diagonal_closed_form(k):
    rng = np.random.default_rng(k)
    lam = rng.uniform(0.3, 4.0, 40)
    d = rng.uniform(0.5, 2.0, 40)              # Jacobi scaling: M^-1 K = diag(lam)
    K, Minv = np.diag(lam * d), 1.0 / d
    b = rng.standard_normal(40)
    x = oracle.cheb_dense(K, Minv, b, k, 0.3, 4.0)
    # error filter on the diagonal: e_k = T_k((theta - lam)/delta)/T_k(sigma1) e_0, e_0 = x*
    xs = b / (lam * d)
    theta, delta = 2.15, 1.85
    Tk = Chebyshev.basis(k)
    ek = Tk((theta - lam) / delta) / Tk(theta / delta) * xs
    np.testing.assert_allclose(xs - x, ek, rtol=0, atol=1e-13 * np.abs(xs).max())


@pytest.mark.parametrize("k,lmin_f", [(3, 1.0), (8, 1.0), (8, 0.1), (20, 0.5)])
def test_cheb_dense_spd_jacobi_closed_form(k, lmin_f):
    rng = np.random.default_rng(100 + k)
    n = 30
    Q, _ = np.linalg.qr(rng.standard_normal((n, n)))
    K = Q @ np.diag(rng.uniform(1.0, 50.0, n)) @ Q.T + 5 * np.eye(n)
    Minv = 1.0 / np.diag(K)
    m = np.sqrt(Minv)
    ev = np.linalg.eigvalsh(m[:, None] * K * m[None, :])
    lmin, lmax = lmin_f * ev.min(), ev.max()   # lmin_f < 1: an interval wider than the spectrum
    b = rng.standard_normal(n)
    x = oracle.cheb_dense(K, Minv, b, k, lmin, lmax)
    xc = _closed_form(K, Minv, b, k, lmin, lmax)
    assert np.linalg.norm(x - xc) <= 1e-12 * np.linalg.norm(xc)


def test_cheb_error_bound():
    """Textbook bound with the exact interval: ||e_k||_M^-1K <= 2 ((sqrt(kappa)-1)/(sqrt(kappa)+1))^k ||e_0||."""
    rng = np.random.default_rng(7)
    n = 25
    lam = np.linspace(1.0, 100.0, n)
    K, Minv, b = np.diag(lam), np.ones(n), rng.standard_normal(n)
    xs = b / lam
    kappa = 100.0
    rate = (np.sqrt(kappa) - 1) / (np.sqrt(kappa) + 1)
    for k in (5, 10, 20):
        e = xs - oracle.cheb_dense(K, Minv, b, k, 1.0, 100.0)
        na = lambda v: np.sqrt(v @ (lam * v))  # noqa: E731
        assert na(e) <= 2 * rate ** k * na(xs) * (1 + 1e-12)


@pytest.mark.parametrize("N,k,iters", [(2, 2, 4), (3, 2, 7), (2, 4, 5)])
def test_poisson_cheb_equals_closed_form_on_assembled_K(N, k, iters):
    """Projected FE solve P Cheb(K_r, P b) against the closed form on the dense K_r
    (dense B by brute-force assembly, tests/test_oracle_B.py), constant mode in the
    null space of M^-1 K (its s_k(0) term is projected out by the final P)."""
    o = Oracle(N, k)
    st = o.setup(_mild_mu(o))
    B = _dense_B(o)
    K = B @ (np.tile(st["Dinv"], 3)[:, None] * B.T)
    Minv = 1.0 / st["diagKr"]
    m = np.sqrt(Minv)
    ev = np.linalg.eigvalsh(m[:, None] * K * m[None, :])
    lmax = ev.max()
    lmin = 0.1 * lmax                            # PETSc-style interval (R16)
    b = np.random.default_rng(3).uniform(-1, 1, o.n_p)
    x = o.poisson_cheb(st["Dinv"], st["diagKr"], b, iters, lmin, lmax)
    xc = o.project(_closed_form(K, Minv, o.project(b), iters, lmin, lmax))
    assert np.linalg.norm(x - xc) <= 1e-12 * np.linalg.norm(xc)
    assert abs(x[::o.n_m].sum()) <= 1e-12 * np.abs(x).max() * o.n_el   # output projected


def test_poisson_cheb_linear():
    """A fixed polynomial filter: linear in b (the property GPU parity rests on)."""
    o = Oracle(3, 2)
    st = o.setup(_mild_mu(o))
    rng = np.random.default_rng(5)
    b1, b2 = rng.uniform(-1, 1, o.n_p), rng.uniform(-1, 1, o.n_p)
    f = lambda b: o.poisson_cheb(st["Cinv"], st["diagKl"], b, 9, 0.2, 2.5)  # noqa: E731
    lhs, rhs = f(2.0 * b1 - 3.0 * b2), 2.0 * f(b1) - 3.0 * f(b2)
    assert np.linalg.norm(lhs - rhs) <= 1e-13 * np.linalg.norm(lhs)


@pytest.mark.parametrize("iters", [1, 3, 10])
def test_eigmax_dense_matrix_powers(iters):
    rng = np.random.default_rng(iters)
    n = 20
    A = rng.standard_normal((n, n))
    K = A @ A.T + np.eye(n)
    Minv = rng.uniform(0.5, 1.5, n)
    v0 = rng.standard_normal(n)
    MK = Minv[:, None] * K
    lam = np.linalg.norm(np.linalg.matrix_power(MK, iters) @ v0) / np.linalg.norm(
        np.linalg.matrix_power(MK, iters - 1) @ v0)
    got = oracle.eigmax_dense(K, Minv, v0, iters)
    assert abs(got - lam) <= 1e-12 * lam


def test_poisson_eigmax_converges_to_spectral_radius():
    o = Oracle(2, 2)
    st = o.setup(_mild_mu(o))
    B = _dense_B(o)
    K = B @ (np.tile(st["Dinv"], 3)[:, None] * B.T)
    Minv = 1.0 / st["diagKr"]
    m = np.sqrt(Minv)
    lmax = np.abs(np.linalg.eigvalsh(m[:, None] * K * m[None, :])).max()
    v0 = np.random.default_rng(9).standard_normal(o.n_p)
    got = o.poisson_eigmax(st["Dinv"], st["diagKr"], v0, 400)
    assert abs(got - lmax) <= 1e-6 * lmax
    # and a few steps equal the matrix-power ratio on the dense K
    MK = Minv[:, None] * K
    for it in (1, 4):
        ref = np.linalg.norm(np.linalg.matrix_power(MK, it) @ v0) / np.linalg.norm(
            np.linalg.matrix_power(MK, it - 1) @ v0)
        assert abs(o.poisson_eigmax(st["Dinv"], st["diagKr"], v0, it) - ref) <= 1e-11 * ref


def test_wbfbt_cheb_equals_closed_form():
    """wBFBT with Chebyshev inner solves (R16) = P F_l P B C^-1 A D^-1 B^T P F_r P r, with
    F_side the closed-form Chebyshev filter of the dense K_side (assembled B and A)."""
    from tests.test_oracle_diagA import _dense_A
    o = Oracle(2, 2)
    st = o.setup(_mild_mu(o, 9), 1.0, 2.0)
    B = _dense_B(o)
    mask = o.boundary_mask().astype(bool)
    A = _dense_A(o, o.mu_q)
    A[mask, :] = 0; A[:, mask] = 0
    Ci, Di = np.tile(st["Cinv"], 3), np.tile(st["Dinv"], 3)
    Kl, Kr = B @ (Ci[:, None] * B.T), B @ (Di[:, None] * B.T)
    Ml, Mr = 1.0 / st["diagKl"], 1.0 / st["diagKr"]
    it, lo_l, hi_l, lo_r, hi_r = 7, 0.2, 2.4, 0.15, 2.2
    r = np.random.default_rng(6).uniform(-1, 1, o.n_p)
    P = o.project
    y = P(_closed_form(Kr, Mr, P(r), it, lo_r, hi_r))
    s = B @ (Ci * (A @ (Di * (B.T @ y))))
    ref = P(_closed_form(Kl, Ml, P(s), it, lo_l, hi_l))
    got = o.wbfbt_cheb(r, it, lo_l, hi_l, lo_r, hi_r)
    assert np.linalg.norm(got - ref) <= 1e-11 * np.linalg.norm(ref)
