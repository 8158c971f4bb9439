"""Pins for the oracle's divergence B, gradient B^T and Poisson operator K.

* B exact on polynomials: (B u)_{e,m} = -int_e q_m div u dx (B u := -div u,
  PAPER.md:962) against exact rational integrals times the Legendre
  normalisation;
* adjointness <Bu, p> = <u, B^T p>;
* divergence theorem: B^T z0 = 0 and z0 . B u = 0 for Dirichlet u
  (the constant pressure spans the Neumann null space,
  PAPER.md:1033-1036);
* K = B diag(Xinv) B^T brute force from the element matrices, its Jacobi
  diagonal, symmetry and K z0 = 0.
"""
from fractions import Fraction
from math import sqrt

import numpy as np
import pytest

import synth
from oracle import Oracle
from tests import polyexact as P
from tests.test_oracle_A import interp, _fields

LEG = {0: {0: Fraction(1)}, 1: {1: Fraction(1)}, 2: {0: Fraction(-1, 2), 2: Fraction(3, 2)},
       3: {1: Fraction(-3, 2), 3: Fraction(5, 2)}}


def _xi_poly(N, e_idx, d):
    """xi_d(x) = 2N (x_d - e_idx/N) - 1 as a polynomial in x_d."""
    ex = [0, 0, 0]
    ex[d] = 1
    return P.add({tuple(ex): Fraction(2 * N)}, {(0, 0, 0): Fraction(-2 * e_idx - 1)})


def _legendre_of_xi(n, xi):
    out = {}
    powk = {(0, 0, 0): Fraction(1)}
    for j in range(max(LEG[n]) + 1):
        if j in LEG[n]:
            out = P.add(out, P.scale(powk, LEG[n][j]))
        powk = P.mul(powk, xi)
    return out


@pytest.mark.parametrize("N,k", [(2, 2), (1, 4), (2, 3)])
def test_B_exact_on_polynomials(N, k):
    o = Oracle(N, k)
    modes = o.tables()["modes"]
    u, _ = _fields(k)
    uh = interp(N, k, u)
    p = o.apply_B(uh, nomask=True).reshape(o.n_el, o.n_m)
    divu = P.add(P.diff(u[0], 0), P.diff(u[1], 1), P.diff(u[2], 2))
    for e in range(o.n_el):
        eidx = (e % N, (e // N) % N, e // (N * N))
        lo = tuple(Fraction(i, N) for i in eidx)
        hi = tuple(Fraction(i + 1, N) for i in eidx)
        for m, md in enumerate(modes):
            q = {(0, 0, 0): Fraction(1)}
            norm = 1.0
            for d in range(3):
                q = P.mul(q, _legendre_of_xi(int(md[d]), _xi_poly(N, eidx[d], d)))
                norm *= sqrt((2 * int(md[d]) + 1) / 2)
            exact = -norm * float(P.integrate_box(P.mul(q, divu), lo, hi))
            assert abs(p[e, m] - exact) <= 1e-13 * max(1.0, np.abs(p).max()), (e, m, p[e, m], exact)


@pytest.mark.parametrize("N,k", [(3, 2), (4, 2), (2, 4)])
def test_adjoint_and_constant_pressure(N, k):
    o = Oracle(N, k)
    rng = np.random.default_rng(11)
    u, p = rng.uniform(-1, 1, o.n_v), rng.uniform(-1, 1, o.n_p)
    Bu, BTp = o.apply_B(u), o.apply_BT(p)
    assert abs(Bu @ p - u @ BTp) <= 1e-14 * np.linalg.norm(Bu) * np.linalg.norm(p) * 10
    z0 = np.zeros(o.n_p)
    z0[::o.n_m] = 2 * sqrt(2)
    normB = np.abs(o.element_B()).max()
    assert np.abs(o.apply_BT(z0)).max() <= 1e-13 * normB
    assert abs(z0 @ Bu) <= 1e-13 * normB * np.abs(u).sum() ** 0 * o.n_el
    # without the Dirichlet mask the constant pressure is NOT in the kernel (boundary flux)
    assert np.abs(o.apply_BT(z0, nomask=True)).max() > 1e-3 * normB


def _dense_B(o: Oracle):
    m = o.dofmap().reshape(o.n_el, o.n_q)
    Be = o.element_B()
    B = np.zeros((o.n_p, o.n_v))
    for e in range(o.n_el):
        cols = np.concatenate([c * o.n_nodes + m[e] for c in range(3)])
        B[e * o.n_m:(e + 1) * o.n_m, cols] = Be
    mask = o.boundary_mask().astype(bool)
    B[:, mask] = 0.0
    return B


@pytest.mark.parametrize("N,k", [(2, 2), (3, 2), (2, 4)])
def test_K_and_jacobi_diag_bruteforce(N, k):
    o = Oracle(N, k)
    if k == 2:
        mu_q = synth.make_inputs("C2", 0, N=N)["mu_q"]
    else:
        mu_q = np.random.default_rng(2).uniform(0.5, 3, o.n_el * o.n_q)
    lm = o.lumped(mu_q)
    B = _dense_B(o)
    Xv = np.tile(lm["Dinv"], 3)
    K = B @ (Xv[:, None] * B.T)
    rng = np.random.default_rng(5)
    p = rng.uniform(-1, 1, o.n_p)
    np.testing.assert_allclose(o.apply_K(lm["Dinv"], p), K @ p, rtol=0, atol=1e-12 * np.abs(K).max())
    np.testing.assert_allclose(o.jacobi_diag(lm["Dinv"]), np.diag(K), rtol=1e-13, atol=0)
    assert np.allclose(K, K.T, rtol=0, atol=1e-13 * np.abs(K).max())
    z0 = np.zeros(o.n_p)
    z0[::o.n_m] = 2 * sqrt(2)
    assert np.abs(o.apply_K(lm["Dinv"], z0)).max() <= 1e-12 * np.abs(K).max()
    # rank n_p - 1 (only the constant pressure in the null space) on a positive D_w
    if lm["n_nonpos_Dw"] == 0:
        ev = np.linalg.eigvalsh(K)
        assert (ev < 1e-10 * ev.max()).sum() == 1


def test_projection():
    o = Oracle(3, 2)
    rng = np.random.default_rng(0)
    v = rng.uniform(-1, 1, o.n_p)
    z0 = np.zeros(o.n_p)
    z0[::o.n_m] = 2 * sqrt(2)
    Pv = o.project(v)
    assert abs(z0 @ Pv) <= 1e-14 * np.linalg.norm(v) * np.linalg.norm(z0)
    np.testing.assert_allclose(Pv[1::4], v[1::4], rtol=0, atol=0)   # only mode 0 changes
    np.testing.assert_allclose(o.project(z0), 0, atol=1e-15)
