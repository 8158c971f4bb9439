"""Pins for the oracle's diag(A) and the Chebyshev-accelerated Jacobi smoother on A
(the paper's smoother for the viscous block; SURVEY.md 8(f) #1's
approximate A^-1; readings R16, R18):

* diag(M A M) equals the diagonal of the densely assembled matrix (element matrices
  of tests/test_oracle_A.py's dense-assembly pin), Dirichlet dofs 0;
* the smoother's iterates equal the closed-form Chebyshev filter on the interior
  block of the dense A with the Jacobi preconditioner (as tests/test_oracle_cheb.py);
* the power iteration equals the matrix-power ratio.
"""
import numpy as np
import pytest

from oracle import Oracle
from tests.test_oracle_cheb import _closed_form


def _dense_A(o, mu_q):
    m = o.dofmap().reshape(o.n_el, o.n_q)
    nq = o.n_q
    A = np.zeros((o.n_v, o.n_v))
    for e in range(o.n_el):
        Ae = o.element_A_matrix(mu_q[e * nq:(e + 1) * nq])
        idx = np.concatenate([c * o.n_nodes + m[e] for c in range(3)])
        A[np.ix_(idx, idx)] += Ae
    return A


@pytest.mark.parametrize("N,k", [(2, 2), (3, 2), (2, 4)])
def test_diag_A_equals_dense_diagonal(N, k):
    o = Oracle(N, k)
    mu = np.exp(np.random.default_rng(N + k).uniform(-3, 3, o.n_el * o.n_q))
    A = _dense_A(o, mu)
    mask = o.boundary_mask().astype(bool)
    want = np.where(mask, 0.0, np.diag(A))
    got = o.diag_A(mu)
    np.testing.assert_allclose(got, want, rtol=1e-13, atol=0)
    assert np.all(got[~mask] > 0)


@pytest.mark.parametrize("N,k,iters", [(3, 2, 6), (2, 4, 4)])
def test_velocity_cheb_closed_form(N, k, iters):
    o = Oracle(N, k)
    mu = np.random.default_rng(1).uniform(0.5, 2.0, o.n_el * o.n_q)
    A = _dense_A(o, mu)
    mask = o.boundary_mask().astype(bool)
    I = ~mask
    AI = A[np.ix_(I, I)]
    MinvI = 1.0 / np.diag(AI)
    m = np.sqrt(MinvI)
    lmax = np.linalg.eigvalsh(m[:, None] * AI * m[None, :]).max()
    lmin = 0.1 * lmax
    b = np.random.default_rng(2).uniform(-1, 1, o.n_v)
    x = o.velocity_cheb(mu, b, iters, lmin, lmax)
    assert np.all(x[mask] == 0.0)
    xc = _closed_form(AI, MinvI, b[I], iters, lmin, lmax)
    assert np.linalg.norm(x[I] - xc) <= 1e-12 * np.linalg.norm(xc)


def test_velocity_eigmax_matrix_powers():
    o = Oracle(2, 2)
    mu = np.random.default_rng(4).uniform(0.5, 2.0, o.n_el * o.n_q)
    A = _dense_A(o, mu)
    mask = o.boundary_mask().astype(bool)
    Am = A.copy(); Am[mask, :] = 0; Am[:, mask] = 0
    Minv = np.where(mask, 0.0, 1.0 / np.where(mask, 1.0, np.diag(A)))
    MK = Minv[:, None] * Am
    v0 = np.random.default_rng(5).standard_normal(o.n_v)
    for it in (1, 5):
        ref = np.linalg.norm(np.linalg.matrix_power(MK, it) @ v0) / np.linalg.norm(
            np.linalg.matrix_power(MK, it - 1) @ v0)
        assert abs(o.velocity_eigmax(mu, v0, it) - ref) <= 1e-11 * ref
