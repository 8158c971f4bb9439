"""Pins for the oracle's Stokes solve (reading R19): flexible GMRES
with the upper block-triangular right preconditioner of eq:precond-stokes.

* FGMRES core, identity preconditioner: after k iterations the residual is the minimum
  over the Krylov space K_k(A, b) (brute force: least squares on an explicit basis);
* exact preconditioner P = A^-1: one iteration;
* the paper's statement (BenziGolubLiesen05): with exact A^-1 and
  St = -S = -B A^-1 B^T the preconditioned Stokes system converges in two iterations
  (dense Stokes matrix of a tiny mesh, pressure null space removed);
* the FE solve with tight inner solves reaches the dense least-squares solution.
"""
import numpy as np
import pytest

import oracle
from oracle import Oracle
from tests.test_oracle_B import _dense_B
from tests.test_oracle_diagA import _dense_A
from tests.test_oracle_wbfbt import _mild_mu


@pytest.mark.parametrize("k", [1, 3, 7])
def test_fgmres_minimal_residual_over_krylov_space(k):
    rng = np.random.default_rng(k)
    n = 30
    A = rng.standard_normal((n, n)) + 6 * np.eye(n)
    b = rng.standard_normal(n)
    x, it, rr = oracle.fgmres_dense(A, np.eye(n), b, 50, k, 0.0)
    assert it == k
    Kb = np.stack([np.linalg.matrix_power(A, j) @ b for j in range(k)], axis=1)
    Q, _ = np.linalg.qr(Kb)
    y, *_ = np.linalg.lstsq(A @ Q, b, rcond=None)
    best = np.linalg.norm(b - A @ Q @ y) / np.linalg.norm(b)
    assert abs(rr - best) <= 1e-10 * max(best, 1e-3)
    assert abs(np.linalg.norm(b - A @ x) / np.linalg.norm(b) - rr) <= 1e-12


def test_fgmres_restart_and_exact_preconditioner():
    rng = np.random.default_rng(9)
    n = 25
    A = rng.standard_normal((n, n)) + 8 * np.eye(n)
    b = rng.standard_normal(n)
    x, it, rr = oracle.fgmres_dense(A, np.linalg.inv(A), b, 10, 10, 1e-12)
    assert it == 1 and rr <= 1e-12
    x, it, rr = oracle.fgmres_dense(A, np.eye(n), b, 4, 200, 1e-10)  # restarted every 4
    assert rr <= 1e-10
    np.testing.assert_allclose(x, np.linalg.solve(A, b), rtol=0, atol=1e-8 * np.abs(x).max())


def _dense_stokes(o, mu):
    A = _dense_A(o, mu)
    B = _dense_B(o)
    mask = o.boundary_mask().astype(bool)
    A[mask, :] = 0; A[:, mask] = 0
    B = B.copy(); B[:, mask] = 0
    return A, B, mask


def test_exact_block_preconditioner_two_iterations():
    o = Oracle(2, 2)
    mu = _mild_mu(o)
    A, B, mask = _dense_stokes(o, mu)
    I = ~mask
    # interior velocity block and pressures off the constant mode (the null space)
    z = np.zeros(o.n_p); z[::o.n_m] = 1.0; z /= np.linalg.norm(z)
    W = np.linalg.svd(np.eye(o.n_p) - np.outer(z, z))[0][:, :o.n_p - 1]  # basis of 1-perp
    AI, BI = A[np.ix_(I, I)], W.T @ B[:, I]
    S = BI @ np.linalg.solve(AI, BI.T)
    nv, npr = AI.shape[0], BI.shape[0]
    K = np.block([[AI, BI.T], [BI, np.zeros((npr, npr))]])
    P = np.block([[AI, BI.T], [np.zeros((npr, nv)), -S]])
    b = np.random.default_rng(1).standard_normal(nv + npr)
    x, it, rr = oracle.fgmres_dense(K, np.linalg.inv(P), b, 20, 20, 1e-10)
    assert it == 2 and rr <= 1e-10


def test_stokes_fgmres_reaches_dense_solution():
    """Tight inner solves (many smoother and PCG steps): the FE FGMRES solution equals the
    dense least-squares solution of the singular Stokes system (pressure projected)."""
    o = Oracle(2, 2)
    mu = _mild_mu(o)
    st = o.setup(mu)
    A, B, mask = _dense_stokes(o, mu)
    rng = np.random.default_rng(2)
    f = np.where(mask, 0.0, rng.uniform(-1, 1, o.n_v))
    g = np.zeros(o.n_p)
    # smoother interval from the dense spectrum of diag(A)^-1 A on the interior
    I = ~mask
    d = np.diag(A)[I]
    ev = np.linalg.eigvalsh(A[np.ix_(I, I)] / np.sqrt(d)[:, None] / np.sqrt(d)[None, :])
    u, p, it, rr = o.stokes_fgmres(f, g, 50, 50, 1e-10, 60, 60, ev.min(), ev.max())
    assert rr <= 1e-10 and it <= 25
    K = np.block([[A, B.T], [B, np.zeros((o.n_p, o.n_p))]])
    sol = np.linalg.lstsq(K, np.concatenate([f, g]), rcond=None)[0]
    us, ps = sol[:o.n_v], o.project(sol[o.n_v:])
    assert np.linalg.norm(u - us) <= 1e-8 * np.linalg.norm(us)
    assert np.linalg.norm(p - ps) <= 1e-8 * np.linalg.norm(ps)
