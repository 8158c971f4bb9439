"""Pins of the Schur-complement variants' oracle (oracle/schur.py)."""
from math import sqrt

import numpy as np

from oracle import Oracle
from oracle import schur as osc
from tests.test_oracle_B import _dense_B
from tests.test_oracle_wbfbt import _pinv_deflated, _z0


def test_mp_constant_mu_is_scaled_identity():
    """Orthonormal modes: int_e q_i q_j = (h/2)^3 delta_ij, so M_p(1/mu)^-1 = mu (2/h)^3 I."""
    for N, k in ((2, 2), (1, 4)):
        o = Oracle(N, k)
        r = np.random.default_rng(0).uniform(-1, 1, o.n_p)
        z = osc.mp_inverse_apply(o, np.full(o.n_el * o.n_q, 3.0), r)
        assert np.allclose(z, 3.0 * (2.0 * N) ** 3 * r, rtol=1e-13)


def test_mp_linear_weight_closed_form():
    """1/mu = a + b xi_x on the reference element (degree 1: Gauss exact):
    M[i][j] = (h/2)^3 (a delta_ij + b int xi_x q_i q_j), int xi L0 L1 = 1/sqrt(3) -> M[0][1] = b (h/2)^3/sqrt(3)."""
    o = Oracle(1, 2)
    t = o.tables()
    xg = t["xg"]
    a, b = 2.0, 0.5
    mu = np.array([1.0 / (a + b * xg[q % 3]) for q in range(27)])
    M = osc.mp_blocks(o, mu)[0]
    h3 = 0.5 ** 3
    ref = h3 * a * np.eye(4)
    ref[0, 1] = ref[1, 0] = h3 * b / sqrt(3)
    assert np.allclose(M, ref, atol=1e-15)


def _mild(o, seed=0):
    return np.random.default_rng(seed).uniform(0.5, 2.0, o.n_el * o.n_q)


def test_dabfbt_converged_equals_dense_formula():
    """eq:bfbt with C = D = diag(A) by dense pseudo-inverses, N = 2."""
    o = Oracle(2, 2)
    mu = _mild(o, 1)
    D = osc.DiagABFBT(o, mu)
    B = _dense_B(o)
    n_v = o.n_v
    A = np.zeros((n_v, n_v))
    for j in range(n_v):
        e = np.zeros(n_v)
        e[j] = 1.0
        A[:, j] = o.apply_A(mu, e)
    X = D.X
    K = B @ (X[:, None] * B.T)
    Kp = _pinv_deflated(K, _z0(o))
    r = o.project(np.random.default_rng(2).uniform(-1, 1, o.n_p))
    ref = Kp @ (B @ (X * (A @ (X * (B.T @ (Kp @ r))))))
    # the smallest PCG count at the residual floor (CG past convergence drifts under the
    # fixed-count rule, as tests/test_oracle_wbfbt.converged_iters notes)
    it = next(i for i in range(5, 200, 5) if np.linalg.norm(K @ D.poisson(r, i) - r) < 1e-12 * np.linalg.norm(r))
    z = D.apply(r, it)
    assert np.linalg.norm(z - ref) <= 1e-8 * np.linalg.norm(ref)


def test_dabfbt_scale_invariance_bitexact():
    """diag(A) and A scale with mu, so dABFBT(16 mu) = 16 dABFBT(mu) bit-exactly."""
    o = Oracle(3, 2)
    mu = _mild(o, 3)
    r = np.random.default_rng(4).uniform(-1, 1, o.n_p)
    z1 = osc.DiagABFBT(o, mu).apply(r, 7)
    z2 = osc.DiagABFBT(o, 16.0 * mu).apply(r, 7)
    assert np.array_equal(z2, 16.0 * z1)
