"""Pins of the Stokes right-hand side: the multi-sinker forcing
f = (0, 0, beta (chi - 1)) (SPEC.md:121-129 examples) and its load vector."""
from fractions import Fraction

import numpy as np
import pytest

import synth
from oracle import Oracle
from oracle import stokes as ost


def test_forcing_examples():
    c = np.array([[0.3, 0.6, 0.2]])
    # x = c_1 -> last component -10; chi = 1 -> 0
    N, k = 1, 2
    f = synth.forcing_at_quadrature(N, k, c, 200.0, 0.1).reshape(3, 1, 27)
    assert np.all(f[0] == 0.0) and np.all(f[1] == 0.0) and np.all(f[2] <= 0.0)
    far = synth.forcing_at_quadrature(1, 2, np.array([[5.0, 5.0, 5.0]]), 200.0, 0.1)
    assert np.allclose(far, 0.0, atol=1e-300)
    near = 10.0 * (synth.chi(c[0], c, 200.0, 0.1) - 1.0)
    assert near == -10.0


def test_load_vector_constant_force_is_lumped_mass():
    """f = (1, 2, 3): F_c = c * (row sums of the unweighted mass) = c * lumped(1) (R8)."""
    for N, k in ((3, 2), (2, 4)):
        o = Oracle(N, k)
        fq = np.concatenate([np.full(o.n_el * o.n_q, v) for v in (1.0, 2.0, 3.0)])
        F = ost.load_vector(o, fq)
        M = o.lumped(np.ones(o.n_el * o.n_q))["Cw"]
        mask = o.boundary_mask().astype(bool)
        for c in range(3):
            ref = (c + 1) * M
            got = F[c * o.n_nodes:(c + 1) * o.n_nodes]
            assert np.allclose(got[~mask[:o.n_nodes]], ref[~mask[:o.n_nodes]], rtol=1e-13, atol=0)


def test_load_vector_integrates_polynomials_exactly():
    """sum_g F_unmasked[g] = int f for f = x y^2 z (degree <= 2k-1 per variable: Gauss exact):
    int_0^1 x dx int y^2 dy int z dz = 1/2 * 1/3 * 1/2 = 1/12."""
    N, k = 3, 2
    o = Oracle(N, k)
    t = o.tables()
    xg = t["xg"]
    h = 1.0 / N
    fz = np.zeros((o.n_el, o.n_q))
    for e in range(o.n_el):
        ex, ey, ez = e % N, (e // N) % N, e // (N * N)
        for q in range(o.n_q):
            qx, qy, qz = q % 3, (q // 3) % 3, q // 9
            x, y, z = h * (ex + (xg[qx] + 1) / 2), h * (ey + (xg[qy] + 1) / 2), h * (ez + (xg[qz] + 1) / 2)
            fz[e, q] = x * y * y * z
    fq = np.concatenate([np.zeros(o.n_el * o.n_q), np.zeros(o.n_el * o.n_q), fz.ravel()])
    F = ost.load_vector(o, fq, mask=False)
    assert F[2 * o.n_nodes:].sum() == pytest.approx(float(Fraction(1, 12)), rel=1e-14)
    assert np.all(F[:2 * o.n_nodes] == 0.0)


def test_python_fgmres_matches_c_core_and_is_minimal_residual():
    """The numpy FGMRES (oracle/stokes.py) against the C oracle's core on a dense system with
    a fixed preconditioner, and the GMRES property: after j iterations (no restart) the
    residual is the least-squares minimum over the preconditioned Krylov space."""
    import oracle
    rng = np.random.default_rng(0)
    n = 30
    A = rng.standard_normal((n, n)) + 8 * np.eye(n)
    Pm = np.diag(1.0 / np.diag(A))
    b = rng.standard_normal(n)
    x, it, rr = ost.fgmres(lambda v: A @ v, lambda v: Pm @ v, b, 40, 6, 0.0)
    xc, itc, rrc = oracle.fgmres_dense(A, Pm, b, 40, 6, 0.0)
    assert it == itc == 6 and np.allclose(x, xc, rtol=0, atol=1e-12 * np.linalg.norm(xc))
    # minimal residual over span{(AP)^i P... }: x = P V y with V the Krylov basis of AP
    W = [b]
    for _ in range(5):
        W.append(A @ (Pm @ W[-1]))
    Kb = Pm @ np.array(W).T
    y, *_ = np.linalg.lstsq(A @ Kb, b, rcond=None)
    assert np.linalg.norm(b - A @ (Kb @ y)) == pytest.approx(np.linalg.norm(b - A @ x), rel=1e-8)
