"""Pins of the seeded input generator synth/ (Sec. 2.1):
the multi-sinker indicator and viscosity at the worked examples the SPEC derives from the
paper's formula, the quadrature-point placement, layout and the seeding contract."""
from math import exp, sqrt

import numpy as np
import pytest

import synth


def test_chi_examples():
    c = np.array([[0.3, 0.6, 0.2]])
    # x = c_1: factor 1 - exp(0) = 0
    assert synth.chi(c[0], c, 200.0, 0.1) == 0.0
    # n = 0: empty product = 1
    assert synth.chi(np.array([0.1, 0.2, 0.3]), np.zeros((0, 3)), 200.0, 0.1) == 1.0
    # |c - x| = omega/2 + 0.1, delta = 200: 1 - exp(-2) ~ 0.8647
    x = c[0] + np.array([0.0, 0.05 + 0.1, 0.0])
    v = float(synth.chi(x, c, 200.0, 0.1))
    assert v == pytest.approx(1 - exp(-2.0), rel=1e-14) and round(v, 4) == 0.8647
    # inside the ball of radius omega/2 the factor is exactly 0 (max(0, .))
    assert synth.chi(c[0] + 0.049, c, 200.0, 0.1) == 0.0 or synth.chi(c[0] + 0.02, c, 200.0, 0.1) == 0.0
    # product over sinkers
    c2 = np.array([[0.3, 0.6, 0.2], [0.8, 0.1, 0.5]])
    y = np.array([0.5, 0.5, 0.5])
    f = [1 - exp(-200 * max(0.0, np.linalg.norm(y - ci) - 0.05) ** 2) for ci in c2]
    assert synth.chi(y, c2, 200.0, 0.1) == pytest.approx(f[0] * f[1], rel=1e-14)


def test_viscosity_examples():
    c = np.array([[0.3, 0.6, 0.2]])
    dr = 1e4
    mn, mx = dr ** -0.5, dr ** 0.5
    # DR 1e4, x = c_1 -> mu = 1e2
    assert synth.viscosity(c[0], c, 200.0, 0.1, mn, mx) == pytest.approx(1e2, rel=1e-15)
    # far from all sinkers -> mu_min
    far = synth.viscosity(np.array([1.0, 0.0, 1.0]), c, 200.0, 0.1, mn, mx)
    assert far == pytest.approx(1e-2, rel=1e-12)
    # n = 0, DR 1e6 -> mu = 1e-3 everywhere
    pts = np.random.default_rng(0).random((50, 3))
    assert np.all(synth.viscosity(pts, np.zeros((0, 3)), 200.0, 0.1, 1e-3, 1e3) == 1e-3)


def test_quadrature_points_and_layout():
    """mu_q[e*n_q + q] = mu(h (e_idx + (xi_q + 1)/2)), e = ex + N(ey + N ez), q x-fastest, with the
    3-point Gauss rule xi in {-sqrt(3/5), 0, sqrt(3/5)} (closed form, not numpy's table)."""
    cfg = synth.Config("T", 3, 2, 5, 200.0, 0.1, 1e-3, 1e3, 1)
    rng = np.random.Generator(np.random.PCG64(4))
    cen = synth.sinker_centers(rng, 5)
    N, k = 3, 2
    mu = synth.viscosity_at_quadrature(N, k, cen, 200.0, 0.1, 1e-3, 1e3)
    assert mu.shape == (N ** 3 * 27,)
    xi = [-sqrt(3 / 5), 0.0, sqrt(3 / 5)]
    h = 1 / N
    for e in (0, 5, 13, 26):
        ex, ey, ez = e % N, (e // N) % N, e // (N * N)
        for q in (0, 1, 4, 13, 20, 26):
            qx, qy, qz = q % 3, (q // 3) % 3, q // 9
            x = np.array([h * (ex + (xi[qx] + 1) / 2), h * (ey + (xi[qy] + 1) / 2), h * (ez + (xi[qz] + 1) / 2)])
            assert mu[e * 27 + q] == pytest.approx(synth.viscosity(x, cen, 200.0, 0.1, 1e-3, 1e3), rel=1e-14)
    assert mu.min() >= 1e-3 and mu.max() <= 1e3


def test_seeding_contract():
    """Deterministic; prefix property of the centres; draw order centres -> u -> p."""
    a = synth.make_inputs("C1", 3)
    b = synth.make_inputs("C1", 3)
    assert all(np.array_equal(a[key], b[key]) for key in ("centers", "mu_q", "u", "p"))
    r8 = synth.sinker_centers(np.random.Generator(np.random.PCG64(42)), 8)
    r4 = synth.sinker_centers(np.random.Generator(np.random.PCG64(42)), 4)
    assert np.array_equal(r8[:4], r4)
    rng = np.random.Generator(np.random.PCG64(3))
    rng.random((4, 3))
    s = synth.sizes(4, 2)
    assert np.array_equal(a["u"], rng.uniform(-1, 1, s["n_v"]))
    assert np.array_equal(a["p"], rng.uniform(-1, 1, s["n_p"]))
    assert np.all((a["centers"] >= 0) & (a["centers"] < 1))


def test_config_table():
    """The five BASELINE.json configs: mesh, order, sinkers, DR, PCG count."""
    t = {n: (c.N, c.k, c.n_sinkers, c.omega, c.dr, c.iters) for n, c in synth.CONFIGS.items()}
    assert t == {"C1": (4, 2, 4, 0.1, 1e4, 20), "C2": (16, 2, 8, 0.1, 1e6, 50), "C3": (32, 2, 16, 0.1, 1e8, 50),
                 "C4": (24, 4, 8, 0.1, pytest.approx(1e6), 50), "C5": (64, 2, 24, 0.05, pytest.approx(1e10), 100)}
