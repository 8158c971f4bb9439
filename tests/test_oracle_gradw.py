"""Pins for the oracle's viscosity-gradient wBFBT weights (rmk:wbfbt-visc-grad,
PAPER.md:2132-2150; grad mu from the element's Gauss-point interpolant, reading R17):

* mu a polynomial of degree <= k in each variable is reproduced exactly by the
  Gauss-point interpolant, so mu_eff = sqrt(mu^2 + |grad mu|^2) must equal the
  closed form evaluated with the analytic gradient (k = 2 and k = 4);
* constant mu: grad mu = 0, so mu_eff = mu and the lumped masses are the
  eq:wbfbt ones;
* scaling mu by 16 scales mu_eff by 16 bit-exactly (the weights' homogeneity).
"""
import numpy as np
import pytest

from oracle import Oracle


def _gauss_coords(o):
    """Physical coordinates of every Gauss point, [n_el * n_q, 3], element-major, q x-fastest."""
    N, n1 = o.N, o.k + 1
    xg = o.tables()["xg"][:n1]
    h = 1.0 / N
    e = np.arange(o.n_el)
    ex, ey, ez = e % N, (e // N) % N, e // (N * N)
    q = np.arange(n1 ** 3)
    qx, qy, qz = q % n1, (q // n1) % n1, q // (n1 * n1)
    X = h * (ex[:, None] + (xg[qx][None, :] + 1) / 2)
    Y = h * (ey[:, None] + (xg[qy][None, :] + 1) / 2)
    Z = h * (ez[:, None] + (xg[qz][None, :] + 1) / 2)
    return X.ravel(), Y.ravel(), Z.ravel()


@pytest.mark.parametrize("N,k", [(3, 2), (2, 4)])
def test_grad_weights_exact_for_polynomial_mu(N, k):
    o = Oracle(N, k)
    x, y, z = _gauss_coords(o)
    if k == 2:  # degree <= 2 in each variable
        mu = 2.0 + 0.3 * x + 0.5 * y ** 2 - 0.2 * x * z + 0.1 * x * y * z + 0.4 * z ** 2 * x ** 2
        gx = 0.3 - 0.2 * z + 0.1 * y * z + 0.8 * z ** 2 * x
        gy = 1.0 * y + 0.1 * x * z
        gz = -0.2 * x + 0.1 * x * y + 0.8 * z * x ** 2
    else:  # degree <= 4 in each variable
        mu = 3.0 + x ** 4 - 0.5 * y ** 3 * z + 0.25 * (x * y * z) ** 2
        gx = 4 * x ** 3 + 0.5 * x * (y * z) ** 2
        gy = -1.5 * y ** 2 * z + 0.5 * y * (x * z) ** 2
        gz = -0.5 * y ** 3 + 0.5 * z * (x * y) ** 2
    want = np.sqrt(mu ** 2 + gx ** 2 + gy ** 2 + gz ** 2)
    got = o.grad_weights(mu)
    np.testing.assert_allclose(got, want, rtol=2e-13, atol=0)


def test_grad_weights_constant_mu_gives_sqrt_weights():
    o = Oracle(3, 2)
    mu = np.full(o.n_el * o.n_q, 7.25)
    eff = o.grad_weights(mu)
    assert np.max(np.abs(eff - mu)) <= 1e-15 * 7.25
    a = o.lumped(mu, 1.5, 2.0)
    b = o.lumped(eff, 1.5, 2.0)
    for key in ("Cw", "Dw"):
        np.testing.assert_allclose(b[key], a[key], rtol=1e-15, atol=0)


def test_grad_weights_homogeneous_bitexact():
    o = Oracle(4, 2)
    mu = np.exp(np.random.default_rng(3).uniform(-4, 4, o.n_el * o.n_q))
    assert np.array_equal(o.grad_weights(16.0 * mu), 16.0 * o.grad_weights(mu))


def test_setup_grad_keeps_mu_for_A():
    """weights="grad" changes only the lumped masses; A still uses mu (eq:wbfbt's A)."""
    o = Oracle(2, 2)
    rng = np.random.default_rng(0)
    mu = rng.uniform(0.5, 2.0, o.n_el * o.n_q)
    s1 = o.setup(mu, weights="sqrt")
    s2 = o.setup(mu, weights="grad")
    assert not np.array_equal(s1["Cw"], s2["Cw"])
    np.testing.assert_array_equal(s2["Cw"], o.lumped(o.grad_weights(mu))["Cw"])
    assert np.array_equal(o.mu_q, mu)
