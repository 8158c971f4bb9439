"""Pins for the oracle's viscous-stress apply A(mu) (eq:stokes).

* polynomial exactness against EXACT rational integrals of 2 mu eps(u):eps(v)
  (tests/polyexact.py) -- catches a dropped factor 2, a missing transpose
  term, wrong derivative scaling 2/h or wrong detJ;
* rigid-body modes in the kernel of the unmasked operator;
* patch test (constant strain -> interior rows vanish);
* symmetry, positivity, exact power-of-two scaling in mu;
* the explicit element matrix (delta_cd form) assembled densely equals the
  quadrature apply (two formulations of the definition).
"""
from fractions import Fraction

import numpy as np
import pytest

import synth
from oracle import Oracle
from tests import polyexact as P

GLL = {2: [-1.0, 0.0, 1.0], 3: [-1.0, -1 / np.sqrt(5), 1 / np.sqrt(5), 1.0],
       4: [-1.0, -np.sqrt(3 / 7), 0.0, np.sqrt(3 / 7), 1.0]}


def node_coords(N, k):
    """Physical coordinates of all nodes (test-side closed-form GLL)."""
    nn1 = k * N + 1
    g = np.arange(nn1 ** 3)
    h = 1.0 / N
    xs = []
    for i in (g % nn1, (g // nn1) % nn1, g // (nn1 * nn1)):
        e, a = np.divmod(i, k)
        last = e == N
        e = np.where(last, N - 1, e)
        a = np.where(last, k, a)
        xs.append(h * (e + (np.take(GLL[k], a) + 1) / 2))
    return xs


def interp(N, k, field):
    x, y, z = node_coords(N, k)
    return np.concatenate([P.evaluate_np(f, x, y, z) for f in field])


def _fields(k):
    """Two polynomial vector fields in [Q_k]^3 (degree <= k per variable)."""
    u = (P.add(P.mono(1, k, 0, 1), P.mono(-2, 1, 2, 0), P.mono(Fraction(1, 3), 0, 1, k)),
         P.add(P.mono(3, 0, k, k), P.mono(1, 1, 0, 0)),
         P.add(P.mono(-1, k, k, 0), P.mono(2, 0, 0, 1), P.mono(1, 1, 1, 1)))
    v = (P.add(P.mono(2, 1, k, 0), P.mono(1, 0, 0, 2)),
         P.add(P.mono(-1, k, 1, 1), P.mono(Fraction(1, 2), 0, 2, 0)),
         P.add(P.mono(1, 0, k, k), P.mono(-3, 1, 0, k)))
    return u, v


@pytest.mark.parametrize("N,k", [(1, 2), (2, 2), (3, 2), (1, 4), (2, 4), (2, 3)])
def test_A_exact_on_polynomials_constant_mu(N, k):
    o = Oracle(N, k)
    mu = Fraction(3, 2)
    mu_q = np.full(o.n_el * o.n_q, float(mu))
    u, v = _fields(k)
    uh, vh = interp(N, k, u), interp(N, k, v)
    got = vh @ o.apply_A(mu_q, uh, nomask=True)
    exact = float(P.strain_energy(u, v, mu))
    assert abs(got - exact) <= 1e-12 * max(1.0, abs(exact)), (got, exact)


@pytest.mark.parametrize("N,k", [(2, 2), (3, 2), (2, 4)])
def test_A_exact_with_dirichlet_bubbles(N, k):
    """Fields vanishing on the boundary: masked apply == exact energy."""
    o = Oracle(N, k)
    b = P.mul(P.mul(P.add(P.mono(1, 1), P.mono(-1, 2)), P.add(P.mono(1, 0, 1), P.mono(-1, 0, 2))),
              P.add(P.mono(1, 0, 0, 1), P.mono(-1, 0, 0, 2)))  # x(1-x)y(1-y)z(1-z), in Q2
    u = (b, P.scale(b, 2), P.scale(b, -1))
    v = (P.scale(b, 3), b, b)
    mu = 5
    mu_q = np.full(o.n_el * o.n_q, float(mu))
    uh, vh = interp(N, k, u), interp(N, k, v)
    got = vh @ o.apply_A(mu_q, uh)
    exact = float(P.strain_energy(u, v, mu))
    assert abs(got - exact) <= 1e-12 * abs(exact)


@pytest.mark.parametrize("N,k", [(2, 2), (3, 2), (2, 4)])
def test_rigid_modes_in_kernel(N, k):
    o = Oracle(N, k)
    cfg = synth.CONFIGS["C2"]
    mu_q = synth.make_inputs(cfg, 0, N=N)["mu_q"] if k == 2 else np.random.default_rng(1).uniform(0.5, 2, o.n_el * o.n_q)
    x, y, z = node_coords(N, k)
    one, zero = np.ones_like(x), np.zeros_like(x)
    modes = [(one, zero, zero), (zero, one, zero), (zero, zero, one),
             (-y, x, zero), (-z, zero, x), (zero, -z, y)]
    scale = np.abs(mu_q).max() * N
    for m in modes:
        r = o.apply_A(mu_q, np.concatenate(m), nomask=True)
        assert np.abs(r).max() <= 1e-12 * scale


@pytest.mark.parametrize("k", [2, 4])
def test_patch_test_constant_strain(k):
    N = 3
    o = Oracle(N, k)
    mu_q = np.full(o.n_el * o.n_q, 0.7)
    x, y, z = node_coords(N, k)
    u = np.concatenate([0.3 * x + 0.2 * y - z, 2 * y + 0.5 * z, -0.4 * x + y + 0.1 * z])
    r = o.apply_A(mu_q, u, nomask=True)
    interior = o.boundary_mask() == 0
    assert np.abs(r[interior]).max() <= 1e-13
    assert np.abs(r[~interior]).max() > 1e-3   # boundary tractions do not vanish


def test_symmetric_positive_scaling_C2_like():
    N = 4
    inp = synth.make_inputs("C2", 0, N=N)
    o = Oracle(N, 2)
    rng = np.random.default_rng(7)
    u, v = rng.uniform(-1, 1, o.n_v), rng.uniform(-1, 1, o.n_v)
    Au, Av = o.apply_A(inp["mu_q"], u), o.apply_A(inp["mu_q"], v)
    assert abs(v @ Au - u @ Av) <= 1e-13 * np.linalg.norm(Au) * np.linalg.norm(v)
    mask = o.boundary_mask() == 0
    assert u[mask] @ Au[mask] > 0
    # exact scaling by powers of two
    assert np.array_equal(o.apply_A(16 * inp["mu_q"], u), 16 * Au)
    assert np.array_equal(o.apply_A(2 * inp["mu_q"], u), 2 * Au)


@pytest.mark.parametrize("N,k", [(1, 2), (2, 2), (1, 4)])
def test_dense_assembly_equals_apply(N, k):
    o = Oracle(N, k)
    rng = np.random.default_rng(3)
    mu_q = rng.uniform(0.1, 10, o.n_el * o.n_q)
    m = o.dofmap().reshape(o.n_el, o.n_q)
    nq = o.n_q
    A = np.zeros((o.n_v, o.n_v))
    for e in range(o.n_el):
        Ae = o.element_A_matrix(mu_q[e * nq:(e + 1) * nq])
        assert np.allclose(Ae, Ae.T, rtol=0, atol=1e-12 * np.abs(Ae).max())
        idx = np.concatenate([c * o.n_nodes + m[e] for c in range(3)])
        A[np.ix_(idx, idx)] += Ae
    u = rng.uniform(-1, 1, o.n_v)
    np.testing.assert_allclose(o.apply_A(mu_q, u, nomask=True), A @ u, rtol=0, atol=1e-12 * np.abs(A).max())
    mask = o.boundary_mask().astype(bool)
    Am = A.copy(); Am[mask, :] = 0; Am[:, mask] = 0
    np.testing.assert_allclose(o.apply_A(mu_q, u), Am @ u, rtol=0, atol=1e-12 * np.abs(A).max())
    # masked A is SPD on the interior block
    if (~mask).sum():
        ev = np.linalg.eigvalsh(A[np.ix_(~mask, ~mask)])
        assert ev.min() > 0


def test_sampled_equals_full():
    inp = synth.make_inputs("C2", 1, N=5)
    o = Oracle(5, 2)
    y = o.apply_A(inp["mu_q"], inp["u"])
    dofs = np.random.default_rng(0).choice(o.n_v, 300, replace=False)
    np.testing.assert_array_equal(o.apply_A_sampled(inp["mu_q"], inp["u"], dofs), y[dofs])
