"""Pins for the oracle on the box mesh N x N x Nz (z-stacked cubes of side 1/N): the global
mesh of the slab decomposition (reading R24).

Every formula of the oracle is per element, so the box changes only the structure code
(element / node numbering, the boundary).  The pins are chosen to fail if any of those still
assumes a cube:

* counts and the boundary against closed forms on the box;
* A against EXACT rational integrals of 2 mu eps(u):eps(v) over [0,1]^2 x [0, Nz/N]
  (tests/polyexact.py), unmasked, and masked with bubbles that vanish on the box boundary;
* B against exact per-element integrals of -q_m div u on every element of the box;
* adjointness, the divergence theorem (B^T of the constant pressure is 0 under the mask);
* lumped masses: separable closed form with the z weights of Nz elements;
* boundary amplification touches exactly the elements with an index 0 / N-1 / Nz-1;
* the sampled A equals the full A on the box;
* Nz = N reproduces the cube oracle bit for bit.
"""
from fractions import Fraction
from math import sqrt

import numpy as np
import pytest

from oracle import Oracle
from tests import polyexact as P
from tests.test_oracle_A import GLL, _fields
from tests.test_oracle_B import _legendre_of_xi, _xi_poly
from tests.test_oracle_lumped import _one_d_weights


def box_coords(N, Nz, k):
    nn1, nnz = k * N + 1, k * Nz + 1
    g = np.arange(nn1 * nn1 * nnz)
    h = 1.0 / N
    xs = []
    for i, ne in ((g % nn1, N), ((g // nn1) % nn1, N), (g // (nn1 * nn1), Nz)):
        e, a = np.divmod(i, k)
        last = e == ne
        e = np.where(last, ne - 1, e)
        a = np.where(last, k, a)
        xs.append(h * (e + (np.take(GLL[k], a) + 1) / 2))
    return xs


def interp_box(N, Nz, k, field):
    x, y, z = box_coords(N, Nz, k)
    return np.concatenate([P.evaluate_np(f, x, y, z) for f in field])


def energy_box(u, v, mu, Lz) -> Fraction:
    tot = {}
    for i in range(3):
        for j in range(3):
            eu = P.scale(P.add(P.diff(u[i], j), P.diff(u[j], i)), Fraction(1, 2))
            ev = P.scale(P.add(P.diff(v[i], j), P.diff(v[j], i)), Fraction(1, 2))
            tot = P.add(tot, P.mul(eu, ev))
    return 2 * Fraction(mu) * P.integrate_box(tot, (0, 0, 0), (1, 1, Lz))


@pytest.mark.parametrize("N,Nz,k", [(2, 4, 2), (3, 1, 2), (2, 6, 2), (1, 2, 4), (2, 3, 3)])
def test_counts_and_boundary(N, Nz, k):
    o = Oracle(N, k, Nz=Nz)
    nn1, nnz = k * N + 1, k * Nz + 1
    assert (o.n_el, o.n_nodes, o.n_v) == (N * N * Nz, nn1 * nn1 * nnz, 3 * nn1 * nn1 * nnz)
    assert o.n_p == o.n_m * N * N * Nz
    m = o.boundary_mask().reshape(3, nnz, nn1, nn1)
    interior = max(nn1 - 2, 0) ** 2 * max(nnz - 2, 0)
    assert int((m == 0).sum()) == 3 * interior
    assert m[:, 0].all() and m[:, -1].all() and m[:, :, 0].all() and m[:, :, :, -1].all()
    dm = o.dofmap().reshape(o.n_el, o.n_q)
    assert dm.min() == 0 and dm.max() == o.n_nodes - 1
    # last element's last node is the last node; element (0,0,1) starts k node layers up
    assert dm[-1, -1] == o.n_nodes - 1
    if Nz > 1:
        assert dm[N * N, 0] == k * nn1 * nn1
    fl = o.boundary_elements().reshape(Nz, N, N)
    expect = np.zeros((Nz, N, N), dtype=bool)
    expect[0] = expect[-1] = True
    expect[:, 0] = expect[:, -1] = True
    expect[:, :, 0] = expect[:, :, -1] = True
    np.testing.assert_array_equal(fl.astype(bool), expect)


@pytest.mark.parametrize("N,Nz,k", [(2, 4, 2), (2, 1, 2), (3, 5, 2), (1, 3, 4), (2, 3, 3)])
def test_A_exact_on_polynomials_box(N, Nz, k):
    o = Oracle(N, k, Nz=Nz)
    mu = Fraction(3, 2)
    mu_q = np.full(o.n_el * o.n_q, float(mu))
    u, v = _fields(k)
    uh, vh = interp_box(N, Nz, k, u), interp_box(N, Nz, k, v)
    got = vh @ o.apply_A(mu_q, uh, nomask=True)
    exact = float(energy_box(u, v, mu, Fraction(Nz, N)))
    assert abs(got - exact) <= 1e-12 * max(1.0, abs(exact)), (got, exact)


@pytest.mark.parametrize("N,Nz,k", [(2, 4, 2), (3, 2, 2), (2, 3, 4)])
def test_A_dirichlet_bubbles_box(N, Nz, k):
    """Fields vanishing on the box boundary: the masked apply gives the exact energy (a mask
    on a wrong z plane would cut the bubble)."""
    o = Oracle(N, k, Nz=Nz)
    Lz = Fraction(Nz, N)
    b = P.mul(P.mul(P.add(P.mono(1, 1), P.mono(-1, 2)), P.add(P.mono(1, 0, 1), P.mono(-1, 0, 2))),
              P.add(P.mono(Lz, 0, 0, 1), P.mono(-1, 0, 0, 2)))  # x(1-x) y(1-y) z(Lz-z)
    u = (b, P.scale(b, 2), P.scale(b, -1))
    v = (P.scale(b, 3), b, b)
    mu_q = np.full(o.n_el * o.n_q, 5.0)
    uh, vh = interp_box(N, Nz, k, u), interp_box(N, Nz, k, v)
    exact = float(energy_box(u, v, 5, Lz))
    assert abs(vh @ o.apply_A(mu_q, uh) - exact) <= 1e-12 * abs(exact)
    # and the masked operator ignores boundary values of its input
    rng = np.random.default_rng(0)
    noise = rng.standard_normal(o.n_v) * o.boundary_mask()
    np.testing.assert_array_equal(o.apply_A(mu_q, uh + noise), o.apply_A(mu_q, uh))


@pytest.mark.parametrize("N,Nz,k", [(2, 3, 2), (1, 2, 4)])
def test_B_exact_on_polynomials_box(N, Nz, k):
    o = Oracle(N, k, Nz=Nz)
    modes = o.tables()["modes"]
    u, _ = _fields(k)
    uh = interp_box(N, Nz, k, u)
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


@pytest.mark.parametrize("N,Nz,k", [(3, 5, 2), (2, 3, 4)])
def test_adjoint_and_constant_pressure_box(N, Nz, k):
    o = Oracle(N, k, Nz=Nz)
    rng = np.random.default_rng(5)
    u, p = rng.standard_normal(o.n_v), rng.standard_normal(o.n_p)
    lhs, rhs = o.apply_B(u) @ p, u @ o.apply_BT(p)
    assert abs(lhs - rhs) <= 1e-13 * max(abs(lhs), 1.0)
    z0 = np.zeros((o.n_el, o.n_m))
    z0[:, 0] = 1.0
    assert np.abs(o.apply_BT(z0.ravel())).max() <= 1e-15
    # projection removes exactly the mean of the mode-0 entries over the box's elements
    v = rng.standard_normal(o.n_p)
    pv = o.project(v).reshape(o.n_el, o.n_m)
    assert abs(pv[:, 0].sum()) <= 1e-12
    np.testing.assert_array_equal(pv[:, 1:], v.reshape(o.n_el, o.n_m)[:, 1:])


@pytest.mark.parametrize("N,Nz,k", [(2, 4, 2), (4, 2, 2), (2, 3, 4)])
def test_lumped_unit_weight_closed_form_box(N, Nz, k):
    o = Oracle(N, k, Nz=Nz)
    lm = o.lumped(np.ones(o.n_el * o.n_q))
    w1 = _one_d_weights(N, k)
    # z: Nz elements of the same side h = 1/N
    loc = {2: np.array([1, 4, 1]) / 3.0, 4: np.array([1 / 10, 49 / 90, 32 / 45, 49 / 90, 1 / 10])}[k]
    wz = np.zeros(k * Nz + 1)
    for e in range(Nz):
        wz[k * e:k * e + k + 1] += loc / (2 * N)
    expect = (wz[:, None, None] * w1[None, :, None] * w1[None, None, :]).ravel()
    np.testing.assert_allclose(lm["Cw"], expect, rtol=1e-14, atol=0)
    assert lm["Cw"].sum() == pytest.approx(Nz / N, rel=1e-13)  # the box volume
    # amplification a_r = 3 only on boundary-touching elements: total = vol + 2 vol(boundary layer)
    lm3 = o.lumped(np.ones(o.n_el * o.n_q), 1.0, 3.0)
    n_int = max(N - 2, 0) ** 2 * max(Nz - 2, 0)
    vol_el = 1.0 / N ** 3
    assert lm3["Dw"].sum() == pytest.approx(vol_el * (n_int + 3 * (o.n_el - n_int)), rel=1e-13)
    np.testing.assert_array_equal(lm3["Cw"], lm["Cw"])


def test_sampled_A_equals_full_on_box():
    N, Nz, k = 3, 5, 2
    o = Oracle(N, k, Nz=Nz)
    rng = np.random.default_rng(2)
    mu_q = rng.uniform(0.1, 10.0, o.n_el * o.n_q)
    u = rng.standard_normal(o.n_v)
    y = o.apply_A(mu_q, u)
    dofs = rng.choice(o.n_v, 300, replace=False)
    np.testing.assert_allclose(o.apply_A_sampled(mu_q, u, dofs), y[dofs], rtol=0, atol=1e-12 * np.abs(y).max())


@pytest.mark.parametrize("N,k", [(3, 2), (2, 4)])
def test_cube_is_the_box_with_Nz_equal_N(N, k):
    a, b = Oracle(N, k), Oracle(N, k, Nz=N)
    rng = np.random.default_rng(9)
    mu_q = rng.uniform(0.1, 10.0, a.n_el * a.n_q)
    u, p = rng.standard_normal(a.n_v), rng.standard_normal(a.n_p)
    np.testing.assert_array_equal(a.apply_A(mu_q, u), b.apply_A(mu_q, u))
    np.testing.assert_array_equal(a.apply_B(u), b.apply_B(u))
    np.testing.assert_array_equal(a.apply_BT(p), b.apply_BT(p))
    sa, sb = a.setup(mu_q, 2.0, 3.0), b.setup(mu_q, 2.0, 3.0)
    for key in ("Cw", "Dw", "Cinv", "Dinv", "diagKl", "diagKr"):
        np.testing.assert_array_equal(sa[key], sb[key])
    np.testing.assert_array_equal(a.wbfbt(p, 5), b.wbfbt(p, 5))
