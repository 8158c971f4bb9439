"""Pins for the oracle's weighted lumped velocity masses C_w, D_w
(eq:lumping PAPER.md:310-323 applied to M_u(w), w = sqrt(mu);
eq:bdramp PAPER.md:2232-2245).

* w = 1 closed forms: products of 1-D nodal integrals (k=2: h/6, 2h/3,
  shared vertex h/3; k=4: (h/2){1/10, 49/90, 32/45, 49/90, 1/10});
* partition of unity: sum_g C[g] = int w dx by Gauss quadrature;
* homogeneity in w and the boundary amplification acting only on elements of D;
* Cinv = mask / C.
"""
import numpy as np
import pytest

import synth
from oracle import Oracle


def _one_d_weights(N, k):
    """Integral of each 1-D global nodal basis function of the GLL grid on [0,1]."""
    loc = {2: np.array([1, 4, 1]) / 3.0, 4: np.array([1 / 10, 49 / 90, 32 / 45, 49 / 90, 1 / 10])}[k]
    h = 1.0 / N
    w = np.zeros(k * N + 1)
    for e in range(N):
        w[k * e:k * e + k + 1] += loc * h / 2
    return w


@pytest.mark.parametrize("N,k", [(1, 2), (4, 2), (3, 4)])
def test_unit_weight_closed_form(N, k):
    o = Oracle(N, k)
    lm = o.lumped(np.ones(o.n_el * o.n_q))
    w1 = _one_d_weights(N, k)
    expect = (w1[None, None, :] * w1[None, :, None] * w1[:, None, None]).ravel()
    np.testing.assert_allclose(lm["Cw"], expect, rtol=1e-14, atol=0)
    np.testing.assert_array_equal(lm["Cw"], lm["Dw"])
    if k == 2 and N >= 2:
        h = 1.0 / N
        # interior vertex shared by 8 elements: (h/3)^3; mid-edge-of-3 mid nodes: (2h/3)^3
        nn1 = 2 * N + 1
        g_vertex = 2 + nn1 * (2 + nn1 * 2)
        g_center = 1 + nn1 * (1 + nn1 * 1)
        assert lm["Cw"][g_vertex] == pytest.approx((h / 3) ** 3, rel=1e-14)
        assert lm["Cw"][g_center] == pytest.approx((2 * h / 3) ** 3, rel=1e-14)


def test_partition_of_unity_and_homogeneity():
    N = 6
    inp = synth.make_inputs("C2", 3, N=N)
    o = Oracle(N, 2)
    lm = o.lumped(inp["mu_q"])
    _, w = np.polynomial.legendre.leggauss(3)
    wq = (w[None, None, :] * w[None, :, None] * w[:, None, None]).ravel()
    h = 1.0 / N
    integral = (np.sqrt(inp["mu_q"]).reshape(o.n_el, o.n_q) * wq[None, :]).sum() * (h / 2) ** 3
    assert lm["Cw"].sum() == pytest.approx(integral, rel=1e-13)
    # w -> 4 w exactly when mu -> 16 mu
    lm16 = o.lumped(16 * inp["mu_q"])
    np.testing.assert_array_equal(lm16["Cw"], 4 * lm["Cw"])


def test_boundary_amplification_only_on_D():
    N = 4
    o = Oracle(N, 2)
    mu = np.full(o.n_el * o.n_q, 2.0)
    base = o.lumped(mu, 1.0, 1.0)
    amp = o.lumped(mu, 3.0, 5.0)
    # nodes touched only by interior elements (all grid indices in [3, 2N-3]) are unchanged
    nn1 = 2 * N + 1
    g = np.arange(o.n_nodes)
    idx = np.stack([g % nn1, (g // nn1) % nn1, g // (nn1 * nn1)])
    inner = np.all((idx >= 3) & (idx <= 2 * N - 3), axis=0)
    np.testing.assert_array_equal(amp["Cw"][inner], base["Cw"][inner])
    # nodes touched only by boundary elements (some index <= 1 or >= 2N-1) scale by a_l, a_r
    outer = np.any((idx <= 1) | (idx >= 2 * N - 1), axis=0)
    np.testing.assert_allclose(amp["Cw"][outer], 3 * base["Cw"][outer], rtol=1e-15)
    np.testing.assert_allclose(amp["Dw"][outer], 5 * base["Dw"][outer], rtol=1e-15)
    # Cinv = mask / C
    bmask = o.boundary_mask()[:o.n_nodes].astype(bool)
    assert np.all(amp["Cinv"][bmask] == 0)
    np.testing.assert_array_equal(amp["Cinv"][~bmask], 1.0 / amp["Cw"][~bmask])


def test_nonpositive_entries_reported_on_C1():
    """Reading R9: row-sum lumping of the sqrt(mu)-weighted Q2 mass may produce
    nonpositive entries on coarse meshes; they are counted, not altered."""
    inp = synth.make_inputs("C1", 0)
    o = Oracle(4, 2)
    lm = o.lumped(inp["mu_q"])
    neg = int(((lm["Cw"] <= 0) & (o.boundary_mask()[:o.n_nodes] == 0)).sum())
    assert lm["n_nonpos_Cw"] == neg
    assert neg > 0   # C1 seed 0: K_w indefinite (SURVEY.md 8(c) ambiguity 8)
    inp2 = synth.make_inputs("C2", 0)
    assert Oracle(16, 2).lumped(inp2["mu_q"])["n_nonpos_Cw"] == 0
