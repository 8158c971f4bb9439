"""Pins for the oracle's dof map, boundary mask and boundary-element set.

Closed forms (SURVEY.md 8(c) pins), conformity of the
numbering (a shared node has one physical position seen from every element),
and brute-force enumeration on small meshes.
"""
import numpy as np
import pytest

from oracle import Oracle


def _node_xyz(o: Oracle, g):
    """Physical position of node g from its grid index (test-side GLL closed form)."""
    k, N = o.k, o.N
    xn = {2: [-1.0, 0.0, 1.0], 4: [-1.0, -np.sqrt(3 / 7), 0.0, np.sqrt(3 / 7), 1.0],
          3: [-1.0, -1 / np.sqrt(5), 1 / np.sqrt(5), 1.0]}[k]
    nn1 = k * N + 1
    idx = [g % nn1, (g // nn1) % nn1, g // (nn1 * nn1)]
    h = 1.0 / N
    out = []
    for i in idx:
        e, a = np.divmod(i, k)
        last = e == N
        e, a = np.where(last, N - 1, e), np.where(last, k, a)
        out.append(h * (e + (np.take(xn, a) + 1) / 2))
    return np.array(out).T


@pytest.mark.parametrize("N,k", [(1, 2), (3, 2), (4, 2), (2, 4), (3, 3)])
def test_dofmap_conforming_and_complete(N, k):
    o = Oracle(N, k)
    m = o.dofmap().reshape(o.n_el, o.n_q)
    n1 = k + 1
    xn = {2: [-1.0, 0.0, 1.0], 4: [-1.0, -np.sqrt(3 / 7), 0.0, np.sqrt(3 / 7), 1.0],
          3: [-1.0, -1 / np.sqrt(5), 1 / np.sqrt(5), 1.0]}[k]
    h = 1.0 / N
    # every node is hit, every element's local nodes are distinct
    assert set(np.unique(m)) == set(range(o.n_nodes))
    assert all(len(set(row)) == o.n_q for row in m)
    # the node each (e, a) maps to sits at the element-local physical position
    for e in range(o.n_el):
        ex, ey, ez = e % N, (e // N) % N, e // (N * N)
        a = np.arange(o.n_q)
        ax, ay, az = a % n1, (a // n1) % n1, a // (n1 * n1)
        loc = np.stack([h * (ex + (np.take(xn, ax) + 1) / 2), h * (ey + (np.take(xn, ay) + 1) / 2),
                        h * (ez + (np.take(xn, az) + 1) / 2)], -1)
        np.testing.assert_allclose(_node_xyz(o, m[e]), loc, atol=1e-15)
    # multiplicity: a node shared by c_x*c_y*c_z elements (c = 2 on interior element faces)
    counts = np.bincount(m.ravel(), minlength=o.n_nodes)
    nn1 = k * N + 1
    g = np.arange(o.n_nodes)
    mult = np.ones(o.n_nodes, dtype=int)
    for i in (g % nn1, (g // nn1) % nn1, g // (nn1 * nn1)):
        mult *= np.where((i % k == 0) & (i > 0) & (i < nn1 - 1), 2, 1)
    np.testing.assert_array_equal(counts, mult)


@pytest.mark.parametrize("N,k", [(1, 2), (4, 2), (16, 2), (3, 4), (5, 3)])
def test_mask_counts(N, k):
    o = Oracle(N, k)
    mask = o.boundary_mask()
    assert mask.sum() == 3 * ((k * N + 1) ** 3 - (k * N - 1) ** 3)
    # same mask for the three components
    nn = o.n_nodes
    assert np.array_equal(mask[:nn], mask[nn:2 * nn]) and np.array_equal(mask[:nn], mask[2 * nn:])


def test_interior_dof_count_spec_example():
    # 3D, k=2, ell=4 -> 3 * 31^3 = 89,373 interior velocity dofs
    o = Oracle(16, 2)
    assert o.n_v - o.boundary_mask().sum() == 89373


@pytest.mark.parametrize("N,expect", [(4, 56), (2, 8), (3, 26), (64, 23816)])
def test_boundary_element_count(N, expect):
    # |D| = N^3 - (N-2)^3 (eq:bdramp set D)
    o = Oracle(N, 2)
    assert int(o.boundary_elements().sum()) == expect == N ** 3 - max(N - 2, 0) ** 3
