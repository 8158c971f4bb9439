"""Oracle pieces of the full Stokes solve (eq:discrete-stokes,
eq:precond-stokes PAPER.md:187-204, 262-291) beyond the C oracle's FGMRES core.

TEST INFRASTRUCTURE ONLY (tests/, bench.py's reference leg).

  * load_vector: F[(c, g)] = sum_e sum_q w_q detJ f_c(x_q) phi_a(xi_q) of a body force given
    at the Gauss points (the multi-sinker forcing f = (0, 0, beta (chi - 1))),
    element contributions scatter-added in ascending element order, Dirichlet rows 0 (R6).
"""
from __future__ import annotations

import numpy as np

from . import Oracle


def load_vector(o: Oracle, fq: np.ndarray, mask: bool = True) -> np.ndarray:
    t = o.tables()
    n1, nq = o.k + 1, o.n_q
    phi, wg = t["phi"], t["wg"]  # phi[a][i] = phi_a(xg_i)
    detJ = (0.5 / o.N) ** 3
    # element-local weights W[a, q] = phi_a(xi_q) w_q (tensor products, q and a x-fastest)
    a_idx = np.arange(nq)
    ax, ay, az = a_idx % n1, (a_idx // n1) % n1, a_idx // (n1 * n1)
    W = np.empty((nq, nq))
    for a in range(nq):
        for q in range(nq):
            qx, qy, qz = q % n1, (q // n1) % n1, q // (n1 * n1)
            W[a, q] = (phi[ax[a], qx] * wg[qx]) * (phi[ay[a], qy] * wg[qy]) * (phi[az[a], qz] * wg[qz])
    f = np.asarray(fq, dtype=np.float64).reshape(3, o.n_el, nq)
    dm = o.dofmap().reshape(o.n_el, nq)
    F = np.zeros(o.n_v)
    for c in range(3):
        Fe = detJ * (f[c] @ W.T)  # [e, a]
        Fc = np.zeros(o.n_nodes)
        np.add.at(Fc, dm.ravel(), Fe.ravel())  # ascending element order (row-major traversal)
        F[c * o.n_nodes:(c + 1) * o.n_nodes] = Fc
    if mask:
        F[o.boundary_mask().astype(bool)] = 0.0
    return F
