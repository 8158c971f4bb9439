"""Oracle of the Schur-complement variants beside wBFBT.

TEST INFRASTRUCTURE ONLY (tests/, bench.py's reference leg).

  * M_p(1/mu): per element M_e[i][j] = sum_q w_q detJ q_i(xi_q) q_j(xi_q) / mu_q
    (orthonormal modes R2, Gauss quadrature R3); applied exactly, z_e = M_e^-1 r_e (reading R21:
    the eq:lumping diagonal M_p 1_{q} vanishes on every non-constant orthonormal mode).
  * diag(A)-BFBT: eq:bfbt with C = D = diag(A):
      z = (B X B^T)^-1 (B X A X B^T) (B X B^T)^-1 r,  X = mask / diag(A) per DOF,
    the Poisson inverses by the O9 Jacobi-PCG (pseudo-inverse diagonal R11, `iters`
    iterations, projected input/output R10), in the O10 order.
"""
from __future__ import annotations

import numpy as np

from . import Oracle


def mp_blocks(o: Oracle, mu_q: np.ndarray) -> np.ndarray:
    t = o.tables()
    leg, wg, modes = t["leg"], t["wg"], t["modes"]
    n1, nq, nm = o.k + 1, o.n_q, o.n_m
    detJ = (0.5 / o.N) ** 3
    Q = np.empty((nm, nq))
    wq = np.empty(nq)
    for q in range(nq):
        qx, qy, qz = q % n1, (q // n1) % n1, q // (n1 * n1)
        wq[q] = wg[qx] * wg[qy] * wg[qz] * detJ
        for m in range(nm):
            Q[m, q] = leg[modes[m][0]][qx] * leg[modes[m][1]][qy] * leg[modes[m][2]][qz]
    mu = np.asarray(mu_q, dtype=np.float64).reshape(o.n_el, nq)
    return np.einsum("iq,jq,eq->eij", Q, Q, wq[None, :] / mu)


def mp_inverse_apply(o: Oracle, mu_q: np.ndarray, r: np.ndarray) -> np.ndarray:
    M = mp_blocks(o, mu_q)
    return np.linalg.solve(M, np.asarray(r, dtype=np.float64).reshape(o.n_el, o.n_m, 1)).reshape(-1)


def _jacobi_dof(o: Oracle, X: np.ndarray) -> np.ndarray:
    Be = o.element_B()
    nq = o.n_q
    dm = o.dofmap().reshape(o.n_el, nq)
    d = np.zeros((o.n_el, o.n_m))
    for c in range(3):
        Xc = X[c * o.n_nodes:(c + 1) * o.n_nodes][dm]  # [e, a]
        d += Xc @ (Be[:, c * nq:(c + 1) * nq] ** 2).T
    return d.reshape(-1)


def _pcg(o: Oracle, K, minv, b, iters):
    r = o.project(b)
    x = np.zeros_like(r)
    z = minv * r
    p = z.copy()
    rz = float(r @ z)
    for _ in range(iters):
        if rz == 0.0:
            break
        q = K(p)
        pq = float(p @ q)
        if pq == 0.0:
            break
        a = rz / pq
        x = x + a * p
        r = r - a * q
        z = minv * r
        rz1 = float(r @ z)
        p = z + (rz1 / rz) * p
        rz = rz1
    return o.project(x)


class DiagABFBT:
    def __init__(self, o: Oracle, mu_q: np.ndarray):
        self.o, self.mu = o, np.asarray(mu_q, dtype=np.float64)
        dA = o.diag_A(self.mu)
        mask = o.boundary_mask().astype(bool)
        self.X = np.where(mask, 0.0, 1.0 / np.where(dA != 0.0, dA, 1.0))
        self.diagK = _jacobi_dof(o, self.X)
        dmax = np.abs(self.diagK).max()
        keep = np.abs(self.diagK) > 1e-13 * dmax
        self.minv = np.where(keep, 1.0 / np.where(keep, self.diagK, 1.0), 0.0)

    def K(self, p):
        return self.o.apply_B(self.o.apply_BT(p) * self.X)

    def poisson(self, b, iters):
        return _pcg(self.o, self.K, self.minv, b, iters)

    def apply(self, r, iters):
        o = self.o
        y = self.poisson(r, iters)
        v = o.apply_BT(y) * self.X
        w = o.apply_A(self.mu, v) * self.X
        s = o.apply_B(w)
        return self.poisson(s, iters)
