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


def fgmres(K, Pinv, b: np.ndarray, m: int, max_iters: int, rtol: float):
    """Flexible GMRES (Saad 1993), restarted every m, modified Gram-Schmidt, Givens rotations,
    x0 = 0; stop when the Givens residual estimate <= rtol ||b|| or after max_iters; restarts
    from the true residual.  The same algorithm as the C oracle's fgmres_run (reading R19),
    with the operator and the (possibly nonlinear) preconditioner as callables.
    Returns (x, iterations, ||b - K x|| / ||b||)."""
    n = len(b)
    x = np.zeros(n)
    w = b.copy()
    bnorm = float(np.sqrt(b @ b))
    beta = bnorm
    total = 0
    while beta > rtol * bnorm and total < max_iters:
        V = np.zeros((m + 1, n))
        Z = np.zeros((m, n))
        H = np.zeros((m + 1, m))
        cs, sn, g = np.zeros(m), np.zeros(m), np.zeros(m + 1)
        V[0] = w / beta
        g[0] = beta
        jend = -1
        for j in range(m):
            if total >= max_iters:
                break
            Z[j] = Pinv(V[j])
            w = K(Z[j])
            for i in range(j + 1):
                hij = float(w @ V[i])
                H[i, j] = hij
                w = w - hij * V[i]
            hn = float(np.sqrt(w @ w))
            for i in range(j):
                a, bb = H[i, j], H[i + 1, j]
                H[i, j] = cs[i] * a + sn[i] * bb
                H[i + 1, j] = -sn[i] * a + cs[i] * bb
            a = H[j, j]
            den = float(np.sqrt(a * a + hn * hn))
            cs[j] = a / den if den > 0 else 1.0
            sn[j] = hn / den if den > 0 else 0.0
            H[j, j] = den
            g[j + 1] = -sn[j] * g[j]
            g[j] = cs[j] * g[j]
            total += 1
            jend = j
            if hn > 0:
                V[j + 1] = w / hn
            if abs(g[j + 1]) <= rtol * bnorm or hn == 0.0:
                break
        y = np.zeros(m)
        for i in range(jend, -1, -1):
            t = g[i] - sum(H[i, k] * y[k] for k in range(i + 1, jend + 1))
            y[i] = t / H[i, i]
        for i in range(jend + 1):
            x = x + y[i] * Z[i]
        w = b - K(x)
        beta = float(np.sqrt(w @ w))
        if jend < 0:
            break
    return x, total, (beta / bnorm if bnorm > 0 else 0.0)


class StokesOracle:
    """[A B^T; B 0] with the eq:precond-stokes right preconditioner (R19), pluggable S~^-1:
    P^-1 (a; b) = (At^-1 (a - B^T y); y), y = -S~^-1 b, At^-1 = the Chebyshev-Jacobi smoother
    on A (R18) with `smooth` steps on [lmin, lmax]."""

    def __init__(self, o: Oracle, mu_q, schur_inv, smooth: int, lmin: float, lmax: float, ainv=None):
        self.o, self.mu = o, np.asarray(mu_q, dtype=np.float64)
        self.schur_inv, self.smooth, self.lmin, self.lmax = schur_inv, smooth, lmin, lmax
        self.ainv = ainv  # At^-1 callable (e.g. velocity V-cycles, R22); default the smoother (R18)

    def K(self, v):
        o = self.o
        u, p = v[:o.n_v], v[o.n_v:]
        return np.concatenate([o.apply_A(self.mu, u) + o.apply_BT(p), o.apply_B(u)])

    def P(self, v):
        o = self.o
        a, b = v[:o.n_v], v[o.n_v:]
        y = -self.schur_inv(b)
        if self.ainv is not None:
            z = self.ainv(np.where(o.boundary_mask().astype(bool), 0.0, a - o.apply_BT(y)))
        else:
            z = o.velocity_cheb(self.mu, a - o.apply_BT(y), self.smooth, self.lmin, self.lmax)
        return np.concatenate([z, y])

    def solve(self, f, g, m, max_iters, rtol):
        o = self.o
        b = np.concatenate([np.where(o.boundary_mask().astype(bool), 0.0, f), g])
        x, it, rr = fgmres(self.K, self.P, b, m, max_iters, rtol)
        return x[:o.n_v], o.project(x[o.n_v:]), it, rr
