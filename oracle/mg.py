"""Oracle of the geometric multigrid V-cycle for the pressure Poisson operators K_w
(second half; PAPER.md:2468-2546 Sec. "Parallel hybrid
spectral-geometric-algebraic multigrid (HMG) for wBFBT").

TEST INFRASTRUCTURE ONLY (imported by tests/ and bench.py's reference leg; the
product package never imports it).  Plain numpy on top of the C oracle's
operators (oracle.Oracle: K apply, Jacobi diagonal, Chebyshev smoother, PCG,
power iteration), each step following DESIGN.md reading R20:

  * levels: N_0 = N, N_{l+1} = N_l / 2 while N_l is even and > 1 (uniform
    element bisection = the paper's geometric coarsening);
  * operators by re-discretisation on every level:
    K_l = B_l X_l B_l^T with the level's own B (Q2 x P1disc on the N_l mesh) and
    X_l = mask / C_l;
  * the coarse weights C_l: the weight DENSITY w(g) = C_{l-1}[g] / M_{l-1}[g]
    (M = the unweighted lumped velocity mass of that level) injected at the
    coincident node, lumped with the coarse mass: C_l[G] = M_l[G] w(iota(G));
  * transfers: P_l = the exact embedding of the coarse P1disc space in the fine
    one (each coarse polynomial restricted to its 8 children), evaluated here by
    L2 projection with Gauss quadrature; restriction = P_l^T (the L2 adjoint
    for dual vectors, "adjoint ... with respect to the L2
    inner products");
  * smoother: nu steps of Chebyshev-accelerated point-Jacobi (PAPER.md:2531-2546:
    three pre- and post-smoothing steps), interval [0.1, 1.1] lambda_l, lambda_l
    the power-iteration estimate of the largest eigenvalue of Minv_l K_l from the
    splitmix64 start vector (the same counter-based generator on both sides);
  * coarsest level: Jacobi-PCG (O9) with min(n_p, 256) iterations (the paper
    uses AMG + a direct solve at 64 elements; reading R20);
  * V(b): x = S(b); x += P V(P^T (b - K x)); x += S(b - K x);
  * MG-PCG: the O9 recurrence with M^-1 := V, fixed iteration count, input and
    output projected off the constant pressure (R10).
"""
from __future__ import annotations

import numpy as np
from numpy.polynomial import legendre as npleg

from . import Oracle

NU = 3            # pre- and post-smoothing steps
EIG_ITERS = 20    # power iterations per level
CHEB_LO, CHEB_HI = 0.1, 1.1
COARSE_CAP = 256  # iterations of the coarsest-level PCG


def splitmix_vector(n: int, seed: int = 0x5EED) -> np.ndarray:
    """v_i = uniform in [-1, 1) from the i-th splitmix64 output of state `seed`: the power-iteration start
    vector, integer arithmetic only, so both sides draw identical doubles."""
    M64 = np.uint64(0xFFFFFFFFFFFFFFFF)
    with np.errstate(over="ignore"):
        # state_i = seed + (i + 1) * golden (the standard splitmix64 stream from state `seed`)
        z = np.uint64(seed) + (np.arange(n, dtype=np.uint64) + np.uint64(1)) * np.uint64(0x9E3779B97F4A7C15) & M64
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    u = (z >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)
    return 2.0 * u - 1.0


def levels_of(N: int) -> list:
    Ns = [N]
    while Ns[-1] % 2 == 0 and Ns[-1] > 1:
        Ns.append(Ns[-1] // 2)
    return Ns


def prolongation_tables(o: Oracle) -> np.ndarray:
    """T[s][mf][mc], s = sx + 2 sy + 4 sz: fine-child coefficient of mode mf from coarse
    mode mc, by L2 projection on the child (orthonormal modes on the reference cube):
    T = int_{[-1,1]^3} q_mc(xi_c(xi)) q_mf(xi) dxi with xi_c = (xi + 2 s - 1) / 2."""
    t = o.tables()
    xg, wg, modes = t["xg"], t["wg"], t["modes"]
    nm = o.n_m

    def lhat(m, x):
        c = np.zeros(m + 1)
        c[m] = 1.0
        return np.sqrt((2 * m + 1) / 2.0) * npleg.legval(x, c)

    T = np.zeros((8, nm, nm))
    for s in range(8):
        sh = np.array([s & 1, (s >> 1) & 1, (s >> 2) & 1]) * 2 - 1
        for mf in range(nm):
            for mc in range(nm):
                acc = 0.0
                for iz in range(len(xg)):
                    for iy in range(len(xg)):
                        for ix in range(len(xg)):
                            xi = np.array([xg[ix], xg[iy], xg[iz]])
                            xc = (xi + sh) / 2.0
                            qc = np.prod([lhat(modes[mc][d], xc[d]) for d in range(3)])
                            qf = np.prod([lhat(modes[mf][d], xi[d]) for d in range(3)])
                            acc += wg[ix] * wg[iy] * wg[iz] * qc * qf
                T[s, mf, mc] = acc
    return T


def child_index(Nc: int):
    """(coarse element, child position s) -> fine element, element-major e = ex + N(ey + N ez)."""
    Nf = 2 * Nc
    ec = np.arange(Nc ** 3)
    cx, cy, cz = ec % Nc, (ec // Nc) % Nc, ec // (Nc * Nc)
    out = np.zeros((Nc ** 3, 8), dtype=np.int64)
    for s in range(8):
        fx, fy, fz = 2 * cx + (s & 1), 2 * cy + ((s >> 1) & 1), 2 * cz + ((s >> 2) & 1)
        out[:, s] = fx + Nf * (fy + Nf * fz)
    return out


def prolong(T, xc: np.ndarray, Nc: int, nm: int) -> np.ndarray:
    """x_f = P x_c (coarse element-major -> fine element-major)."""
    ch = child_index(Nc)
    xf = np.zeros(8 * Nc ** 3 * nm)
    X = xc.reshape(-1, nm)
    for s in range(8):
        xf.reshape(-1, nm)[ch[:, s]] = X @ T[s].T
    return xf


def restrict(T, rf: np.ndarray, Nc: int, nm: int) -> np.ndarray:
    """r_c = P^T r_f; children summed in ascending s."""
    ch = child_index(Nc)
    R = rf.reshape(-1, nm)
    rc = np.zeros((Nc ** 3, nm))
    for s in range(8):
        rc += R[ch[:, s]] @ T[s]
    return rc.reshape(-1)


def inject_weights(Cf: np.ndarray, Mf: np.ndarray, Mc: np.ndarray, Nc: int, k: int = 2) -> np.ndarray:
    """C_c[G] = M_c[G] * C_f[iota(G)] / M_f[iota(G)], iota(G) = the fine node at the coarse
    node's position (coarse GLL grid index i -> fine index 2 i per axis, k = 2)."""
    nc, nf = k * Nc + 1, 2 * k * Nc + 1
    g = np.arange(nc)
    idx = (2 * g[None, None, :] + nf * (2 * g[None, :, None] + nf * 2 * g[:, None, None])).ravel()
    return Mc * (Cf[idx] / Mf[idx])


class MGLevel:
    def __init__(self, N, k, C):
        self.o = Oracle(N, k)
        self.N, self.C = N, C
        mask = self.o.boundary_mask()[: self.o.n_nodes].astype(bool)
        self.X = np.where(mask, 0.0, 1.0 / np.where(C != 0.0, C, 1.0))
        self.diagK = self.o.jacobi_diag(self.X)
        self.n_nonpos = int(np.sum((C <= 0.0) & ~mask))
        self.lam = self.o.poisson_eigmax(self.X, self.diagK, splitmix_vector(self.o.n_p), EIG_ITERS)

    def K(self, p):
        return self.o.apply_K(self.X, p)

    def smooth(self, b):
        return self.o.poisson_cheb(self.X, self.diagK, b, NU, CHEB_LO * self.lam, CHEB_HI * self.lam)


def p_transfer_table(of: Oracle, oc: Oracle) -> np.ndarray:
    """T[mf][mc]: fine-order (P_{kf-1}) coefficient of mode mf from coarse-order (P_{kc-1}) mode
    mc on the SAME element, by L2 projection with the fine order's Gauss rule (the spectral
    level of the paper's HMG): int q_mc^c q_mf^f over the reference cube."""
    tf, tc = of.tables(), oc.tables()
    xg, wg = tf["xg"], tf["wg"]

    def lhat(m, x):
        cc = np.zeros(m + 1)
        cc[m] = 1.0
        return np.sqrt((2 * m + 1) / 2.0) * npleg.legval(x, cc)

    T = np.zeros((of.n_m, oc.n_m))
    for mf in range(of.n_m):
        for mc in range(oc.n_m):
            acc = 0.0
            for iz in range(len(xg)):
                for iy in range(len(xg)):
                    for ix in range(len(xg)):
                        xi = (xg[ix], xg[iy], xg[iz])
                        qc = np.prod([lhat(tc["modes"][mc][d], xi[d]) for d in range(3)])
                        qf = np.prod([lhat(tf["modes"][mf][d], xi[d]) for d in range(3)])
                        acc += wg[ix] * wg[iy] * wg[iz] * qc * qf
            T[mf, mc] = acc
    return T


class MG:
    """The V-cycle hierarchy of one side's K_w, built from that side's lumped mass C_w.
    k = 2: h-levels N, N/2, ... (R20).  k = 4: the paper's HMG order --
    first a spectral level (Q4 x P3disc -> Q2 x P1disc on the same mesh), then the k = 2
    h-levels.  Every level re-discretised, weights by density injection at coincident nodes
    (the Q2 GLL nodes are Q4 GLL nodes: index 2i per axis, as on the bisected mesh)."""

    def __init__(self, N: int, Cw: np.ndarray, k: int = 2):
        assert k in (2, 4), "pressure multigrid for k = 2 (h) and k = 4 (p then h) (R20)"
        self.spec = [(N, k)] + ([(N, 2)] if k == 4 else [])
        while self.spec[-1][0] % 2 == 0 and self.spec[-1][0] > 1:
            self.spec.append((self.spec[-1][0] // 2, 2))
        self.Ns = [n for n, _ in self.spec]
        self.levels = []
        C = np.asarray(Cw, dtype=np.float64)
        M_prev = None
        for li, (Nl, kl) in enumerate(self.spec):
            o = Oracle(Nl, kl)
            M = o.lumped(np.ones(o.n_el * o.n_q))["Cw"]  # unweighted lumped velocity mass
            if li > 0:
                C = inject_weights(C, M_prev, M, Nl, kl)
            self.levels.append(MGLevel(Nl, kl, C))
            M_prev = M
        # transfers per level pair: ("h", T[8][4][4]) on k = 2, ("p", T[nm_f][nm_c]) spectral
        self.trans = []
        for li in range(len(self.spec) - 1):
            (Nf, kf), (Nc, kc) = self.spec[li], self.spec[li + 1]
            if Nf == Nc:
                self.trans.append(("p", p_transfer_table(self.levels[li].o, self.levels[li + 1].o)))
            else:
                self.trans.append(("h", prolongation_tables(self.levels[li + 1].o)))
        self.T = prolongation_tables(Oracle(2, 2))
        self.nm = 4

    def _restrict(self, l, r):
        kind, T = self.trans[l]
        if kind == "p":
            ne = self.levels[l].o.n_el
            return (r.reshape(ne, -1) @ T).reshape(-1)
        return restrict(T, r, self.Ns[l + 1], 4)

    def _prolong(self, l, xc):
        kind, T = self.trans[l]
        if kind == "p":
            ne = self.levels[l].o.n_el
            return (xc.reshape(ne, -1) @ T.T).reshape(-1)
        return prolong(T, xc, self.Ns[l + 1], 4)

    def coarse_iters(self) -> int:
        return min(self.levels[-1].o.n_p, COARSE_CAP)

    def vcycle(self, b: np.ndarray, l: int = 0) -> np.ndarray:
        L = self.levels[l]
        if l == len(self.levels) - 1:
            return L.o.poisson(L.X, L.diagK, b, self.coarse_iters())
        x = L.smooth(b)
        r = b - L.K(x)
        xc = self.vcycle(self._restrict(l, r), l + 1)
        x = x + self._prolong(l, xc)
        r = b - L.K(x)
        return x + L.smooth(r)

    def pcg(self, b: np.ndarray, iters: int) -> np.ndarray:
        """MG-preconditioned CG (O9 recurrence, M^-1 = V), exactly `iters` iterations."""
        L0 = self.levels[0]
        o = L0.o
        r = o.project(b)
        x = np.zeros_like(r)
        z = self.vcycle(r)
        p = z.copy()
        rz = float(r @ z)
        for _ in range(iters):
            if rz == 0.0:
                break
            q = L0.K(p)
            pq = float(p @ q)
            if pq == 0.0:
                break
            a = rz / pq
            x = x + a * p
            r = r - a * q
            z = self.vcycle(r)
            rz1 = float(r @ z)
            p = z + (rz1 / rz) * p
            rz = rz1
        return o.project(x)


def wbfbt_mg(o: Oracle, mu_q, state: dict, mg_l: MG, mg_r: MG, r: np.ndarray, iters: int) -> np.ndarray:
    """eq:wbfbt in the O10 order with both Poisson inverses replaced by
    MG-PCG (`iters` iterations): y = P MGPCG(K_r, P r); v = Dinv o B^T y; v = A v;
    v = Cinv o v; s = P B v; z = P MGPCG(K_l, s)."""
    y = mg_r.pcg(r, iters)
    v = o.apply_BT(y) * np.tile(state["Dinv"], 3)
    v = o.apply_A(mu_q, v)
    v = v * np.tile(state["Cinv"], 3)
    s = o.project(o.apply_B(v))
    return mg_l.pcg(s, iters)


# ---------------------------------------------------------------- velocity multigrid (R22)
def coarsen_mu(mu_f: np.ndarray, Nc: int, wg: np.ndarray) -> np.ndarray:
    """mu at the coarse Gauss points: the mean, over the fine children whose closure contains
    the point, of each child's Gauss-weighted mean sum_q w_q mu_q / sum_q w_q (k = 2; the
    coarse abscissae -sqrt(3/5), 0, +sqrt(3/5) lie in child 0, on the face, in child 1)."""
    Nf = 2 * Nc
    w3 = np.array([wg[q % 3] * wg[(q // 3) % 3] * wg[q // 9] for q in range(27)])
    m = (np.asarray(mu_f).reshape(Nf ** 3, 27) @ w3 / 8.0).reshape(Nc, 2, Nc, 2, Nc, 2)  # [cz][sz][cy][sy][cx][sx]
    sets = [[0], [0, 1], [1]]
    out = np.zeros((Nc, Nc, Nc, 27))
    for q in range(27):
        qx, qy, qz = q % 3, (q // 3) % 3, q // 9
        vals = [m[:, sz, :, sy, :, sx] for sz in sets[qz] for sy in sets[qy] for sx in sets[qx]]
        acc = vals[0].copy()
        for v in vals[1:]:
            acc = acc + v
        out[..., q] = acc / len(vals)
    return out.reshape(-1)


def q2_prolongation_1d(Nc: int, xn: np.ndarray) -> np.ndarray:
    """P[i_f, I]: coarse Q2 nodal basis (GLL nodes xn of the oracle) evaluated at the fine
    nodes; fine element nodes sit at coarse-element coordinates -1, -1/2, 0, 1/2, 1."""
    nc, nf = 2 * Nc + 1, 4 * Nc + 1
    P = np.zeros((nf, nc))
    for e in range(Nc):
        for j, t in enumerate((-1.0, -0.5, 0.0, 0.5, 1.0)):
            for a in range(3):
                v = 1.0
                for b in range(3):
                    if b != a:
                        v *= (t - xn[b]) / (xn[a] - xn[b])
                P[4 * e + j, 2 * e + a] = v
    return P


def _tp3(P: np.ndarray, X: np.ndarray) -> np.ndarray:
    """(P x P x P) X for a [z][y][x] array X: the 1-D map P applied along each axis."""
    X = np.tensordot(P, X, axes=(1, 0))                     # z
    X = np.tensordot(P, X, axes=(1, 1)).transpose(1, 0, 2)  # y
    return np.tensordot(X, P, axes=(2, 1))                  # x


def vprolong(P1: np.ndarray, xc: np.ndarray) -> np.ndarray:
    nf, nc = P1.shape
    return np.concatenate([_tp3(P1, xc[c * nc ** 3:(c + 1) * nc ** 3].reshape(nc, nc, nc)).ravel() for c in range(3)])


def vrestrict(P1: np.ndarray, xf: np.ndarray) -> np.ndarray:
    nf, nc = P1.shape
    return np.concatenate([_tp3(P1.T, xf[c * nf ** 3:(c + 1) * nf ** 3].reshape(nf, nf, nf)).ravel() for c in range(3)])


def coarsen_mu_p(mu_f: np.ndarray, n_el: int, wg4: np.ndarray) -> np.ndarray:
    """The spectral velocity level (k = 4 -> 2 on the same element): mu at the 3 Gauss points
    per axis as the Gauss-weighted mean of the 5-point samples grouped by position (per axis
    {0, 1} -> the point at -sqrt(3/5), {2} -> 0, {3, 4} -> +sqrt(3/5)), tensor product."""
    groups = [[0, 1], [2], [3, 4]]
    m = np.asarray(mu_f).reshape(n_el, 5, 5, 5)  # [e][qz][qy][qx]
    out = np.zeros((n_el, 3, 3, 3))
    for cz in range(3):
        for cy in range(3):
            for cx in range(3):
                num, den = 0.0, 0.0
                for iz in groups[cz]:
                    for iy in groups[cy]:
                        for ix in groups[cx]:
                            w = wg4[ix] * wg4[iy] * wg4[iz]
                            num = num + w * m[:, iz, iy, ix]
                            den += w
                out[:, cz, cy, cx] = num / den
    return out.reshape(-1)


def p_prolongation_1d(N: int, xn2: np.ndarray, xn4: np.ndarray) -> np.ndarray:
    """P[i_f, I]: the Q2 nodal basis of each element evaluated at its Q4 GLL nodes (same mesh)."""
    nf, nc = 4 * N + 1, 2 * N + 1
    P = np.zeros((nf, nc))
    for e in range(N):
        for j in range(5):
            t = xn4[j]
            for a in range(3):
                v = 1.0
                for b in range(3):
                    if b != a:
                        v *= (t - xn2[b]) / (xn2[a] - xn2[b])
                P[4 * e + j, 2 * e + a] = v
    return P


class VMG:
    """V-cycle hierarchy of the masked viscous block M A M (R22): levels as the pressure
    multigrid (k = 4: first the spectral level to Q2 on the same mesh), A_l re-discretised with
    the coarsened mu, Q2 (or Q2-in-Q4) nodal transfers, nu Chebyshev-Jacobi steps (R18) on
    [0.1, 1.1] x a 20-step power estimate (splitmix64 start), 30 on the coarsest level."""

    def __init__(self, N: int, mu_q: np.ndarray, nu: int = NU, k: int = 2):
        assert k in (2, 4)
        self.nu = nu
        self.spec = [(N, k)] + ([(N, 2)] if k == 4 else [])
        while self.spec[-1][0] % 2 == 0 and self.spec[-1][0] > 1:
            self.spec.append((self.spec[-1][0] // 2, 2))
        self.Ns = [n for n, _ in self.spec]
        self.lev = []
        mu = np.asarray(mu_q, dtype=np.float64)
        for li, (Nl, kl) in enumerate(self.spec):
            o = Oracle(Nl, kl)
            if li > 0:
                if Nl == self.spec[li - 1][0]:
                    mu = coarsen_mu_p(mu, o.n_el, self.lev[-1]["o"].tables()["wg"])
                else:
                    mu = coarsen_mu(mu, Nl, o.tables()["wg"])
            lam = o.velocity_eigmax(mu, splitmix_vector(o.n_v), EIG_ITERS)
            self.lev.append(dict(N=Nl, o=o, mu=mu, lam=lam, mask=o.boundary_mask().astype(bool)))
        xn2 = Oracle(1, 2).tables()["xn"]
        self.P = []
        for l in range(len(self.spec) - 1):
            if self.spec[l][0] == self.spec[l + 1][0]:
                self.P.append(p_prolongation_1d(self.Ns[l], xn2, self.lev[l]["o"].tables()["xn"]))
            else:
                self.P.append(q2_prolongation_1d(self.Ns[l + 1], xn2))

    def A(self, l, v):
        L = self.lev[l]
        return L["o"].apply_A(L["mu"], v)

    def smooth(self, l, b, its):
        L = self.lev[l]
        return L["o"].velocity_cheb(L["mu"], b, its, CHEB_LO * L["lam"], CHEB_HI * L["lam"])

    def vcycle(self, b, l=0):
        if l == len(self.lev) - 1:
            return self.smooth(l, b, 30)
        L = self.lev[l]
        x = self.smooth(l, b, self.nu)
        r = b - self.A(l, x)
        rc = vrestrict(self.P[l], np.where(L["mask"], 0.0, r))  # Dirichlet rows carry no residual (R6)
        rc[self.lev[l + 1]["mask"]] = 0.0
        xc = self.vcycle(rc, l + 1)
        x = x + np.where(L["mask"], 0.0, vprolong(self.P[l], xc))
        r = b - self.A(l, x)
        return x + self.smooth(l, r, self.nu)

    def cycles(self, b, k):
        x = self.vcycle(b)
        for _ in range(1, k):
            x = x + self.vcycle(b - self.A(0, x))
        return x
