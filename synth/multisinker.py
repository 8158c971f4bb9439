"""Multi-sinker benchmark inputs (Sec. 2.1 "multi-sinker test
problem") for the five BASELINE.json configs.

Recipe:
  * rng = numpy Generator(PCG64(seed)), seed 0 by default.
  * Draw order: sinker centres rng.random((n, 3)) ~ U[0,1)^3, then the velocity
    vector u = rng.uniform(-1, 1, n_v), then the pressure vector
    p = rng.uniform(-1, 1, n_p).  (Prefix property: the first m centres of an
    n-sinker draw equal an m-sinker draw.)
  * mu(x) = (mu_max - mu_min)(1 - chi_n(x)) + mu_min,
    chi_n(x) = prod_i [1 - exp(-delta * max(0, |c_i - x| - omega/2)^2)]
    (PAPER.md:621-633), evaluated in fp64 at the tensor Gauss-Legendre points
    of every element: x_q = h * (e_idx + (xi_q + 1)/2) per axis, h = 1/N.
    The 1-D Gauss points come from numpy.polynomial.legendre.leggauss (a
    library routine; neither the oracle nor the CUDA path uses it).
  * Layout: mu_q[e * n_q + q], e = ex + N*(ey + N*ez), q = qx + n1*(qy + n1*qz)
    (x fastest), n1 = k+1, n_q = n1^3.
  * Velocity vectors are SoA: u[c * n_nodes + g].  Boundary entries are drawn
    too; the library ignores them (Dirichlet elimination).
"""
from __future__ import annotations

from dataclasses import dataclass
from math import comb

import numpy as np


@dataclass(frozen=True)
class Config:
    name: str
    N: int          # elements per axis
    k: int          # velocity order (Q_k x P_{k-1}^disc)
    n_sinkers: int
    delta: float
    omega: float
    mu_min: float
    mu_max: float
    iters: int      # Jacobi-PCG iterations per Poisson inverse

    @property
    def dr(self) -> float:
        return self.mu_max / self.mu_min


# BASELINE.json "configs", in order.  C4 names only "ratio 1e6": mu_min = DR^-1/2,
# mu_max = DR^1/2; C4 names no PCG count, 50 is our reading.
CONFIGS = {
    "C1": Config("C1", 4, 2, 4, 200.0, 0.1, 1e-2, 1e2, 20),
    "C2": Config("C2", 16, 2, 8, 200.0, 0.1, 1e-3, 1e3, 50),
    "C3": Config("C3", 32, 2, 16, 200.0, 0.1, 1e-4, 1e4, 50),
    "C4": Config("C4", 24, 4, 8, 200.0, 0.1, 1e-3, 1e3, 50),
    "C5": Config("C5", 64, 2, 24, 200.0, 0.05, 1e-5, 1e5, 100),
}


def sizes(N: int, k: int) -> dict:
    """Structured counts: n_v counts boundary dofs, as PAPER.md
    Table 3 does."""
    n1 = k + 1
    n_nodes = (k * N + 1) ** 3
    n_m = comb(k + 2, 3)
    return dict(n_el=N ** 3, n_nodes=n_nodes, n_v=3 * n_nodes, n_m=n_m,
                n_p=n_m * N ** 3, n_q=n1 ** 3, n1=n1)


def gauss_points_1d(k: int) -> np.ndarray:
    """(k+1) Gauss-Legendre points on [-1, 1], ascending (numpy library routine)."""
    x, _ = np.polynomial.legendre.leggauss(k + 1)
    return np.sort(x)


def sinker_centers(rng: np.random.Generator, n: int) -> np.ndarray:
    return rng.random((n, 3))


def chi(x: np.ndarray, centers: np.ndarray, delta: float, omega: float) -> np.ndarray:
    """Indicator chi_n at points x (..., 3) -- PAPER.md:626-633."""
    x = np.asarray(x, dtype=np.float64)
    out = np.ones(x.shape[:-1], dtype=np.float64)
    for c in np.asarray(centers, dtype=np.float64):
        d = np.sqrt(((x - c) ** 2).sum(axis=-1))
        s = np.maximum(0.0, d - omega / 2.0)
        out *= 1.0 - np.exp(-delta * s * s)
    return out


def viscosity(x: np.ndarray, centers: np.ndarray, delta: float, omega: float,
              mu_min: float, mu_max: float) -> np.ndarray:
    """mu(x) = (mu_max - mu_min)(1 - chi_n(x)) + mu_min -- PAPER.md:622-623."""
    return (mu_max - mu_min) * (1.0 - chi(x, centers, delta, omega)) + mu_min


def viscosity_at_quadrature(N: int, k: int, centers: np.ndarray, delta: float, omega: float,
                            mu_min: float, mu_max: float, chunk: int = 4096) -> np.ndarray:
    """mu sampled at every element's tensor Gauss points, element-major, q x-fastest."""
    n1 = k + 1
    h = 1.0 / N
    xi = gauss_points_1d(k)
    # q-local offsets (x fastest)
    qz, qy, qx = np.meshgrid(np.arange(n1), np.arange(n1), np.arange(n1), indexing="ij")
    loc = np.stack([(xi[qx.ravel()] + 1) / 2, (xi[qy.ravel()] + 1) / 2, (xi[qz.ravel()] + 1) / 2], -1)
    n_el = N ** 3
    out = np.empty((n_el, n1 ** 3), dtype=np.float64)
    for e0 in range(0, n_el, chunk):
        e = np.arange(e0, min(e0 + chunk, n_el))
        ex, ey, ez = e % N, (e // N) % N, e // (N * N)
        base = np.stack([ex, ey, ez], -1).astype(np.float64)
        x = h * (base[:, None, :] + loc[None, :, :])
        out[e0:e0 + len(e)] = viscosity(x, centers, delta, omega, mu_min, mu_max)
    return out.reshape(-1)


def forcing_at_quadrature(N: int, k: int, centers: np.ndarray, delta: float, omega: float,
                          beta: float = 10.0, chunk: int = 4096) -> np.ndarray:
    """Body force f(x) = (0, 0, beta (chi_n(x) - 1)), beta = 10 (the
    right-hand side of eq:discrete-stokes), sampled at every element's Gauss points:
    component-major [c][e][q] (the layout of mu_q per component)."""
    n1 = k + 1
    h = 1.0 / N
    xi = gauss_points_1d(k)
    qz, qy, qx = np.meshgrid(np.arange(n1), np.arange(n1), np.arange(n1), indexing="ij")
    loc = np.stack([(xi[qx.ravel()] + 1) / 2, (xi[qy.ravel()] + 1) / 2, (xi[qz.ravel()] + 1) / 2], -1)
    n_el = N ** 3
    out = np.zeros((3, n_el, n1 ** 3), dtype=np.float64)
    for e0 in range(0, n_el, chunk):
        e = np.arange(e0, min(e0 + chunk, n_el))
        ex, ey, ez = e % N, (e // N) % N, e // (N * N)
        base = np.stack([ex, ey, ez], -1).astype(np.float64)
        x = h * (base[:, None, :] + loc[None, :, :])
        out[2, e0:e0 + len(e)] = beta * (chi(x, centers, delta, omega) - 1.0)
    return out.reshape(-1)


def make_inputs(cfg: Config | str, seed: int = 0, *, N: int | None = None) -> dict:
    """All seeded inputs of one config: centres, mu_q, u, p (numpy fp64).

    `N` overrides the mesh size (small-size parity cases of the same recipe)."""
    if isinstance(cfg, str):
        cfg = CONFIGS[cfg]
    N = cfg.N if N is None else N
    s = sizes(N, cfg.k)
    rng = np.random.Generator(np.random.PCG64(seed))
    centers = sinker_centers(rng, cfg.n_sinkers)
    u = rng.uniform(-1.0, 1.0, s["n_v"])
    p = rng.uniform(-1.0, 1.0, s["n_p"])
    mu_q = viscosity_at_quadrature(N, cfg.k, centers, cfg.delta, cfg.omega, cfg.mu_min, cfg.mu_max)
    return dict(N=N, k=cfg.k, centers=centers, mu_q=mu_q, u=u, p=p, sizes=s, cfg=cfg)
