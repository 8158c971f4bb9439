"""ctypes wrapper of the CPU oracle (oracle/oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs.  The product package
(paper_1607_03936_b200) never imports this module.

The oracle is built from source on first use (gcc, -O2 -fno-fast-math
-ffp-contract=off -fopenmp) into oracle/liboracle.so.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

_D = C.POINTER(C.c_double)
_I64 = C.POINTER(C.c_int64)


def build(force: bool = False) -> str:
    """Compile oracle.c -> liboracle.so (in-tree)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-fno-fast-math", "-ffp-contract=off", "-fopenmp", "-shared", "-fPIC",
               "-o", _LIB + ".tmp", _SRC, "-lm"]
        subprocess.check_call(cmd)
        os.replace(_LIB + ".tmp", _LIB)
    return _LIB


def lib():
    global _lib
    with _lock:
        if _lib is None:
            build()
            L = C.CDLL(_LIB)
            L.or_create.restype = C.c_void_p
            L.or_create.argtypes = [C.c_int, C.c_int]
            L.or_create_box.restype = C.c_void_p
            L.or_create_box.argtypes = [C.c_int, C.c_int, C.c_int]
            L.or_destroy.argtypes = [C.c_void_p]
            L.or_sizes.argtypes = [C.c_void_p, _I64]
            L.or_tables.argtypes = [C.c_void_p, _D, _D, _D, _D, _D, _D, C.POINTER(C.c_int)]
            L.or_element_B.argtypes = [C.c_void_p, _D]
            L.or_element_A_matrix.argtypes = [C.c_void_p, _D, _D]
            L.or_dofmap.argtypes = [C.c_void_p, _I64]
            L.or_sizes_only.argtypes = [C.c_int, C.c_int, _I64]
            L.or_boundary_elements.argtypes = [C.c_void_p, C.POINTER(C.c_uint8)]
            L.or_boundary_mask.argtypes = [C.c_void_p, C.POINTER(C.c_uint8)]
            L.or_apply_A.argtypes = [C.c_void_p, _D, _D, _D, C.c_int]
            L.or_apply_A_sampled.argtypes = [C.c_void_p, _D, _D, _I64, C.c_int64, _D]
            L.or_apply_B.argtypes = [C.c_void_p, _D, _D, C.c_int]
            L.or_apply_BT.argtypes = [C.c_void_p, _D, _D, C.c_int]
            L.or_lumped.argtypes = [C.c_void_p, _D, C.c_double, C.c_double, _D, _D, _D, _D, _I64]
            L.or_apply_K.argtypes = [C.c_void_p, _D, _D, _D, _D]
            L.or_jacobi_diag.argtypes = [C.c_void_p, _D, _D]
            L.or_project.argtypes = [C.c_void_p, _D]
            L.or_pcg.argtypes = [C.c_void_p, _D, _D, _D, _D, C.c_int]
            L.or_pcg_rec.argtypes = [C.c_void_p, _D, _D, _D, _D, C.c_int, _D, _D]
            L.or_pcg_rec.restype = C.c_int
            L.or_pcg_step.argtypes = [C.c_void_p, _D, _D, _D, _D, _D, _D]
            L.or_poisson.argtypes = [C.c_void_p, _D, _D, _D, _D, C.c_int]
            L.or_wbfbt.argtypes = [C.c_void_p, _D, _D, _D, _D, _D, _D, _D, C.c_int]
            L.or_poisson_relres.restype = C.c_double
            L.or_poisson_relres.argtypes = [C.c_void_p, _D, _D, _D]
            L.or_grad_weights.argtypes = [C.c_void_p, _D, _D]
            L.or_diag_A.argtypes = [C.c_void_p, _D, _D]
            L.or_wbfbt_cheb.argtypes = [C.c_void_p, _D, _D, _D, _D, _D, _D, _D, C.c_int, C.c_double, C.c_double,
                                        C.c_double, C.c_double]
            L.or_fgmres_dense.argtypes = [C.c_int64, _D, _D, _D, _D, C.c_int, C.c_int, C.c_double, _D]
            L.or_fgmres_dense.restype = C.c_int
            L.or_stokes_fgmres.argtypes = [C.c_void_p, _D, _D, _D, _D, _D, _D, _D, _D, _D, C.c_int, C.c_int,
                                           C.c_double, C.c_int, C.c_int, C.c_double, C.c_double, _D, _D]
            L.or_stokes_fgmres.restype = C.c_int
            L.or_velocity_cheb.argtypes = [C.c_void_p, _D, _D, _D, C.c_int, C.c_double, C.c_double]
            L.or_velocity_eigmax.argtypes = [C.c_void_p, _D, _D, C.c_int]
            L.or_velocity_eigmax.restype = C.c_double
            L.or_cheb_dense.argtypes = [C.c_int64, _D, _D, _D, _D, C.c_int, C.c_double, C.c_double]
            L.or_poisson_cheb.argtypes = [C.c_void_p, _D, _D, _D, _D, C.c_int, C.c_double, C.c_double]
            L.or_eigmax_dense.argtypes = [C.c_int64, _D, _D, _D, C.c_int]
            L.or_eigmax_dense.restype = C.c_double
            L.or_poisson_eigmax.argtypes = [C.c_void_p, _D, _D, _D, C.c_int]
            L.or_poisson_eigmax.restype = C.c_double
            L.or_num_threads.restype = C.c_int
            L.or_set_order.argtypes = [C.c_int]
            _lib = L
    return _lib


def _p(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(_D)


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def cheb_dense(A, Minv, b, iters, lmin, lmax) -> np.ndarray:
    """The Chebyshev recurrence of or_poisson_cheb on a dense matrix A (row-major), x0 = 0."""
    A, Minv, b = _f64(A), _f64(Minv), _f64(b)
    x = np.zeros(len(b))
    lib().or_cheb_dense(len(b), _p(A), _p(Minv), _p(b), _p(x), int(iters), float(lmin), float(lmax))
    return x


def eigmax_dense(A, Minv, v0, iters) -> float:
    """The power iteration of or_poisson_eigmax on a dense matrix A (row-major)."""
    A, Minv, v0 = _f64(A), _f64(Minv), _f64(v0)
    return float(lib().or_eigmax_dense(len(v0), _p(A), _p(Minv), _p(v0), int(iters)))


def fgmres_dense(A, P, b, restart, max_iters, rtol):
    """(x, iterations, relres) of the oracle's FGMRES core on a dense system, right preconditioner P."""
    A, P, b = _f64(A), _f64(P), _f64(b)
    x, rr = np.zeros(len(b)), np.zeros(1)
    it = lib().or_fgmres_dense(len(b), _p(A), _p(P), _p(b), _p(x), int(restart), int(max_iters), float(rtol),
                               _p(rr))
    return x, int(it), float(rr[0])


def sizes_only(N: int, k: int) -> dict:
    """Oracle's structured counts without building tables."""
    s = np.zeros(6, dtype=np.int64)
    lib().or_sizes_only(N, k, s.ctypes.data_as(_I64))
    return dict(zip(("n_el", "n_nodes", "n_v", "n_p", "n_q", "n_m"), (int(v) for v in s)))


class Oracle:
    """One structured mesh (N^3 elements, Q_k x P_{k-1}^disc) on the unit cube; with Nz given,
    the box of N x N x Nz elements of side 1/N (z-stacked cubes: the global mesh of the slab
    decomposition; reading R24)."""

    def __init__(self, N: int, k: int, Nz: int | None = None):
        self.L = lib()
        self.h = self.L.or_create(N, k) if Nz is None else self.L.or_create_box(N, Nz, k)
        if not self.h:
            raise ValueError(f"oracle: bad N={N} k={k} Nz={Nz}")
        self.N, self.k, self.Nz = N, k, (N if Nz is None else Nz)
        s = np.zeros(6, dtype=np.int64)
        self.L.or_sizes(self.h, s.ctypes.data_as(_I64))
        self.n_el, self.n_nodes, self.n_v, self.n_p, self.n_q, self.n_m = (int(v) for v in s)
        self.mu_q = None

    def __del__(self):
        try:
            if self.h:
                self.L.or_destroy(self.h)
                self.h = None
        except Exception:
            pass

    # ---- tables / structure
    def tables(self) -> dict:
        n1 = self.k + 1
        xn, xg, wg = np.zeros(n1), np.zeros(n1), np.zeros(n1)
        phi, dphi, leg = np.zeros((n1, n1)), np.zeros((n1, n1)), np.zeros((n1, n1))
        modes = np.zeros((self.n_m, 3), dtype=np.int32)
        self.L.or_tables(self.h, _p(xn), _p(xg), _p(wg), _p(phi), _p(dphi), _p(leg),
                         modes.ctypes.data_as(C.POINTER(C.c_int)))
        return dict(xn=xn, xg=xg, wg=wg, phi=phi, dphi=dphi, leg=leg, modes=modes)

    def element_B(self) -> np.ndarray:
        B = np.zeros((self.n_m, 3 * self.n_q))
        self.L.or_element_B(self.h, _p(B))
        return B

    def element_A_matrix(self, mue) -> np.ndarray:
        mue = _f64(mue)
        A = np.zeros((3 * self.n_q, 3 * self.n_q))
        self.L.or_element_A_matrix(self.h, _p(mue), _p(A))
        return A

    def dofmap(self) -> np.ndarray:
        m = np.zeros(self.n_el * self.n_q, dtype=np.int64)
        self.L.or_dofmap(self.h, m.ctypes.data_as(_I64))
        return m

    def boundary_elements(self) -> np.ndarray:
        f = np.zeros(self.n_el, dtype=np.uint8)
        self.L.or_boundary_elements(self.h, f.ctypes.data_as(C.POINTER(C.c_uint8)))
        return f

    def boundary_mask(self) -> np.ndarray:
        m = np.zeros(self.n_v, dtype=np.uint8)
        self.L.or_boundary_mask(self.h, m.ctypes.data_as(C.POINTER(C.c_uint8)))
        return m

    # ---- operators
    def apply_A(self, mu_q, u, nomask=False) -> np.ndarray:
        mu_q, u = _f64(mu_q), _f64(u)
        y = np.zeros(self.n_v)
        self.L.or_apply_A(self.h, _p(mu_q), _p(u), _p(y), int(nomask))
        return y

    def apply_A_sampled(self, mu_q, u, dofs) -> np.ndarray:
        mu_q, u = _f64(mu_q), _f64(u)
        dofs = np.ascontiguousarray(dofs, dtype=np.int64)
        y = np.zeros(len(dofs))
        self.L.or_apply_A_sampled(self.h, _p(mu_q), _p(u), dofs.ctypes.data_as(_I64), len(dofs), _p(y))
        return y

    def apply_B(self, u, nomask=False) -> np.ndarray:
        u = _f64(u)
        p = np.zeros(self.n_p)
        self.L.or_apply_B(self.h, _p(u), _p(p), int(nomask))
        return p

    def apply_BT(self, p, nomask=False) -> np.ndarray:
        p = _f64(p)
        y = np.zeros(self.n_v)
        self.L.or_apply_BT(self.h, _p(p), _p(y), int(nomask))
        return y

    def lumped(self, mu_q, a_l=1.0, a_r=1.0) -> dict:
        mu_q = _f64(mu_q)
        Cw, Dw, Ci, Di = (np.zeros(self.n_nodes) for _ in range(4))
        npos = np.zeros(2, dtype=np.int64)
        self.L.or_lumped(self.h, _p(mu_q), float(a_l), float(a_r), _p(Cw), _p(Dw), _p(Ci), _p(Di),
                         npos.ctypes.data_as(_I64))
        return dict(Cw=Cw, Dw=Dw, Cinv=Ci, Dinv=Di, n_nonpos_Cw=int(npos[0]), n_nonpos_Dw=int(npos[1]))

    def apply_K(self, Xinv, p) -> np.ndarray:
        Xinv, p = _f64(Xinv), _f64(p)
        q = np.zeros(self.n_p)
        tv = np.zeros(self.n_v)
        self.L.or_apply_K(self.h, _p(Xinv), _p(p), _p(q), _p(tv))
        return q

    def jacobi_diag(self, Xinv) -> np.ndarray:
        Xinv = _f64(Xinv)
        d = np.zeros(self.n_p)
        self.L.or_jacobi_diag(self.h, _p(Xinv), _p(d))
        return d

    def project(self, v) -> np.ndarray:
        v = _f64(v).copy()
        self.L.or_project(self.h, _p(v))
        return v

    def pcg(self, Xinv, diagK, b, iters) -> np.ndarray:
        Xinv, diagK, b = _f64(Xinv), _f64(diagK), _f64(b)
        x = np.zeros(self.n_p)
        self.L.or_pcg(self.h, _p(Xinv), _p(diagK), _p(b), _p(x), int(iters))
        return x

    def pcg_scalars(self, Xinv, diagK, b, iters):
        """PCG (O9) recording its scalars: (x, alpha[iters], beta[iters], iterations run);
        alpha_i = rz_i / pq_i, beta_i = rz_{i+1} / rz_i (0 for iterations not run)."""
        Xinv, diagK, b = _f64(Xinv), _f64(diagK), _f64(b)
        x, a, bt = np.zeros(self.n_p), np.zeros(int(iters)), np.zeros(int(iters))
        run = self.L.or_pcg_rec(self.h, _p(Xinv), _p(diagK), _p(b), _p(x), int(iters), _p(a), _p(bt))
        return x, a, bt, int(run)

    def pcg_step(self, Xinv, diagK, x, r, p, rz):
        """One PCG iteration from state (x, r, p, rz); returns new (x, r, p, rz)."""
        Xinv, diagK = _f64(Xinv), _f64(diagK)
        x, r, p = _f64(x).copy(), _f64(r).copy(), _f64(p).copy()
        rzv = C.c_double(rz)
        self.L.or_pcg_step(self.h, _p(Xinv), _p(diagK), _p(x), _p(r), _p(p), C.byref(rzv))
        return x, r, p, rzv.value

    def poisson(self, Xinv, diagK, b, iters) -> np.ndarray:
        Xinv, diagK, b = _f64(Xinv), _f64(diagK), _f64(b)
        x = np.zeros(self.n_p)
        self.L.or_poisson(self.h, _p(Xinv), _p(diagK), _p(b), _p(x), int(iters))
        return x

    def poisson_cheb(self, Xinv, diagK, b, iters, lmin, lmax) -> np.ndarray:
        """x = P Cheb(K, P b): Chebyshev-accelerated Jacobi, interval [lmin, lmax] of Minv K (R16)."""
        Xinv, diagK, b = _f64(Xinv), _f64(diagK), _f64(b)
        x = np.zeros(self.n_p)
        self.L.or_poisson_cheb(self.h, _p(Xinv), _p(diagK), _p(b), _p(x), int(iters), float(lmin), float(lmax))
        return x

    def poisson_eigmax(self, Xinv, diagK, v0, iters) -> float:
        """Power-iteration estimate of the largest |eigenvalue| of Minv K from start vector v0."""
        Xinv, diagK, v0 = _f64(Xinv), _f64(diagK), _f64(v0)
        return float(self.L.or_poisson_eigmax(self.h, _p(Xinv), _p(diagK), _p(v0), int(iters)))

    def diag_A(self, mu_q) -> np.ndarray:
        """diag(M A M), n_v, Dirichlet dofs 0 (R18)."""
        mu_q = _f64(mu_q)
        d = np.zeros(self.n_v)
        self.L.or_diag_A(self.h, _p(mu_q), _p(d))
        return d

    def velocity_cheb(self, mu_q, b, iters, lmin, lmax) -> np.ndarray:
        """x = Cheb(M A M, M b) with the Jacobi inverse mask/diag(A), x0 = 0 (R16, R18)."""
        mu_q, b = _f64(mu_q), _f64(b)
        x = np.zeros(self.n_v)
        self.L.or_velocity_cheb(self.h, _p(mu_q), _p(b), _p(x), int(iters), float(lmin), float(lmax))
        return x

    def velocity_eigmax(self, mu_q, v0, iters) -> float:
        mu_q, v0 = _f64(mu_q), _f64(v0)
        return float(self.L.or_velocity_eigmax(self.h, _p(mu_q), _p(v0), int(iters)))

    def stokes_fgmres(self, f, g, restart, max_iters, rtol, pcg_iters, smooth_iters, lmin, lmax, state=None,
                      inner=None):
        """(u, p, iterations, relres): FGMRES on [A B^T; B 0] with eq:precond-stokes (R19).
        inner = (lmin_l, lmax_l, lmin_r, lmax_r): wBFBT with Chebyshev inner solves."""
        st = self.state if state is None else state
        f, g = _f64(f), _f64(g)
        u, p, rr = np.zeros(self.n_v), np.zeros(self.n_p), np.zeros(1)
        inn = _f64(inner) if inner is not None else None
        it = self.L.or_stokes_fgmres(self.h, _p(self.mu_q), _p(st["Cinv"]), _p(st["Dinv"]), _p(st["diagKl"]),
                                     _p(st["diagKr"]), _p(f), _p(g), _p(u), _p(p), int(restart), int(max_iters),
                                     float(rtol), int(pcg_iters), int(smooth_iters), float(lmin), float(lmax), _p(rr),
                                     _p(inn) if inn is not None else None)
        return u, p, int(it), float(rr[0])

    def poisson_relres(self, Xinv, b, x) -> float:
        Xinv, b, x = _f64(Xinv), _f64(b), _f64(x)
        return float(self.L.or_poisson_relres(self.h, _p(Xinv), _p(b), _p(x)))

    def grad_weights(self, mu_q) -> np.ndarray:
        """mu_eff = sqrt(mu^2 + |grad mu|^2) at the Gauss points (rmk:wbfbt-visc-grad, R17):
        lumping mu_eff (weight sqrt(mu_eff)) gives the viscosity-gradient wBFBT weights."""
        mu_q = _f64(mu_q)
        out = np.zeros_like(mu_q)
        self.L.or_grad_weights(self.h, _p(mu_q), _p(out))
        return out

    # ---- composite
    def setup(self, mu_q, a_l=1.0, a_r=1.0, weights="sqrt") -> dict:
        """Lumped diagonals and both Jacobi diagonals (rows a3, a4).  weights: "sqrt"
        (w = sqrt(mu), eq:wbfbt) or "grad" (w = (mu^2 + |grad mu|^2)^(1/4), rmk:wbfbt-visc-grad);
        A always uses mu itself."""
        self.mu_q = _f64(mu_q)
        assert weights in ("sqrt", "grad")
        lm = self.lumped(self.mu_q if weights == "sqrt" else self.grad_weights(self.mu_q), a_l, a_r)
        lm["diagKl"] = self.jacobi_diag(lm["Cinv"])
        lm["diagKr"] = self.jacobi_diag(lm["Dinv"])
        self.state = lm
        return lm

    def wbfbt(self, r, iters, state=None) -> np.ndarray:
        s = self.state if state is None else state
        r = _f64(r)
        z = np.zeros(self.n_p)
        self.L.or_wbfbt(self.h, _p(self.mu_q), _p(s["Cinv"]), _p(s["Dinv"]), _p(s["diagKl"]),
                        _p(s["diagKr"]), _p(r), _p(z), int(iters))
        return z

    def wbfbt_cheb(self, r, iters, lmin_l, lmax_l, lmin_r, lmax_r, state=None) -> np.ndarray:
        """wBFBT with Chebyshev-Jacobi inner Poisson solves on the given intervals (R16)."""
        s = self.state if state is None else state
        r = _f64(r)
        z = np.zeros(self.n_p)
        self.L.or_wbfbt_cheb(self.h, _p(self.mu_q), _p(s["Cinv"]), _p(s["Dinv"]), _p(s["diagKl"]),
                             _p(s["diagKr"]), _p(r), _p(z), int(iters), float(lmin_l), float(lmax_l),
                             float(lmin_r), float(lmax_r))
        return z

    @staticmethod
    def set_order(order) -> None:
        """Summation order of element scatter-adds and dot products (process-wide), changed
        only to measure the self-discrepancy delta_self: 0 / False
        ascending (default), 1 / True reversed, 2 even-then-odd dot products."""
        lib().or_set_order(int(order))

    @staticmethod
    def num_threads() -> int:
        return int(lib().or_num_threads())
