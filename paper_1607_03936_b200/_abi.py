"""ctypes binding of libwbfbt.so (include/wbfbt.h).  Argument marshalling only.

Every method of `Context` maps 1:1 onto a C entry point of the same name
without the `wb_` prefix; see include/wbfbt.h for the operation each one
computes (with its PAPER.md citation), the layouts and the error behaviour.
Device arrays are torch.float64 CUDA tensors, contiguous; the C calls are
enqueued on the context's stream (torch's current stream at creation, or the
one given to `set_stream`).
"""
from __future__ import annotations

import ctypes as C
import os
from math import comb

HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(HERE, "libwbfbt.so")

WB_STRICT_LUMP = 1
WB_DEBUG_NOMASK = 2
WB_DEBUG_SCALARS = 4

_STATUS = {0: "WB_OK", -1: "WB_EINVAL", -2: "WB_ENONPOS_MU", -3: "WB_ENONPOS_LUMP", -4: "WB_ECUDA",
           -5: "WB_ENOMEM", -6: "WB_EALIAS", -7: "WB_ESTATE"}

_vp, _d, _i, _u, _i64p = C.c_void_p, C.c_double, C.c_int, C.c_uint, C.POINTER(C.c_int64)

# (name, restype, argtypes) -- the exported C ABI, in header order
SYMBOLS = [
    ("wb_version", C.c_char_p, []),
    ("wb_create", _i, [C.POINTER(_vp), _i, _i, _u, _vp]),
    ("wb_destroy", None, [_vp]),
    ("wb_set_stream", _i, [_vp, _vp]),
    ("wb_last_error", C.c_char_p, [_vp]),
    ("wb_sizes", _i, [_vp, _i64p, _i64p, _i64p, _i64p, _i64p]),
    ("wb_get_dofmap", _i, [_vp, _vp]),
    ("wb_get_boundary_mask", _i, [_vp, _vp]),
    ("wb_set_viscosity", _i, [_vp, _vp, _d, _d]),
    ("wb_apply_A", _i, [_vp, _vp, _vp]),
    ("wb_apply_B", _i, [_vp, _vp, _vp]),
    ("wb_apply_BT", _i, [_vp, _vp, _vp]),
    ("wb_apply_K", _i, [_vp, _i, _vp, _vp]),
    ("wb_poisson_pcg", _i, [_vp, _i, _vp, _vp, _i]),
    ("wb_poisson_cheb", _i, [_vp, _i, _vp, _vp, _i, _d, _d]),
    ("wb_poisson_eigmax", _i, [_vp, _i, _vp, _i, C.POINTER(_d)]),
    ("wb_get_diagA", _i, [_vp, _vp]),
    ("wb_set_inner_cheb", _i, [_vp, _d, _d, _d, _d]),
    ("wb_set_schur", _i, [_vp, _i]),
    ("wb_apply_dabfbt", _i, [_vp, _vp, _vp, _i]),
    ("wb_apply_mpinv", _i, [_vp, _vp, _vp]),
    ("wb_load_vector", _i, [_vp, _vp, _vp]),
    ("wb_setup_mg", _i, [_vp, _i, _vp]),
    ("wb_velocity_vcycle", _i, [_vp, _vp, _vp]),
    ("wb_set_velocity_mg", _i, [_vp, _i]),
    ("wb_mg_vcycle", _i, [_vp, _i, _vp, _vp]),
    ("wb_poisson_mgcg", _i, [_vp, _i, _vp, _vp, _i]),
    ("wb_set_inner_mg", _i, [_vp, _i]),
    ("wb_mg_get_lumped", _i, [_vp, _i, _vp, _vp]),
    ("wb_velocity_cheb", _i, [_vp, _vp, _vp, _i, _d, _d]),
    ("wb_velocity_eigmax", _i, [_vp, _vp, _i, C.POINTER(_d)]),
    ("wb_stokes_fgmres", _i, [_vp, _vp, _vp, _vp, _vp, _i, _i, _d, _i, _i, _d, _d, C.POINTER(_i), C.POINTER(_d)]),
    ("wb_apply_wbfbt", _i, [_vp, _vp, _vp, _i]),
    ("wb_hotpath", _i, [_vp, _vp, _d, _d, _vp, _vp, _i, _vp, _vp, _vp, _vp]),
    ("wb_hotpath_host", _i, [_vp, _vp, _d, _d, _vp, _vp, _i, _vp, _vp, _vp, _vp]),
    ("wb_slab_create", _i, [C.POINTER(_vp), _i, _i, _i, _i, _u, _vp]),
    ("wb_slab_set_comm", _i, [_vp, _vp]),
    ("wb_debug_pcg_step", _i, [_vp, _i, _vp, _vp, _vp, C.POINTER(_d)]),
    ("wb_get_lumped", _i, [_vp, _vp, _vp, _vp, _vp]),
    ("wb_get_jacobi", _i, [_vp, _vp, _vp]),
    ("wb_query", _i, [_vp, C.c_char_p, C.POINTER(_d)]),
    ("wb_set_option", _i, [_vp, C.c_char_p, _d]),
    ("wb_sync", _i, [_vp]),
]

_lib = None


class WBError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{_STATUS.get(status, status)}: {msg}")
        self.status = status


def library_path() -> str:
    return _LIB_PATH


def lib():
    """Load libwbfbt.so (must have been built; see paper_1607_03936_b200/build.py)."""
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            raise ImportError(f"libwbfbt.so not built at {_LIB_PATH}: run "
                              "`python -m paper_1607_03936_b200.build` (no CPU fallback exists)")
        L = C.CDLL(_LIB_PATH)
        for name, res, args in SYMBOLS:
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def version() -> str:
    return lib().wb_version().decode()


def sizes(N: int, k: int) -> dict:
    n1 = k + 1
    n_nodes = (k * N + 1) ** 3
    return dict(n_el=N ** 3, n_nodes=n_nodes, n_v=3 * n_nodes, n_p=comb(k + 2, 3) * N ** 3, n_q=n1 ** 3,
                n_m=comb(k + 2, 3))


def _ptr(t, n: int, dtype_name: str = "float64"):
    import torch
    if not isinstance(t, torch.Tensor):
        raise TypeError("expected a torch tensor")
    if not t.is_cuda:
        raise ValueError("expected a CUDA tensor (device pointer)")
    if str(t.dtype) != f"torch.{dtype_name}":
        raise TypeError(f"expected torch.{dtype_name}, got {t.dtype}")
    if not t.is_contiguous():
        raise ValueError("expected a contiguous tensor")
    if t.numel() != n:
        raise ValueError(f"expected {n} elements, got {t.numel()}")
    return C.c_void_p(t.data_ptr())


def _hptr(a, n: int):
    """Host float64 buffer (numpy array or CPU torch tensor) -> pointer."""
    import numpy as np
    try:
        import torch
        if isinstance(a, torch.Tensor):
            if a.is_cuda or a.dtype != torch.float64 or not a.is_contiguous() or a.numel() != n:
                raise ValueError("expected a contiguous CPU float64 tensor of the right size")
            return C.c_void_p(a.data_ptr())
    except ImportError:
        pass
    if not (isinstance(a, np.ndarray) and a.dtype == np.float64 and a.flags.c_contiguous and a.size == n):
        raise ValueError("expected a contiguous float64 numpy array of the right size")
    return C.c_void_p(a.ctypes.data)


class Context:
    """One mesh (N^3 elements, Q_k x P_{k-1}^disc) on one CUDA stream."""

    def __init__(self, N: int, k: int, flags: int = 0, stream=None):
        import torch
        self._L = lib()
        if stream is None:
            stream = torch.cuda.current_stream().cuda_stream
        h = C.c_void_p()
        st = self._L.wb_create(C.byref(h), int(N), int(k), int(flags), C.c_void_p(int(stream)))
        if st != 0:
            raise WBError(st, f"wb_create(N={N}, k={k}) failed")
        self._h = h
        self.N, self.k, self.flags = N, k, flags
        v = [C.c_int64() for _ in range(5)]
        self._check(self._L.wb_sizes(h, *[C.byref(x) for x in v]))
        self.n_el, self.n_nodes, self.n_v, self.n_p, self.n_q = (int(x.value) for x in v)

    # -- plumbing
    def _check(self, st: int):
        if st != 0:
            msg = self._L.wb_last_error(self._h)
            raise WBError(st, msg.decode() if msg else "")

    def close(self):
        if getattr(self, "_h", None):
            self._L.wb_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_stream(self, stream):
        self._check(self._L.wb_set_stream(self._h, C.c_void_p(int(stream))))

    def sync(self):
        self._check(self._L.wb_sync(self._h))

    def query(self, key: str) -> float:
        v = C.c_double()
        self._check(self._L.wb_query(self._h, key.encode(), C.byref(v)))
        return v.value

    def set_option(self, key: str, value: float):
        self._check(self._L.wb_set_option(self._h, key.encode(), float(value)))

    # -- row a1
    def get_dofmap(self, out):
        self._check(self._L.wb_get_dofmap(self._h, _ptr(out, self.n_el * self.n_q, "int64")))
        return out

    def get_boundary_mask(self, out):
        self._check(self._L.wb_get_boundary_mask(self._h, _ptr(out, self.n_v, "uint8")))
        return out

    # -- rows a3, a4
    def set_viscosity(self, mu_q, a_l: float = 1.0, a_r: float = 1.0):
        self._check(self._L.wb_set_viscosity(self._h, _ptr(mu_q, self.n_el * self.n_q), float(a_l), float(a_r)))

    def get_lumped(self, Cw=None, Dw=None, Cinv=None, Dinv=None):
        f = lambda t: _ptr(t, self.n_nodes) if t is not None else None  # noqa: E731
        self._check(self._L.wb_get_lumped(self._h, f(Cw), f(Dw), f(Cinv), f(Dinv)))

    def get_jacobi(self, dKl=None, dKr=None):
        f = lambda t: _ptr(t, self.n_p) if t is not None else None  # noqa: E731
        self._check(self._L.wb_get_jacobi(self._h, f(dKl), f(dKr)))

    # -- rows a5 - a10
    def apply_A(self, u, y):
        self._check(self._L.wb_apply_A(self._h, _ptr(u, self.n_v), _ptr(y, self.n_v)))
        return y

    def apply_B(self, u, p):
        self._check(self._L.wb_apply_B(self._h, _ptr(u, self.n_v), _ptr(p, self.n_p)))
        return p

    def apply_BT(self, p, y):
        self._check(self._L.wb_apply_BT(self._h, _ptr(p, self.n_p), _ptr(y, self.n_v)))
        return y

    def apply_K(self, side: int, p, q):
        self._check(self._L.wb_apply_K(self._h, int(side), _ptr(p, self.n_p), _ptr(q, self.n_p)))
        return q

    def poisson_pcg(self, side: int, b, x, iters: int):
        self._check(self._L.wb_poisson_pcg(self._h, int(side), _ptr(b, self.n_p), _ptr(x, self.n_p), int(iters)))
        return x

    def poisson_cheb(self, side: int, b, x, iters: int, lmin: float, lmax: float):
        self._check(self._L.wb_poisson_cheb(self._h, int(side), _ptr(b, self.n_p), _ptr(x, self.n_p), int(iters),
                                            float(lmin), float(lmax)))
        return x

    def poisson_eigmax(self, side: int, v0, iters: int) -> float:
        lam = C.c_double(0.0)
        self._check(self._L.wb_poisson_eigmax(self._h, int(side), _ptr(v0, self.n_p), int(iters), C.byref(lam)))
        return lam.value

    def set_inner_cheb(self, lmin_l=0.0, lmax_l=0.0, lmin_r=0.0, lmax_r=0.0):
        self._check(self._L.wb_set_inner_cheb(self._h, float(lmin_l), float(lmax_l), float(lmin_r), float(lmax_r)))

    # -- Schur-complement variants
    def set_schur(self, kind: int):
        self._check(self._L.wb_set_schur(self._h, int(kind)))

    def apply_dabfbt(self, r, z, iters: int):
        self._check(self._L.wb_apply_dabfbt(self._h, _ptr(r, self.n_p), _ptr(z, self.n_p), int(iters)))
        return z

    def apply_mpinv(self, r, z):
        self._check(self._L.wb_apply_mpinv(self._h, _ptr(r, self.n_p), _ptr(z, self.n_p)))
        return z

    # -- load vector of a body force sampled at the Gauss points
    def load_vector(self, fq, F):
        self._check(self._L.wb_load_vector(self._h, _ptr(fq, 3 * self.n_el * self.n_q), _ptr(F, self.n_v)))
        return F

    # -- geometric pressure multigrid (R20)
    def setup_mg(self, nu: int = 3, mu=None):
        self._check(self._L.wb_setup_mg(self._h, int(nu),
                                        _ptr(mu, self.n_el * self.n_q) if mu is not None else None))

    def velocity_vcycle(self, b, x):
        self._check(self._L.wb_velocity_vcycle(self._h, _ptr(b, self.n_v), _ptr(x, self.n_v)))
        return x

    def set_velocity_mg(self, cycles: int = 0):
        self._check(self._L.wb_set_velocity_mg(self._h, int(cycles)))

    def mg_vcycle(self, side: int, b, x):
        self._check(self._L.wb_mg_vcycle(self._h, int(side), _ptr(b, self.n_p), _ptr(x, self.n_p)))
        return x

    def poisson_mgcg(self, side: int, b, x, iters: int):
        self._check(self._L.wb_poisson_mgcg(self._h, int(side), _ptr(b, self.n_p), _ptr(x, self.n_p), int(iters)))
        return x

    def set_inner_mg(self, iters: int = 0):
        self._check(self._L.wb_set_inner_mg(self._h, int(iters)))

    def mg_get_lumped(self, level: int, Cw=None, Dw=None):
        n = (int(self.query(f"mg_k_{int(level)}")) * int(self.query(f"mg_N_{int(level)}")) + 1) ** 3
        f = lambda t: _ptr(t, n) if t is not None else None  # noqa: E731
        self._check(self._L.wb_mg_get_lumped(self._h, int(level), f(Cw), f(Dw)))

    def get_diagA(self, dA):
        self._check(self._L.wb_get_diagA(self._h, _ptr(dA, self.n_v)))
        return dA

    def velocity_cheb(self, b, x, iters: int, lmin: float, lmax: float):
        self._check(self._L.wb_velocity_cheb(self._h, _ptr(b, self.n_v), _ptr(x, self.n_v), int(iters), float(lmin),
                                             float(lmax)))
        return x

    def velocity_eigmax(self, v0, iters: int) -> float:
        lam = C.c_double(0.0)
        self._check(self._L.wb_velocity_eigmax(self._h, _ptr(v0, self.n_v), int(iters), C.byref(lam)))
        return lam.value

    def stokes_fgmres(self, f, g, u, p, restart: int, max_iters: int, rtol: float, pcg_iters: int,
                      smooth_iters: int, lmin: float, lmax: float):
        """Returns (u, p, iterations, relres)."""
        it, rr = C.c_int(0), C.c_double(0.0)
        self._check(self._L.wb_stokes_fgmres(self._h, _ptr(f, self.n_v), _ptr(g, self.n_p), _ptr(u, self.n_v),
                                             _ptr(p, self.n_p), int(restart), int(max_iters), float(rtol),
                                             int(pcg_iters), int(smooth_iters), float(lmin), float(lmax),
                                             C.byref(it), C.byref(rr)))
        return u, p, it.value, rr.value

    def apply_wbfbt(self, r, z, iters: int):
        self._check(self._L.wb_apply_wbfbt(self._h, _ptr(r, self.n_p), _ptr(z, self.n_p), int(iters)))
        return z

    def hotpath(self, mu_q, u, p, iters: int, yA, pB, yBT, z, a_l: float = 1.0, a_r: float = 1.0):
        self._check(self._L.wb_hotpath(self._h, _ptr(mu_q, self.n_el * self.n_q), float(a_l), float(a_r),
                                       _ptr(u, self.n_v), _ptr(p, self.n_p), int(iters), _ptr(yA, self.n_v),
                                       _ptr(pB, self.n_p), _ptr(yBT, self.n_v), _ptr(z, self.n_p)))

    def hotpath_host(self, mu_q, u, p, iters: int, yA, pB, yBT, z, a_l: float = 1.0, a_r: float = 1.0):
        self._check(self._L.wb_hotpath_host(self._h, _hptr(mu_q, self.n_el * self.n_q), float(a_l), float(a_r),
                                            _hptr(u, self.n_v), _hptr(p, self.n_p), int(iters),
                                            _hptr(yA, self.n_v), _hptr(pB, self.n_p), _hptr(yBT, self.n_v),
                                            _hptr(z, self.n_p)))

    def debug_pcg_step(self, side: int, x, r, p, rz: float) -> float:
        v = C.c_double(rz)
        self._check(self._L.wb_debug_pcg_step(self._h, int(side), _ptr(x, self.n_p), _ptr(r, self.n_p),
                                              _ptr(p, self.n_p), C.byref(v)))
        return v.value
