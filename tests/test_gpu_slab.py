"""z-slab domain decomposition (wbfbt.h "z-slab") against the oracle on
the GLOBAL box mesh N x N x (R N) (oracle/: or_create_box, pinned in tests/test_oracle_box.py).

R slab contexts live in this one process on the one GPU, each driven by its own host thread
(`ThreadComm`: the threads meet at host barriers; no kernel waits for another).  Every rank's
local result is compared element by element with the oracle's global result restricted to the
rank's cube, shared planes included (both owners must hold the full sum, bit-identical).

Tolerances are the single-GPU ones: applies 1e-11 relative l2, lumped 1e-13 of the maximum,
PCG prefixes 1e-12 (1e-10 at 10 iterations), wBFBT with few iterations 1e-9.
"""
import threading

import numpy as np
import pytest

import synth
from tests.gpu_common import dev, empty, host, rel_l2

pytestmark = pytest.mark.gpu

# (N, k, R): even (TMA-capable) and odd cubes, k = 2 and 4, 1..3 ranks; (16, 2, 2) spans several
# kernel tiles per rank; the C5-size case is test_full_size_C5_per_rank_two_ranks below
CASES = [(4, 2, 1), (4, 2, 2), (5, 2, 2), (6, 2, 3), (16, 2, 2), (13, 2, 3), (3, 4, 2), (8, 4, 2), (6, 3, 2)]


def run_ranks(R, fn, comms=None):
    """fn(rank) on R host threads; re-raises the first failure (a failing rank breaks the
    barrier so that the others leave their collective with an error instead of waiting)."""
    out, errs = [None] * R, []

    def body(r):
        try:
            out[r] = fn(r)
        except BaseException as e:  # noqa: BLE001
            errs.append(e)
            if comms:
                comms[0].sh["barrier"].abort()

    th = [threading.Thread(target=body, args=(r,)) for r in range(R)]
    for t in th:
        t.start()
    for t in th:
        t.join(600)
    if errs:
        raise errs[0]
    return out


class SlabCase:
    def __init__(self, N, k, R, a_l=1.0, a_r=1.0, seed=0, cfg=None):
        from oracle import Oracle
        from tests.gpu_common import K3
        cfg = cfg or {2: "C2", 3: K3, 4: "C4"}[k]
        from paper_1607_03936_b200 import SlabContext, ThreadComm
        self.N, self.k, self.R = N, k, R
        self.o = Oracle(N, k, Nz=R * N)
        o = self.o
        # per-rank multi-sinker viscosity (the recipe of synth/ on each cube), global = z-stacked
        parts = [synth.make_inputs(cfg, seed + r, N=N)["mu_q"] for r in range(R)]
        self.mu = np.concatenate(parts)
        assert self.mu.size == o.n_el * o.n_q
        rng = np.random.default_rng(100 + seed)
        self.u = rng.standard_normal(o.n_v)
        self.p = rng.standard_normal(o.n_p)
        self.ost = o.setup(self.mu, a_l, a_r)
        self.a_l, self.a_r = a_l, a_r
        comms = ThreadComm.group(R, SlabContext.plane_cap(N, k), "cuda")
        self.comms = comms
        self.ctx = [SlabContext(N, k, comms[r]) for r in range(R)]
        c0 = self.ctx[0]
        self.nl_el, self.nl_nodes, self.nl_p = c0.n_el, c0.n_nodes, c0.n_p
        self.np_plane = (k * N + 1) ** 2
        mus = [dev(parts[r]) for r in range(R)]
        run_ranks(R, lambda r: self.ctx[r].set_viscosity(mus[r], a_l, a_r), comms)

    # global -> rank-local views
    def loc_p(self, v, r):
        return np.ascontiguousarray(v[r * self.nl_p:(r + 1) * self.nl_p])

    def loc_nodal(self, v, r):
        """One nodal field of the global box -> the rank's cube (both z planes included)."""
        g0 = r * self.k * self.N * self.np_plane
        return np.ascontiguousarray(v[g0:g0 + self.nl_nodes])

    def loc_v(self, v, r):
        n = self.o.n_nodes
        return np.concatenate([self.loc_nodal(v[c * n:(c + 1) * n], r) for c in range(3)])

    def close(self):
        for c in self.ctx:
            c.close()


@pytest.fixture(scope="module", params=CASES, ids=lambda c: f"N{c[0]}-k{c[1]}-R{c[2]}")
def case(request):
    N, k, R = request.param
    c = SlabCase(N, k, R, a_l=2.0, a_r=3.0)
    yield c
    c.close()


def test_sizes_and_mask(case):
    import torch
    for r, ctx in enumerate(case.ctx):
        assert (ctx.n_el, ctx.n_p) == (case.N ** 3, case.o.n_p // case.R)
        b = torch.empty(ctx.n_v, dtype=torch.uint8, device="cuda")
        ctx.get_boundary_mask(b)
        assert np.array_equal(host(b), case.loc_v(case.o.boundary_mask(), r).astype(np.uint8))


def test_lumped_and_jacobi(case):
    def f(r):
        ctx = case.ctx[r]
        Cw, Dw, Ci, Di = (empty(ctx.n_nodes) for _ in range(4))
        ctx.get_lumped(Cw, Dw, Ci, Di)
        dl, dr = empty(ctx.n_p), empty(ctx.n_p)
        ctx.get_jacobi(dl, dr)
        return [host(t) for t in (Cw, Dw, Ci, Di, dl, dr)]
    res = run_ranks(case.R, f, case.comms)
    st = case.ost
    for r in range(case.R):
        Cw, Dw, Ci, Di, dl, dr = res[r]
        for got, key in ((Cw, "Cw"), (Dw, "Dw")):
            ref = case.loc_nodal(st[key], r)
            assert np.abs(got - ref).max() <= 1e-13 * np.abs(st[key]).max()
        for got, key in ((Ci, "Cinv"), (Di, "Dinv")):
            ref = case.loc_nodal(st[key], r)
            assert np.array_equal(got == 0.0, ref == 0.0)  # the global mask
            if _definite(case):  # (indefinite coarse meshes: entries that cancel to rounding, R9)
                assert rel_l2(got, ref) <= 1e-9
        assert rel_l2(dl, case.loc_p(st["diagKl"], r)) <= 1e-12
        assert rel_l2(dr, case.loc_p(st["diagKr"], r)) <= 1e-12
    # the amplification really differs between the sides on the global boundary layer only
    assert not np.array_equal(st["Cw"], st["Dw"])


def test_shared_planes_bit_identical(case):
    if case.R < 2:
        pytest.skip("one rank")
    ps = [dev(case.loc_p(case.p, r)) for r in range(case.R)]
    us = [dev(case.loc_v(case.u, r)) for r in range(case.R)]

    def f(r):
        ctx = case.ctx[r]
        return host(ctx.apply_BT(ps[r], empty(ctx.n_v))), host(ctx.apply_A(us[r], empty(ctx.n_v)))
    res = run_ranks(case.R, f, case.comms)
    npl, nn = case.np_plane, case.nl_nodes
    for r in range(case.R - 1):
        for which in (0, 1):
            lo, hi = res[r][which].reshape(3, nn), res[r + 1][which].reshape(3, nn)
            assert np.array_equal(lo[:, nn - npl:], hi[:, :npl])


def test_apply_A_B_BT(case):
    us = [dev(case.loc_v(case.u, r)) for r in range(case.R)]
    ps = [dev(case.loc_p(case.p, r)) for r in range(case.R)]

    def f(r):
        ctx = case.ctx[r]
        return (host(ctx.apply_A(us[r], empty(ctx.n_v))), host(ctx.apply_B(us[r], empty(ctx.n_p))),
                host(ctx.apply_BT(ps[r], empty(ctx.n_v))))
    res = run_ranks(case.R, f, case.comms)
    yA, pB, yBT = case.o.apply_A(case.mu, case.u), case.o.apply_B(case.u), case.o.apply_BT(case.p)
    for r in range(case.R):
        assert rel_l2(res[r][0], case.loc_v(yA, r)) <= 1e-11
        assert rel_l2(res[r][1], case.loc_p(pB, r)) <= 1e-11
        assert rel_l2(res[r][2], case.loc_v(yBT, r)) <= 1e-11


@pytest.mark.parametrize("side", [0, 1])
def test_apply_K(case, side):
    ps = [dev(case.loc_p(case.p, r)) for r in range(case.R)]
    res = run_ranks(case.R, lambda r: host(case.ctx[r].apply_K(side, ps[r], empty(case.nl_p))), case.comms)
    q = case.o.apply_K(case.ost["Cinv" if side == 0 else "Dinv"], case.p)
    for r in range(case.R):
        assert rel_l2(res[r], case.loc_p(q, r)) <= 1e-11


def _definite(case):
    return case.ost["n_nonpos_Cw"] == 0 and case.ost["n_nonpos_Dw"] == 0


@pytest.mark.parametrize("iters", [1, 5, 10])
def test_pcg_prefix(case, iters):
    if not _definite(case):
        pytest.skip("indefinite K_w on this coarse mesh (R9)")
    bs = [dev(case.loc_p(case.p, r)) for r in range(case.R)]
    for side, xk, dk in ((0, "Cinv", "diagKl"), (1, "Dinv", "diagKr")):
        res = run_ranks(case.R, lambda r: host(case.ctx[r].poisson_pcg(side, bs[r], empty(case.nl_p), iters)),
                        case.comms)
        x = case.o.poisson(case.ost[xk], case.ost[dk], case.p, iters)
        got = np.concatenate(res)
        assert rel_l2(got, x) <= (1e-12 if iters <= 5 else 1e-10), (side, iters)
        # every rank used the same scalars: the global projection holds on the assembled result
        assert abs(got.reshape(-1, case.ctx[0].n_p // case.nl_el)[:, 0].sum()) <= 1e-9 * np.abs(got).sum()


def test_wbfbt(case):
    if not _definite(case):
        pytest.skip("indefinite K_w on this coarse mesh (R9)")
    rs = [dev(case.loc_p(case.p, r)) for r in range(case.R)]
    res = run_ranks(case.R, lambda r: host(case.ctx[r].apply_wbfbt(rs[r], empty(case.nl_p), 4)), case.comms)
    z = case.o.wbfbt(case.p, 4)
    assert rel_l2(np.concatenate(res), z) <= 1e-9


def test_hotpath_and_refusals(case):
    from paper_1607_03936_b200 import WBError
    ctx = case.ctx[0]
    with pytest.raises(WBError) as ei:
        ctx.poisson_cheb(0, empty(ctx.n_p), empty(ctx.n_p), 2, 0.1, 1.0)
    assert ei.value.status == -7
    with pytest.raises(WBError):
        ctx.setup_mg(3, None)
    # comm counters: the collective calls really went through the communicator
    if case.R > 1:
        assert case.comms[0].n_exchange > 0 and case.comms[0].n_allreduce > 0


def test_full_size_C5_per_rank_two_ranks():
    """BASELINE.json's C5 size on every rank (64^3 per rank, the 64 x 64 x 128 box; the z-marching
    B / B^T kernels and the tile A kernel of the large meshes): A, K_w and a 5-iteration PCG prefix
    against the oracle on the whole box."""
    c = SlabCase(64, 2, 2, cfg="C5")
    try:
        us = [dev(c.loc_v(c.u, r)) for r in range(2)]
        ps = [dev(c.loc_p(c.p, r)) for r in range(2)]

        def f(r):
            ctx = c.ctx[r]
            return (host(ctx.apply_A(us[r], empty(ctx.n_v))), host(ctx.apply_K(1, ps[r], empty(ctx.n_p))),
                    host(ctx.poisson_pcg(1, ps[r], empty(ctx.n_p), 5)))
        res = run_ranks(2, f, c.comms)
        yA = c.o.apply_A(c.mu, c.u)
        q = c.o.apply_K(c.ost["Dinv"], c.p)
        x = c.o.poisson(c.ost["Dinv"], c.ost["diagKr"], c.p, 5)
        for r in range(2):
            assert rel_l2(res[r][0], c.loc_v(yA, r)) <= 1e-11
            assert rel_l2(res[r][1], c.loc_p(q, r)) <= 1e-11
        assert rel_l2(np.concatenate([res[0][2], res[1][2]]), x) <= 1e-12
    finally:
        c.close()


def test_one_rank_slab_equals_cube_context():
    """nranks = 1 through the slab code path (unfused K_w, device-scalar PCG) against the plain
    cube context (fused kernels): same operators, rounding-level differences only."""
    from paper_1607_03936_b200 import Context, SlabContext, ThreadComm
    N, k = 8, 2
    inp = synth.make_inputs("C2", 3, N=N)
    mu = dev(inp["mu_q"])
    a = Context(N, k)
    b = SlabContext(N, k, ThreadComm.group(1, SlabContext.plane_cap(N, k), "cuda")[0])
    a.set_viscosity(mu, 1.0, 2.0)
    b.set_viscosity(mu, 1.0, 2.0)
    p = dev(inp["p"])
    za, zb = host(a.apply_wbfbt(p, empty(a.n_p), 5)), host(b.apply_wbfbt(p, empty(b.n_p), 5))
    assert rel_l2(zb, za) <= 1e-10


def test_slab_argument_and_callback_errors():
    """Boundary behaviour of the slab entry points (wbfbt.h "z-slab")."""
    import ctypes as C
    from paper_1607_03936_b200 import Context, SlabContext, ThreadComm, WBError, WB_DEBUG_NOMASK, lib
    L = lib()
    h = C.c_void_p()
    for N, k, rank, R, flags in [(4, 2, 2, 2, 0), (4, 2, -1, 2, 0), (4, 2, 0, 0, 0), (4, 2, 0, 2, WB_DEBUG_NOMASK),
                                 (0, 2, 0, 2, 0), (4, 5, 0, 2, 0)]:
        assert L.wb_slab_create(C.byref(h), N, k, rank, R, flags, None) == -1 and not h.value
    # buffers too small for the planes
    with pytest.raises(ValueError):
        SlabContext(8, 2, ThreadComm.group(1, 10, "cuda")[0])
    # not a slab context / null communicator
    ctx = Context(4, 2)
    assert L.wb_slab_set_comm(ctx._h, None) == -1
    comms = ThreadComm.group(2, SlabContext.plane_cap(4, 2), "cuda")
    s0 = SlabContext(4, 2, comms[0])
    assert L.wb_slab_set_comm(ctx._h, C.byref(s0._cs)) == -7
    # a multi-rank slab context refuses work before its communicator is registered
    raw = C.c_void_p()
    assert L.wb_slab_create(C.byref(raw), 4, 2, 0, 2, 0, None) == 0
    mu = dev(synth.make_inputs("C1", 0)["mu_q"])
    assert L.wb_set_viscosity(raw, C.c_void_p(mu.data_ptr()), 1.0, 1.0) == -7
    L.wb_destroy(raw)

    # a failing callback surfaces as an error with the Python exception attached
    class Bad(ThreadComm):
        def exchange(self, n):
            raise RuntimeError("link down")

        def allreduce(self, offset, n, op):
            raise RuntimeError("link down")
    shared = {"comms": [None, None], "barrier": None}
    bad = SlabContext(4, 2, Bad(0, 2, SlabContext.plane_cap(4, 2), "cuda", shared))
    with pytest.raises(WBError) as ei:
        bad.set_viscosity(mu)
    assert "link down" in str(ei.value)
    for c in (ctx, s0, bad):
        c.close()
