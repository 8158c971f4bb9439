"""GPU tests of the C-ABI contract (error codes, masking, aliasing, host entry)
and full-size (BASELINE.json C4/C5) parity in the launch configuration
bench.py times: complete B / B^T / A vectors where the oracle is fast enough,
sampled A outputs otherwise, and size-independent properties."""
import numpy as np
import pytest

import synth
from tests.gpu_common import Pair, dev, empty, host, rel_l2

pytestmark = pytest.mark.gpu


def test_errors():
    import torch
    from paper_1607_03936_b200 import Context, WBError
    ctx = Context(3, 2)
    u = empty(ctx.n_v)
    with pytest.raises(WBError, match="WB_ESTATE"):
        ctx.apply_A(u, empty(ctx.n_v))
    mu = torch.ones(ctx.n_el * ctx.n_q, dtype=torch.float64, device="cuda")
    mu[5] = 0.0
    with pytest.raises(WBError, match="WB_ENONPOS_MU"):
        ctx.set_viscosity(mu)
    mu[5] = float("nan")
    with pytest.raises(WBError, match="WB_ENONPOS_MU"):
        ctx.set_viscosity(mu)
    mu[5] = 1.0
    with pytest.raises(WBError, match="WB_EINVAL"):
        ctx.set_viscosity(mu, 0.5, 1.0)
    ctx.set_viscosity(mu)
    with pytest.raises(WBError, match="WB_EALIAS"):
        ctx.apply_A(u, u)
    with pytest.raises(WBError, match="WB_EINVAL"):
        ctx.apply_K(2, empty(ctx.n_p), empty(ctx.n_p))
    with pytest.raises(WBError, match="WB_EINVAL"):
        Context(0, 2)
    with pytest.raises(WBError, match="WB_EINVAL"):
        Context(4, 5)
    with pytest.raises(WBError, match="WB_EINVAL"):
        Context(4, 2, flags=8)  # unknown flag bit


def test_strict_lump_flag():
    from paper_1607_03936_b200 import WB_STRICT_LUMP, WBError
    p = Pair("C1", setup=False, flags=WB_STRICT_LUMP)
    with pytest.raises(WBError, match="WB_ENONPOS_LUMP"):
        p.ctx.set_viscosity(p.mu)


def test_boundary_inputs_ignored():
    p = Pair("C2", N=6)
    u = p.inp["u"].copy()
    mask = p.o.boundary_mask().astype(bool)
    u2 = u.copy()
    u2[mask] = 1e30
    for op, n in (("apply_A", p.ctx.n_v), ("apply_B", p.ctx.n_p)):
        a = host(getattr(p.ctx, op)(dev(u), empty(n)))
        b = host(getattr(p.ctx, op)(dev(u2), empty(n)))
        assert np.array_equal(a, b)


def test_nomask_rigid_modes():
    """Without the mask, A annihilates the six rigid modes (closed form)."""
    from paper_1607_03936_b200 import WB_DEBUG_NOMASK
    for cfg, N in (("C2", 4), ("C4", 2)):
        p = Pair(cfg, N=N, flags=WB_DEBUG_NOMASK)
        k, n = p.k, p.k * N + 1
        g = np.linspace(0, 1, n)  # GLL nodes are symmetric; positions only matter via linearity
        from oracle import Oracle
        xn = Oracle(1, k).tables()["xn"]
        line = np.concatenate([[(e + (xn[a] + 1) / 2) / N for a in range(k)] for e in range(N)] + [[1.0]])
        Z, Y, X = np.meshgrid(line, line, line, indexing="ij")
        x, y, z = X.ravel(), Y.ravel(), Z.ravel()
        zero = np.zeros_like(x)
        one = np.ones_like(x)
        modes = [np.concatenate(m) for m in ((one, zero, zero), (zero, one, zero), (zero, zero, one),
                                             (-y, x, zero), (-z, zero, x), (zero, -z, y))]
        ref = np.linalg.norm(host(p.ctx.apply_A(dev(p.inp["u"]), empty(p.ctx.n_v))))
        for m in modes:
            r = host(p.ctx.apply_A(dev(m), empty(p.ctx.n_v)))
            assert np.linalg.norm(r) <= 1e-12 * ref * np.linalg.norm(m) / np.linalg.norm(p.inp["u"])


def test_hotpath_host_equals_device():
    import torch
    p = Pair("C2", N=8, setup=False)
    c = p.ctx
    it = 10
    outs_d = [empty(c.n_v), empty(c.n_p), empty(c.n_v), empty(c.n_p)]
    c.hotpath(p.mu, dev(p.inp["u"]), dev(p.inp["p"]), it, *outs_d)
    outs_h = [np.empty(c.n_v), np.empty(c.n_p), np.empty(c.n_v), np.empty(c.n_p)]
    c.hotpath_host(p.inp["mu_q"], p.inp["u"], p.inp["p"], it, *outs_h)
    for a, b in zip(outs_d, outs_h):
        assert np.array_equal(host(a), b)
    pin = [torch.empty(n, dtype=torch.float64).pin_memory() for n in (c.n_v, c.n_p, c.n_v, c.n_p)]
    c.hotpath_host(torch.from_numpy(p.inp["mu_q"]).pin_memory(), torch.from_numpy(p.inp["u"]).pin_memory(),
                   torch.from_numpy(p.inp["p"]).pin_memory(), it, *pin)
    for a, b in zip(outs_d, pin):
        assert np.array_equal(host(a), b.numpy())


def test_unaligned_pointers():
    """Caller tensors need only 8-byte alignment (torch views at odd offsets)."""
    import torch
    for cfg, N in (("C2", 5), ("C4", 2)):
        p = Pair(cfg, N=N)
        c = p.ctx
        outs = {}
        for off in (0, 1):
            u = torch.zeros(c.n_v + 1, dtype=torch.float64, device="cuda")
            q = torch.zeros(c.n_p + 1, dtype=torch.float64, device="cuda")
            u[off:off + c.n_v] = dev(p.inp["u"])
            q[off:off + c.n_p] = dev(p.inp["p"])
            yA, yBT = empty(c.n_v + 1), empty(c.n_v + 1)
            pB, z = empty(c.n_p + 1), empty(c.n_p + 1)
            uu, qq = u[off:off + c.n_v], q[off:off + c.n_p]
            c.apply_A(uu, yA[off:off + c.n_v])
            c.apply_B(uu, pB[off:off + c.n_p])
            c.apply_BT(qq, yBT[off:off + c.n_v])
            c.apply_wbfbt(qq, z[off:off + c.n_p], 5)
            outs[off] = [host(t[off:off + n]) for t, n in ((yA, c.n_v), (pB, c.n_p), (yBT, c.n_v), (z, c.n_p))]
        for a, b in zip(outs[0], outs[1]):
            assert np.array_equal(a, b)


def test_amplified_boundary_weights():
    """a_l, a_r != 1 (eq:bdramp): lumped diagonals and wBFBT parity."""
    p = Pair("C2", a_l=1.0, a_r=4.0)
    st = p.ost
    Cw, Dw = empty(p.ctx.n_nodes), empty(p.ctx.n_nodes)
    p.ctx.get_lumped(Cw, Dw)
    assert np.max(np.abs(host(Dw) - st["Dw"])) <= 1e-13 * np.max(np.abs(st["Dw"]))
    assert np.max(np.abs(host(Cw) - st["Cw"])) <= 1e-13 * np.max(np.abs(st["Cw"]))
    z = host(p.ctx.apply_wbfbt(dev(p.inp["p"]), empty(p.ctx.n_p), 20))
    assert rel_l2(z, p.o.wbfbt(p.inp["p"], 20)) <= 1e-8


# ------------------------------------------------------------------ full BASELINE sizes
@pytest.fixture(scope="module", params=["C4", "C5"])
def full(request):
    return Pair(request.param)


def test_full_size_B_BT(full):
    u, p = full.inp["u"], full.inp["p"]
    assert rel_l2(host(full.ctx.apply_B(dev(u), empty(full.ctx.n_p))), full.o.apply_B(u)) <= 1e-11
    assert rel_l2(host(full.ctx.apply_BT(dev(p), empty(full.ctx.n_v))), full.o.apply_BT(p)) <= 1e-11


def test_full_size_A(full):
    """The complete A(mu)u vector at the BASELINE size against the oracle (north_star: <= 1e-11),
    plus the low-viscosity-region check (global l2 is dominated by the mu_max regions)."""
    u, mu = full.inp["u"], full.inp["mu_q"]
    y = host(full.ctx.apply_A(dev(u), empty(full.ctx.n_v)))
    yo = full.o.apply_A(mu, u)
    assert rel_l2(y, yo) <= 1e-11
    o = full.o
    low_el = mu.reshape(o.n_el, o.n_q).max(axis=1) < 10 * full.cfg.mu_min
    dm = o.dofmap().reshape(o.n_el, o.n_q)
    hi = np.zeros(o.n_nodes, bool)
    hi[np.unique(dm[~low_el])] = True
    sel = np.tile(~hi, 3) & ~o.boundary_mask().astype(bool)
    assert sel.sum() > 1000
    assert rel_l2(y[sel], yo[sel]) <= 1e-11


def test_full_size_lumped(full):
    Cw = empty(full.ctx.n_nodes)
    full.ctx.get_lumped(Cw)
    o = full.ost["Cw"]
    assert np.max(np.abs(host(Cw) - o)) <= 1e-13 * np.max(np.abs(o))
    assert full.ctx.query("n_nonpos_Cw") == full.ost["n_nonpos_Cw"] == 0


@pytest.mark.parametrize("iters", [1, 5, 10, 20])
def test_full_size_pcg_prefix(full, iters):
    """Prefix parity of the Poisson solve at the BASELINE size (SURVEY 8(c) 12(i')): <= 1e-12."""
    b = full.inp["p"]
    st = full.ost
    x = host(full.ctx.poisson_pcg(1, dev(b), empty(full.ctx.n_p), iters))
    assert rel_l2(x, full.o.poisson(st["Dinv"], st["diagKr"], b, iters)) <= 1e-12


def test_full_size_apply_K(full):
    b = full.inp["p"]
    for side, X in ((0, full.ost["Cinv"]), (1, full.ost["Dinv"])):
        q = host(full.ctx.apply_K(side, dev(b), empty(full.ctx.n_p)))
        assert rel_l2(q, full.o.apply_K(X, b)) <= 1e-11


def test_full_size_repeat_bitwise(full):
    """Race detector: repeated launches at full size are bitwise identical
    (A's tile look-back and staged loads, the fused K kernel, the PCG loop)."""
    c = full.ctx
    u, r = dev(full.inp["u"]), dev(full.inp["p"])
    ya = host(c.apply_A(u, empty(c.n_v)))
    for _ in range(10):
        assert np.array_equal(host(c.apply_A(u, empty(c.n_v))), ya)
    xk = host(c.poisson_pcg(1, r, empty(c.n_p), 10))
    for _ in range(5):
        assert np.array_equal(host(c.poisson_pcg(1, r, empty(c.n_p), 10)), xk)


def test_full_size_wbfbt(full):
    """Free-running wBFBT at the BASELINE size with the config's PCG count (C4: 2 x 50,
    C5: 2 x 100), compared element by element with the oracle:
    rel l2 <= 1e-8, or -- only where the oracle's self-discrepancy delta_self (itself under
    other summation orders) exceeds 1e-9, i.e. the fixed-iteration CG itself amplifies
    rounding that far -- the Poisson relative residuals agreeing within 2x.  Also
    finite, projected and bitwise deterministic."""
    import json
    import os
    c = full.ctx
    it = full.cfg.iters
    r = full.inp["p"]
    z1 = host(c.apply_wbfbt(dev(r), empty(c.n_p), it))
    z2 = host(c.apply_wbfbt(dev(r), empty(c.n_p), it))
    assert np.all(np.isfinite(z1)) and np.array_equal(z1, z2)
    assert abs(z1[::full.o.n_m].sum()) <= 1e-10 * np.abs(z1[::full.o.n_m]).sum()
    zo = full.o.wbfbt(r, it)
    err = rel_l2(z1, zo)
    rec = dict(cfg=full.cfg.name, N=full.N, k=full.k, iters=it, err=err)
    if err > 1e-8:
        from tests.test_gpu_parity import self_discrepancy
        ds = self_discrepancy(full.o, r, it, zo=zo, orders=(1,))  # one other order decides > 1e-9
        rec["delta_self"] = ds
        st = full.ost
        b = full.o.project(r)
        xg = host(c.poisson_pcg(1, dev(b), empty(c.n_p), it))
        rg = full.o.poisson_relres(st["Dinv"], b, xg)
        ro = full.o.poisson_relres(st["Dinv"], b, full.o.poisson(st["Dinv"], st["diagKr"], b, it))
        rec.update(relres_gpu=rg, relres_oracle=ro)
    print("full-size wBFBT parity:", json.dumps(rec))
    out = os.environ.get("WB_PARITY_LOG")
    if out:
        with open(out, "a") as f:
            f.write(json.dumps(rec) + "\n")
    if err <= 1e-8:
        return
    # where delta_self > 1e-9 the free-running criterion is limited by the
    # fixed-iteration CG's sensitivity, and the robust check is the Poisson residuals within 2x
    assert rec["delta_self"] > 1e-9, rec
    assert rec["relres_gpu"] <= 2 * rec["relres_oracle"] and rec["relres_oracle"] <= 2 * rec["relres_gpu"], rec


@pytest.mark.parametrize("cfg,N", [("C2", 6), ("C1", None)])
def test_pcg_scalars_match_oracle(cfg, N):
    """WB_DEBUG_SCALARS: the last solve's alpha_i / beta_i (device histories) against the
    oracle's recorded O9 scalars on the same projected right-hand side.  The first
    iterations agree to rounding; later ones drift with CG's sensitivity, so they are
    checked at a looser bound."""
    from paper_1607_03936_b200 import WB_DEBUG_SCALARS, WBError
    p = Pair(cfg, N=N, flags=WB_DEBUG_SCALARS)
    iters = 12
    b = p.inp["p"]
    p.ctx.poisson_pcg(1, dev(b), empty(p.ctx.n_p), iters)
    assert p.ctx.query("pcg_iters") == iters
    _, al, be, run = p.o.pcg_scalars(p.ost["Dinv"], p.ost["diagKr"], p.o.project(b), iters)
    assert run == iters
    ga = np.array([p.ctx.query(f"alpha_{i}") for i in range(iters)])
    gb = np.array([p.ctx.query(f"beta_{i}") for i in range(iters)])
    assert p.ctx.query("last_alpha_beta") == ga[-1] and p.ctx.query("last_beta") == gb[-1]
    # (no sign check: with row-sum lumping D_w may have nonpositive entries, K indefinite)
    np.testing.assert_allclose(ga[:4], al[:4], rtol=1e-10)
    np.testing.assert_allclose(gb[:4], be[:4], rtol=1e-9)
    np.testing.assert_allclose(ga, al, rtol=1e-3)  # C1's K is indefinite: rounding grows
    with pytest.raises(WBError, match="WB_EINVAL"):
        p.ctx.query(f"alpha_{iters}")


def test_pcg_scalars_need_flag():
    from paper_1607_03936_b200 import WBError
    p = Pair("C1")
    p.ctx.poisson_pcg(1, dev(p.inp["p"]), empty(p.ctx.n_p), 3)
    with pytest.raises(WBError, match="WB_ESTATE"):
        p.ctx.query("alpha_0")


@pytest.mark.parametrize("N", [44, 46, 45])
def test_large_poisson_paths_ragged_tiles(N):
    """The large-mesh Poisson kernels with tiles ragged in y and z (4x8x8 tiles): the TMA
    kernel (even N with >= 75,776 elements: N = 44, 46) and the pointer kernel it falls
    back to for odd N (N = 45).  apply_K on both sides and a 5-iteration PCG against the
    oracle; for the TMA kernel its four variants (z box or r + Minv boxes, plain or
    warp-specialised) bitwise equal."""
    p = Pair("C5", N=N)
    tma = 1 if N % 2 == 0 else 0
    assert p.ctx.query("k_tma") == tma
    st = p.ost
    b = p.inp["p"]
    for ws in (0, 1):
        p.ctx.set_option("k_ws", ws)
        assert p.ctx.query("k_ws") == ws * tma
        if st["n_nonpos_Cw"] == 0:
            for side, X in ((0, st["Cinv"]), (1, st["Dinv"])):
                q = host(p.ctx.apply_K(side, dev(b), empty(p.ctx.n_p)))
                assert rel_l2(q, p.o.apply_K(X, b)) <= 1e-11
    xs = []
    for ws in (0, 1):
        p.ctx.set_option("k_ws", ws)
        for kz in (1, 0):
            p.ctx.set_option("kz", kz)
            xs.append(host(p.ctx.poisson_pcg(1, dev(b), empty(p.ctx.n_p), 5)))
    for x in xs[1:]:
        assert np.array_equal(xs[0], x)
    assert rel_l2(xs[0], p.o.poisson(st["Dinv"], st["diagKr"], b, 5)) <= 1e-12
    if tma:  # the opt-in node-owner z-march kernel (k_zm), every tile variant
        p.ctx.set_option("k_ws", 0)
        p.ctx.set_option("k_zm", 1)
        assert p.ctx.query("k_zm") == 1
        try:
            for var in range(5):
                p.ctx.set_option("zm_var", var)
                q = host(p.ctx.apply_K(1, dev(b), empty(p.ctx.n_p)))
                assert rel_l2(q, p.o.apply_K(st["Dinv"], b)) <= 1e-11
                x = host(p.ctx.poisson_pcg(1, dev(b), empty(p.ctx.n_p), 5))
                assert rel_l2(x, p.o.poisson(st["Dinv"], st["diagKr"], b, 5)) <= 1e-12
        finally:
            p.ctx.set_option("k_zm", 0)


def test_nonpos_counts_per_side():
    """n_nonpos_Cw / n_nonpos_Dw count their own side (a_l != a_r makes them differ):
    each equals the number of nonpositive interior entries of the returned array."""
    p = Pair("C3", N=12, a_l=1.0, a_r=3.0)
    Cw, Dw = empty(p.ctx.n_nodes), empty(p.ctx.n_nodes)
    p.ctx.get_lumped(Cw, Dw)
    interior = p.o.boundary_mask()[:p.ctx.n_nodes] == 0
    nc = int(np.sum((host(Cw) <= 0) & interior))
    nd = int(np.sum((host(Dw) <= 0) & interior))
    assert nc != nd
    assert p.ctx.query("n_nonpos_Cw") == nc
    assert p.ctx.query("n_nonpos_Dw") == nd


def test_pcg_failure_detection():
    """a healthy solve reports no non-finite PCG scalars; a right-hand side with a
    NaN entry does (the status of an asynchronous apply cannot carry it)."""
    import torch
    from paper_1607_03936_b200 import WBError
    p = Pair("C2", N=6)
    with pytest.raises(WBError, match="WB_ESTATE"):
        p.ctx.query("pcg_nonfinite")
    b = p.inp["p"].copy()
    p.ctx.poisson_pcg(1, dev(b), empty(p.ctx.n_p), 10)
    assert p.ctx.query("pcg_nonfinite") == 0
    b[17] = float("nan")
    x = p.ctx.poisson_pcg(1, dev(b), empty(p.ctx.n_p), 10)
    assert p.ctx.query("pcg_nonfinite") > 0
    assert not bool(torch.isfinite(x).all())
