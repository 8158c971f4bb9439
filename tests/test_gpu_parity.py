"""GPU-vs-oracle parity (rows a1-a10 of SURVEY.md Sec. 8), through the C ABI.

Tolerances (north_star): dof map / mask bit-exact; single
applies of A, B, B^T relative l2 <= 1e-11; wBFBT relative l2 <= 1e-8 with the
PCG parity protocol (one-step <= 1e-13, prefix <= 1e-12) separating
implementation error from the fixed-iteration CG's own roundoff sensitivity.
Inputs: the seeded multi-sinker recipe of synth/ (DESIGN.md "Input recipe"),
at the BASELINE.json config sizes and at smaller/ragged N of the same recipe.
"""
import numpy as np
import pytest

import synth
from tests.gpu_common import K3, Pair, dev, empty, host, rel_l2

pytestmark = pytest.mark.gpu

# (config, N override) cases: small, ragged (N not a multiple of any block
# tile), and the configs' own sizes where the oracle is quick.
# k = 4 at N = 8 and 12 and k = 3 at N = 6 have positive lumped masses (definite K_w), so the
# Poisson, PCG and wBFBT parity tests run at high order too; C4 at N = 3, 5 and k = 3 at N = 3
# are indefinite (R9) and keep the one-step and apply checks.
SMALL = [("C1", None), ("C1", 1), ("C1", 2), ("C1", 5), ("C2", 7), ("C2", None), ("C4", 3), ("C4", 5),
         ("C4", 8), ("C4", 12), ("K3", None), ("K3", 3), ("C3", None)]


@pytest.fixture(scope="module", params=SMALL, ids=lambda c: f"{c[0]}-N{c[1]}")
def pair(request):
    cfg, N = request.param
    return Pair(K3 if cfg == "K3" else cfg, N)


# ------------------------------------------------------------------ a1
@pytest.mark.parametrize("N,k", [(1, 2), (2, 2), (5, 2), (3, 3), (1, 4), (4, 4), (24, 4), (64, 2)])
def test_dofmap_and_mask_bit_exact(N, k):
    import torch
    from oracle import Oracle
    from paper_1607_03936_b200 import Context
    ctx = Context(N, k)
    m = torch.empty(ctx.n_el * ctx.n_q, dtype=torch.int64, device="cuda")
    b = torch.empty(ctx.n_v, dtype=torch.uint8, device="cuda")
    ctx.get_dofmap(m)
    ctx.get_boundary_mask(b)
    if N <= 24:
        o = Oracle(N, k)
        assert np.array_equal(host(m), o.dofmap())
        assert np.array_equal(host(b), o.boundary_mask())
    nn1 = k * N + 1
    assert int(host(b).sum()) == 3 * (nn1 ** 3 - max(nn1 - 2, 0) ** 3)
    mm = host(m).reshape(ctx.n_el, ctx.n_q)
    assert mm.min() == 0 and mm.max() == nn1 ** 3 - 1
    assert len(np.unique(mm)) == nn1 ** 3


# ------------------------------------------------------------------ a5, a6, a7
def test_apply_A(pair):
    u = pair.inp["u"]
    y = host(pair.ctx.apply_A(dev(u), empty(pair.ctx.n_v)))
    yo = pair.o.apply_A(pair.inp["mu_q"], u)
    assert rel_l2(y, yo) <= 1e-11
    mask = pair.o.boundary_mask().astype(bool)
    assert np.all(y[mask] == 0.0)


def test_apply_A_low_mu_region(pair):
    """Relative error restricted to nodes whose elements all have mu < 10 mu_min
    (global l2 is dominated by the mu_max regions; SURVEY 8(c) pins)."""
    o, mu = pair.o, pair.inp["mu_q"]
    u = pair.inp["u"]
    y = host(pair.ctx.apply_A(dev(u), empty(pair.ctx.n_v)))
    yo = o.apply_A(mu, u)
    low_el = mu.reshape(o.n_el, o.n_q).max(axis=1) < 10 * pair.cfg.mu_min
    dm = o.dofmap().reshape(o.n_el, o.n_q)
    hi_nodes = np.zeros(o.n_nodes, bool)
    hi_nodes[np.unique(dm[~low_el])] = True
    sel = np.tile(~hi_nodes, 3) & ~o.boundary_mask().astype(bool)
    if sel.sum() < 10:
        pytest.skip("no low-viscosity region")
    assert rel_l2(y[sel], yo[sel]) <= 1e-11


def test_apply_B(pair):
    u = pair.inp["u"]
    p = host(pair.ctx.apply_B(dev(u), empty(pair.ctx.n_p)))
    assert rel_l2(p, pair.o.apply_B(u)) <= 1e-11


def test_apply_BT(pair):
    p = pair.inp["p"]
    y = host(pair.ctx.apply_BT(dev(p), empty(pair.ctx.n_v)))
    assert rel_l2(y, pair.o.apply_BT(p)) <= 1e-11
    assert np.all(y[pair.o.boundary_mask().astype(bool)] == 0.0)


def test_B_BT_adjoint_and_constants(pair):
    u, p = pair.inp["u"], pair.inp["p"]
    ctx = pair.ctx
    Bu = host(ctx.apply_B(dev(u), empty(ctx.n_p)))
    BTp = host(ctx.apply_BT(dev(p), empty(ctx.n_v)))
    um = u * (1 - pair.o.boundary_mask())
    lhs, rhs = Bu @ p, um @ BTp
    assert abs(lhs - rhs) <= 1e-13 * np.linalg.norm(Bu) * np.linalg.norm(p) * 10
    z0 = np.zeros(ctx.n_p)
    z0[::pair.o.n_m] = 2 * np.sqrt(2)
    y0 = host(ctx.apply_BT(dev(z0), empty(ctx.n_v)))
    assert np.linalg.norm(y0) <= 1e-13 * np.linalg.norm(BTp) * np.sqrt(ctx.n_p) + 1e-300


# ------------------------------------------------------------------ a3, a4
def test_lumped_and_jacobi(pair):
    ctx, st = pair.ctx, pair.ost
    Cw, Dw, Ci, Di = (empty(ctx.n_nodes) for _ in range(4))
    ctx.get_lumped(Cw, Dw, Ci, Di)
    for g, o in ((Cw, st["Cw"]), (Dw, st["Dw"])):
        assert np.max(np.abs(host(g) - o)) <= 1e-13 * np.max(np.abs(o))
    assert ctx.query("n_nonpos_Cw") == st["n_nonpos_Cw"]
    assert ctx.query("n_nonpos_Dw") == st["n_nonpos_Dw"]
    # inverses: compare where the lumped entry is well away from zero
    big = np.abs(st["Cw"]) > 1e-6 * np.max(np.abs(st["Cw"]))
    assert rel_l2(host(Ci)[big], st["Cinv"][big]) <= 1e-12
    dl, dr = empty(ctx.n_p), empty(ctx.n_p)
    ctx.get_jacobi(dl, dr)
    # diag K = sum_(c,a) B_e[m,(c,a)]^2 X[g]: entries of mixed sign on indefinite meshes are
    # compared in absolute terms against the largest contribution magnitude
    for g, o, X in ((dl, st["diagKl"], st["Cinv"]), (dr, st["diagKr"], st["Dinv"])):
        if st["n_nonpos_Cw"] == 0:
            assert rel_l2(host(g), o) <= 1e-12
        scale = pair.o.jacobi_diag(np.abs(X)).max()
        assert np.max(np.abs(host(g) - o)) <= 1e-12 * scale


# ------------------------------------------------------------------ a8
def test_apply_K(pair):
    """K_w p = B X^-1 B^T p on every case, indefinite ones included (a single apply is
    well-conditioned whatever the sign of X).  Where X changes sign the rounding scale is
    |B| |X| |B^T| |p|, so the bound there is relative to K evaluated with |X|."""
    p = pair.inp["p"]
    for side, X in ((0, pair.ost["Cinv"]), (1, pair.ost["Dinv"])):
        q = host(pair.ctx.apply_K(side, dev(p), empty(pair.ctx.n_p)))
        qo = pair.o.apply_K(X, p)
        assert rel_l2(q, qo) <= 1e-11 or np.linalg.norm(q - qo) <= 1e-12 * np.linalg.norm(
            pair.o.apply_K(np.abs(X), np.abs(p)))
        if not (pair.ost["n_nonpos_Cw"] or pair.ost["n_nonpos_Dw"]):
            assert rel_l2(q, qo) <= 1e-11


# ------------------------------------------------------------------ a9: PCG protocol
def test_pcg_one_step(pair):
    """One iteration from the same state on both sides: <= 1e-12 on
    every vector.  Runs on every case, indefinite K_w included: one step is one K apply,
    two dot products and axpys.  Definite cases: each side uses its own setup.  Where the
    lumped masses change sign (R9) the Jacobi diagonal sum_(c,a) B^2 X cancels and its
    near-zero entries amplify setup rounding without bound, so there the oracle step takes
    the GPU's X and diag K (both compared on their own in test_lumped_and_jacobi) and the
    bound carries the cancellation factors of <p, K p> and <r, Minv r>."""
    ctx, o, st = pair.ctx, pair.o, pair.ost
    rng = np.random.default_rng(7)
    indef = bool(st["n_nonpos_Cw"] or st["n_nonpos_Dw"])
    if indef:
        Cg, Dg, Cig, Dig, dlg, drg = (empty(n) for n in (ctx.n_nodes,) * 4 + (ctx.n_p,) * 2)
        ctx.get_lumped(Cg, Dg, Cig, Dig)
        ctx.get_jacobi(dlg, drg)
        sides = ((0, host(Cig), host(dlg)), (1, host(Dig), host(drg)))
    else:
        sides = ((0, st["Cinv"], st["diagKl"]), (1, st["Dinv"], st["diagKr"]))
    for side, X, dk in sides:
        x, r, p = (o.project(rng.uniform(-1, 1, o.n_p)) for _ in range(3))
        keep = np.abs(dk) > 1e-13 * np.abs(dk).max()  # DESIGN.md R11 (pseudo-inverse of diag K)
        minv = np.where(keep, 1.0 / np.where(keep, dk, 1.0), 0.0)
        rz = float(r @ (minv * r))
        xg, rg, pg = dev(x), dev(r), dev(p)
        rzg = ctx.debug_pcg_step(side, xg, rg, pg, rz)
        xo, ro, po, rzo = o.pcg_step(X, dk, x, r, p, rz)
        k_rz, k_pq = 1.0, 1.0
        if indef:
            qo = o.apply_K(X, p)
            k_pq = max(1.0, float(np.sum(np.abs(p * qo)) / abs(float(p @ qo))))
            k_rz = max(1.0, float(np.sum(np.abs(ro * minv * ro)) / abs(float(ro @ (minv * ro)))))
        assert rel_l2(host(xg), xo) <= 1e-12 * k_pq
        assert rel_l2(host(rg), ro) <= 1e-12 * k_pq
        assert rel_l2(host(pg), po) <= 1e-12 * max(k_pq, k_rz)
        assert abs(rzg - rzo) <= 1e-12 * max(k_pq, k_rz) * abs(rzo)


@pytest.mark.parametrize("iters", [0, 1, 5, 10, 20])
def test_pcg_prefix(pair, iters):
    ctx, o, st = pair.ctx, pair.o, pair.ost
    if st["n_nonpos_Dw"]:
        pytest.skip("indefinite K_r (C1-like, DESIGN.md R8): one-step parity only")
    b = pair.inp["p"]
    x = host(ctx.poisson_pcg(1, dev(b), empty(ctx.n_p), iters))
    xo = o.poisson(st["Dinv"], st["diagKr"], b, iters)
    if iters == 0:
        assert np.all(x == 0.0) and np.all(xo == 0.0)
        return
    assert rel_l2(x, xo) <= 1e-12


# ------------------------------------------------------------------ a10
def self_discrepancy(o, r, iters, seed=11, zo=None, orders=(1, 2)):
    """delta_self: the oracle against itself with another summation
    order -- reversed element (scatter-add) and dot-product order (1), and dot products
    summed even-then-odd (2) -- the same arithmetic in other rounding orders, i.e. how far
    the fixed-iteration CG amplifies summation-order rounding alone.  The max over the
    orders.  `seed` is unused (kept for call compatibility)."""
    from oracle import Oracle
    ref = o.wbfbt(r, iters) if zo is None else zo
    ds = 0.0
    for order in orders:
        Oracle.set_order(order)
        try:
            zr = o.wbfbt(r, iters)
        finally:
            Oracle.set_order(0)
        ds = max(ds, rel_l2(zr, ref))
    return ds


def test_wbfbt_free_running(pair):
    """Free-running wBFBT at the config's PCG count: rel l2 <= 1e-8, or, where the
    oracle's self-discrepancy delta_self > 1e-9 shows the fixed-iteration CG is that
    sensitive, Poisson residuals agreeing within 2x."""
    ctx, o, st = pair.ctx, pair.o, pair.ost
    iters = pair.cfg.iters
    r = pair.inp["p"]
    z = host(ctx.apply_wbfbt(dev(r), empty(ctx.n_p), iters))
    zo = o.wbfbt(r, iters)
    err = rel_l2(z, zo)
    if st["n_nonpos_Cw"] or st["n_nonpos_Dw"]:
        # indefinite K_w: CG is chaotic from iteration 2; check only
        # finiteness here; one-step parity covers the kernels.
        assert np.all(np.isfinite(z))
        return
    assert abs(z[::o.n_m].sum()) <= 1e-12 * np.linalg.norm(z) * np.sqrt(o.n_el)
    if err <= 1e-8:
        return
    ds = self_discrepancy(o, r, iters, zo=zo)
    print(f"wBFBT {pair.cfg.name} N={pair.N}: err {err:.3e}, oracle delta_self {ds:.3e}")
    assert ds > 1e-9, f"wBFBT rel err {err:.3e}, delta_self {ds:.3e}"
    b = o.project(r)
    xg = host(ctx.poisson_pcg(1, dev(b), empty(ctx.n_p), iters))
    rg = o.poisson_relres(st["Dinv"], b, xg)
    ro = o.poisson_relres(st["Dinv"], b, o.poisson(st["Dinv"], st["diagKr"], b, iters))
    assert rg <= 2 * ro and ro <= 2 * rg


def test_wbfbt_scale_invariance_bit_exact(pair):
    """wBFBT(16 mu) = 16 wBFBT(mu) bit-exactly."""
    from paper_1607_03936_b200 import Context
    ctx = pair.ctx
    r = dev(pair.inp["p"])
    it = min(pair.cfg.iters, 20)
    z1 = host(ctx.apply_wbfbt(r, empty(ctx.n_p), it))
    c2 = Context(pair.N, pair.k)
    c2.set_viscosity(dev(16.0 * pair.inp["mu_q"]))
    z2 = host(c2.apply_wbfbt(r, empty(ctx.n_p), it))
    assert np.array_equal(z2, 16.0 * z1)


def test_determinism(pair):
    ctx = pair.ctx
    r = dev(pair.inp["p"])
    it = pair.cfg.iters
    z1 = host(ctx.apply_wbfbt(r, empty(ctx.n_p), it))
    z2 = host(ctx.apply_wbfbt(r, empty(ctx.n_p), it))
    assert np.array_equal(z1, z2)
    u = dev(pair.inp["u"])
    assert np.array_equal(host(ctx.apply_A(u, empty(ctx.n_v))), host(ctx.apply_A(u, empty(ctx.n_v))))
