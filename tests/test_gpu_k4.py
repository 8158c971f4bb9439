"""The fused k = 3, 4 Poisson kernel (csrc/k4_fused.cuh, rows a8 / a9 at high order; C4 is
Q4 x P3disc) in every tile variant, against the oracle: K_w applies (<= 1e-11, every case,
the indefinite ones with the |X| rounding scale as in test_gpu_parity), PCG prefixes on the
definite meshes (<= 1e-12), and the direction-update modes through one-step parity.  The
meshes are ragged for every tile shape (N = 5, 7, 8 against tiles of 2, 3 and 4 elements).
The default variant is also covered by every k = 3, 4 case of test_gpu_parity / test_gpu_api."""
import numpy as np
import pytest

import synth
from tests.gpu_common import K3, Pair, dev, empty, host, rel_l2

pytestmark = pytest.mark.gpu

CASES = [("C4", 5), ("C4", 8), ("C4", 1), ("K3", 7), ("K3", 3)]


@pytest.fixture(scope="module", params=CASES, ids=lambda c: f"{c[0]}-N{c[1]}")
def pair(request):
    cfg, N = request.param
    return Pair(K3 if cfg == "K3" else cfg, N)


def variants(k):
    return [0, 1, 2, 3, 4, 5, 6, 7, 8, 9] if k == 4 else [0, 1]


def test_k4_fused_apply_K(pair):
    p = pair.inp["p"]
    for var in variants(pair.k):
        pair.ctx.set_option("k4f", 1)
        pair.ctx.set_option("k4_var", var)
        for side, X in ((0, pair.ost["Cinv"]), (1, pair.ost["Dinv"])):
            q = host(pair.ctx.apply_K(side, dev(p), empty(pair.ctx.n_p)))
            qo = pair.o.apply_K(X, p)
            scale = np.linalg.norm(pair.o.apply_K(np.abs(X), np.abs(p)))
            assert rel_l2(q, qo) <= 1e-11 or np.linalg.norm(q - qo) <= 1e-12 * scale, (var, side)


def test_k4_fused_matches_unfused(pair):
    """The fused kernel and the B^T / gather / B kernels (option k4f 0) compute the same
    K_w: rounding-level agreement on the same input."""
    p = dev(pair.inp["p"])
    pair.ctx.set_option("k4f", 0)
    q0 = host(pair.ctx.apply_K(1, p, empty(pair.ctx.n_p)))
    for var in variants(pair.k):
        pair.ctx.set_option("k4f", 1)
        pair.ctx.set_option("k4_var", var)
        q1 = host(pair.ctx.apply_K(1, p, empty(pair.ctx.n_p)))
        assert rel_l2(q1, q0) <= 1e-12 or pair.ost["n_nonpos_Dw"], var


@pytest.mark.parametrize("iters", [1, 5, 10])
def test_k4_fused_pcg_prefix(pair, iters):
    if pair.ost["n_nonpos_Dw"]:
        pytest.skip("indefinite K_r (DESIGN.md R9): apply parity only")
    b = pair.inp["p"]
    xo = pair.o.poisson(pair.ost["Dinv"], pair.ost["diagKr"], b, iters)
    for var in variants(pair.k):
        pair.ctx.set_option("k4f", 1)
        pair.ctx.set_option("k4_var", var)
        x = host(pair.ctx.poisson_pcg(1, dev(b), empty(pair.ctx.n_p), iters))
        assert rel_l2(x, xo) <= 1e-12, var


def test_k4_fused_bitwise_repeat():
    """Fixed-order sums only: two runs of the default variant agree bit for bit."""
    pr = Pair("C4", 8)
    b = dev(pr.inp["p"])
    x1 = host(pr.ctx.poisson_pcg(1, b, empty(pr.ctx.n_p), 20))
    x2 = host(pr.ctx.poisson_pcg(1, b, empty(pr.ctx.n_p), 20))
    assert np.array_equal(x1, x2)


def test_k4_fused_full_c4_prefix():
    """Full C4 (24^3, Q4 x P3disc): PCG prefix <= 1e-12 at 5 and 10 iterations (default
    variant) and the wBFBT apply through the fused kernel against the oracle (prefix regime,
    10 iterations per Poisson solve)."""
    pr = Pair("C4")
    b = pr.inp["p"]
    for iters in (5, 10):
        x = host(pr.ctx.poisson_pcg(1, dev(b), empty(pr.ctx.n_p), iters))
        assert rel_l2(x, pr.o.poisson(pr.ost["Dinv"], pr.ost["diagKr"], b, iters)) <= 1e-12, iters
    z = host(pr.ctx.apply_wbfbt(dev(b), empty(pr.ctx.n_p), 10))
    assert rel_l2(z, pr.o.wbfbt(b, 10)) <= 1e-10
    assert synth.CONFIGS["C4"].N == 24


@pytest.mark.parametrize("opt", [0, 1, 2])
def test_k4_tile_B_BT(pair, opt):
    """Standalone B and B^T at high order through each path (option k4bt: 0 element kernels
    + gather, 1 the B^T tile kernel, 2 the B^T and B tile kernels) against the oracle,
    masked and X-scaled forms (<= 1e-11; boundary rows exactly 0)."""
    ctx, o = pair.ctx, pair.o
    ctx.set_option("k4bt", opt)
    u, p = pair.inp["u"], pair.inp["p"]
    y = host(ctx.apply_BT(dev(p), empty(ctx.n_v)))
    assert rel_l2(y, o.apply_BT(p)) <= 1e-11
    assert np.all(y[o.boundary_mask().astype(bool)] == 0.0)
    q = host(ctx.apply_B(dev(u), empty(ctx.n_p)))
    assert rel_l2(q, o.apply_B(u)) <= 1e-11
    ctx.set_option("k4bt", 1)
