"""k = 2 B and B^T by z-marching columns (csrc/k2_zc.cuh, option bbt_zc = 2, 4, 8 element
layers per chunk; the default on N >= 48 meshes, so the full-size C5 tests of test_gpu_api /
test_gpu_parity run it too) against the oracle (rows a6, a7: <= 1e-11, boundary rows exactly 0), on
ragged and chunk-ragged meshes, and inside wBFBT (the X-scaled forms) against the default
tile / box kernels."""
import numpy as np
import pytest

from tests.gpu_common import Pair, dev, empty, host, rel_l2

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", params=[("C1", None), ("C2", 7), ("C2", None), ("C3", None), ("C1", 1)],
                ids=lambda c: f"{c[0]}-N{c[1]}")
def pair(request):
    return Pair(request.param[0], request.param[1])


@pytest.mark.parametrize("cz", [2, 4, 8])
def test_zc_B_BT(pair, cz):
    ctx, o = pair.ctx, pair.o
    ctx.set_option("bbt_zc", cz)
    try:
        u, p = pair.inp["u"], pair.inp["p"]
        y = host(ctx.apply_BT(dev(p), empty(ctx.n_v)))
        assert rel_l2(y, o.apply_BT(p)) <= 1e-11
        assert np.all(y[o.boundary_mask().astype(bool)] == 0.0)
        q = host(ctx.apply_B(dev(u), empty(ctx.n_p)))
        assert rel_l2(q, o.apply_B(u)) <= 1e-11
    finally:
        ctx.set_option("bbt_zc", -1)


def test_zc_in_wbfbt(pair):
    """wBFBT (B^T with D_w^-1, B with C_w^-1) with 5 PCG iterations per inner solve: the
    z-march kernels agree with the tile / box kernels to rounding."""
    ctx = pair.ctx
    r = dev(pair.inp["p"])
    try:
        ctx.set_option("bbt_zc", 0)
        z0 = host(ctx.apply_wbfbt(r, empty(ctx.n_p), 5))
        ctx.set_option("bbt_zc", 4)
        z1 = host(ctx.apply_wbfbt(r, empty(ctx.n_p), 5))
    finally:
        ctx.set_option("bbt_zc", -1)
    tol = 1e-9 if (pair.ost["n_nonpos_Cw"] or pair.ost["n_nonpos_Dw"]) else 1e-12
    assert rel_l2(z1, z0) <= tol


def test_k2_pair_bitwise():
    """Option k2_pair (the TMA Poisson kernel with paired class-(0,*) / (1,*) pencils, same
    per-row arithmetic): PCG results bitwise equal to the default kernel, on a ragged mesh
    (N = 18: not a multiple of the 4 x 8 x 8 tile; C2's recipe is definite from N = 16 on, R9, so
    the 12-iteration prefix also matches the oracle)."""
    pr = Pair("C2", 18)
    b = dev(pr.inp["p"])
    x0 = host(pr.ctx.poisson_pcg(1, b, empty(pr.ctx.n_p), 12))
    pr.ctx.set_option("k2_pair", 1)
    x1 = host(pr.ctx.poisson_pcg(1, b, empty(pr.ctx.n_p), 12))
    pr.ctx.set_option("k2_pair", 0)
    assert np.array_equal(x0, x1)
    assert rel_l2(x1, pr.o.poisson(pr.ost["Dinv"], pr.ost["diagKr"], pr.inp["p"], 12)) <= 1e-12
