"""GPU parity of the batched zeta / Hessian kernels through the C ABI (needs a B200)."""
import math

import numpy as np
import pytest

from conftest import emetric
from oracle import oracle as O
from paper_2504_11989_b200 import PoleError, named_lattice
from paper_2504_11989_b200 import _native as N
from paper_2504_11989_b200.epstein import EpsteinContext, epstein_context, polynomial_weighted_zeta

pytestmark = pytest.mark.gpu
ZETA_TOL = 1e-12  # BASELINE north_star: <= 1e-12 per zeta value (E = min(abs, rel))


def _ctx(name, nu):
    return EpsteinContext(named_lattice(name), nu, device=0)


def test_native_library_is_loaded():
    assert N.device_count() >= 1
    assert "sm_100a" in N.lib().lz_version().decode()


def test_c1_parity_all_points(golden):
    """Config 1: Z^2, nu = 3.5, 4096 seeded k; every point vs the reference (golden)."""
    sq = named_lattice("square")
    k = np.random.default_rng(0).uniform(-0.5, 0.5, size=(4096, 2))
    z = _ctx("square", 3.5).zeta(k)
    e = emetric(z, golden["c1"]["zeta"])
    assert e.max() <= ZETA_TOL, e.max()
    assert abs(math.fsum(z) - golden["c1"]["zeta_fsum"]) <= 1e-10 * abs(golden["c1"]["zeta_fsum"])
    # and vs the long-double oracle
    assert emetric(z, O.zeta(sq.a, 3.5, k)).max() <= ZETA_TOL


@pytest.mark.parametrize("idx", range(29))
def test_zeta_cases_vs_reference(golden, idx):
    c = golden["cases"][idx]
    lat = named_lattice(c["lattice"])
    ctx = EpsteinContext(lat, c["nu"], device=0)
    k = np.array(c["k"]).reshape(-1, lat.d)
    z = ctx.zeta(k)
    assert emetric(z, c["zeta"]).max() <= ZETA_TOL
    inside = np.ones(len(k), bool)
    inside[3] = False  # reg_zeta: k must lie in the BZ closure
    zr = ctx.reg_zeta(k)
    assert emetric(zr[inside], np.array(c["reg_zeta"])[inside]).max() <= ZETA_TOL
    # (index 3 lies outside the BZ: reg_zeta there is out of contract -- the q = 0 series of
    #  L/epstein.py:250-259 cancels catastrophically for |k|^2 >> 1 in every implementation)
    if c["branch"] != "trivial":
        if c.get("zeta_at_zero") == "pole":
            with pytest.raises(PoleError):
                ctx.zeta_at_zero()
        else:
            assert emetric(ctx.zeta_at_zero(), c["zeta_at_zero"]) <= ZETA_TOL


def test_scalar_and_shapes():
    ctx = _ctx("square", 3.5)
    k = np.array([0.1, 0.2])
    v = ctx.zeta(k)
    assert isinstance(v, float)
    assert ctx.zeta(np.zeros((0, 2))).shape == (0,)
    kk = np.random.default_rng(5).uniform(-0.5, 0.5, size=(3, 7, 2))
    out = ctx.zeta(kk)
    assert out.shape == (3, 7)
    assert np.array_equal(out.ravel(), ctx.zeta(kk.reshape(-1, 2)))
    with pytest.raises(ValueError):
        ctx.zeta(np.array([[np.nan, 0.0]]))


@pytest.mark.parametrize("n", [1, 2, 31, 32, 33, 1000, 4097])
def test_ragged_batches_bitwise(n):
    """Batch size and lane split never change a point's value beyond rounding."""
    ctx = _ctx("fcc", 3.0)
    lat = named_lattice("fcc")
    k = np.random.default_rng(n).uniform(-0.5, 0.5, size=(n, 3)) @ lat.a_inv_t.T
    z = ctx.zeta(k)
    zo = O.zeta(lat.a, 3.0, k)
    assert emetric(z, zo).max() <= ZETA_TOL


def test_lanes_per_point_agree():
    import torch
    ctx = _ctx("bcc", 5.0)
    lat = named_lattice("bcc")
    k = np.random.default_rng(3).uniform(-0.5, 0.5, size=(777, 3)) @ lat.a_inv_t.T
    kt = torch.tensor(k, device="cuda")
    outs = []
    for lanes in (1, 2, 8, 32):
        z, st = ctx.zeta_device(kt, lanes_per_point=lanes)
        torch.cuda.synchronize()
        assert int(st.item()) == 0
        outs.append(z.cpu().numpy())
    for o in outs[1:]:
        assert emetric(o, outs[0]).max() <= 1e-13  # summation order only


def test_pole_and_singular_semantics():
    c2 = _ctx("square", 2.0)
    with pytest.raises(PoleError):
        c2.zeta(np.zeros(2))
    with pytest.raises(PoleError):
        c2.zeta(np.array([[1.0, -1.0]]))  # reduces to k = 0
    # log-case singular part undefined at 0; generic nu < d diverges at 0
    with pytest.raises(ValueError):
        c2.singular(np.zeros(2))
    with pytest.raises(ValueError):
        _ctx("square", 1.5).singular(np.zeros(2))
    c = _ctx("square", 3.5)
    k = np.array([[0.13, -0.21], [0.3, 0.4]])
    rho = np.sum(k * k, axis=1)
    assert np.allclose(c.singular(k), c.singular_coef() * rho ** 0.75, rtol=1e-14)
    assert emetric(c.zeta(k), c.reg_zeta(k) + c.singular(k) / c.vol).max() <= 1e-14
    # trivial branch: constant -1 at nu = 0, 0 at nu = -2
    assert _ctx("square", 0.0).zeta(np.array([0.2, 0.1])) == -1.0
    assert _ctx("square", -2.0).zeta(np.array([0.2, 0.1])) == 0.0


def test_size_independent_properties_2pow20():
    """Throughput-sized batch: evenness, periodicity and BZ reduction (no oracle needed)."""
    ctx = _ctx("square", 3.5)
    k = np.random.default_rng(1).uniform(-0.5, 0.5, size=(1 << 20, 2))
    z = ctx.zeta(k)
    assert np.all(np.isfinite(z))
    zm = ctx.zeta(-k)
    assert np.abs(z - zm).max() <= 1e-13 * max(1.0, np.abs(z).max())
    shift = np.array([3.0, -2.0])
    zs = ctx.zeta(k[:65536] + shift)
    assert emetric(zs, z[:65536]).max() <= 1e-12
    # sub-sample against the oracle
    idx = np.random.default_rng(2).choice(len(k), 2048, replace=False)
    assert emetric(z[idx], O.zeta(np.eye(2), 3.5, k[idx])).max() <= ZETA_TOL


@pytest.mark.parametrize("name", ["fcc", "bcc", "square", "integer_1d", "hexagonal"])
def test_hessian_vs_oracle_and_trace_identity(name):
    lat = named_lattice(name)
    d = lat.d
    rng = np.random.default_rng(11)
    kap = rng.uniform(-0.5, 0.5, size=(64, d))
    k = kap @ lat.a_inv_t.T
    ctx5 = EpsteinContext(lat, 5.0, device=0)
    H = ctx5.zeta_hessian(k)
    Ho = O.hessian(lat.a, 5.0, k)
    scale = np.abs(Ho).max(axis=(1, 2), keepdims=True)
    assert (np.abs(H - Ho) / np.maximum(scale, 1.0)).max() <= ZETA_TOL
    # tr M_5 = Z_3 exactly (Laplacian of the lattice sum)
    M = polynomial_weighted_zeta(lat, 5.0, k)
    z3 = epstein_context(lat, 3.0).zeta(k)
    assert emetric(np.trace(M, axis1=1, axis2=2), z3).max() <= 1e-12 * max(1.0, np.abs(z3).max())


def test_hessian_vs_reference_fd(golden):
    for h in golden["hessian_fd"]:
        lat = named_lattice(h["lattice"])
        M = polynomial_weighted_zeta(lat, 5.0, np.array(h["k"]))
        assert abs(np.trace(M) - h["z3"]) <= 1e-12 * max(1.0, abs(h["z3"]))
        assert np.abs(M - np.array(h["M_fd"]).reshape(3, 3)).max() < 1e-4


@pytest.mark.parametrize("scale", [0.35, 0.5, 0.65, 1.0, 1.6])
def test_split_invariance(scale):
    """Z and its Hessian do not depend on the theta split (the fused ATM plan uses a tuned one)."""
    fcc = named_lattice("fcc")
    t = scale * fcc.volume ** (-2.0 / 3.0)
    kap = np.random.default_rng(7).uniform(-0.5, 0.5, size=(256, 3))
    k = kap @ fcc.a_inv_t.T
    z = EpsteinContext(fcc, 3.0, splitting=t, device=0).zeta(k)
    assert emetric(z, O.zeta(fcc.a, 3.0, k)).max() <= ZETA_TOL
    H = EpsteinContext(fcc, 5.0, splitting=t, device=0).zeta_hessian(k)
    Ho = O.hessian(fcc.a, 5.0, k)
    scale_h = np.maximum(np.abs(Ho).max(axis=(1, 2), keepdims=True), 1.0)
    assert (np.abs(H - Ho) / scale_h).max() <= ZETA_TOL


@pytest.mark.parametrize("nu", [5.0, 6.0, 4.5, 2.5])
def test_four_dimensional_lattice(nu):
    """d = 4 (L/lattice.py:20 upper limit): batch zeta and Hessian vs the oracle."""
    from paper_2504_11989_b200 import Lattice
    a = np.array([[1.0, 0.2, 0.0, 0.1], [0.0, 1.1, 0.3, 0.0], [0.0, 0.0, 0.9, 0.2], [0.1, 0.0, 0.0, 1.0]])
    lat = Lattice(a)
    kap = np.random.default_rng(3).uniform(-0.5, 0.5, size=(64, 4))
    k = kap @ lat.a_inv_t.T
    ctx = EpsteinContext(lat, nu, device=0)
    assert emetric(ctx.zeta(k), O.zeta(lat.a, nu, k)).max() <= ZETA_TOL
    H = ctx.zeta_hessian(k)
    Ho = O.hessian(lat.a, nu, k)
    sc = np.maximum(np.abs(Ho).max(axis=(1, 2), keepdims=True), 1.0)
    assert (np.abs(H - Ho) / sc).max() <= ZETA_TOL


@pytest.mark.parametrize("name,nu", [("fcc", 3.0), ("fcc", 5.0), ("bcc", 6.5), ("square", 3.5),
                                     ("hexagonal", 4.0), ("integer_1d", 2.5)])
@pytest.mark.parametrize("order", [1, 2, 3, 4])
def test_general_derivatives_vs_oracle(name, nu, order):
    """d^alpha Z(k), |alpha| = 1..4, at random k in the cell vs the long-double oracle (the
    polynomial-weighted zeta of SURVEY 8(f) item 2), scaled per point like the Hessian test."""
    lat = named_lattice(name)
    d = lat.d
    kap = np.random.default_rng(order * 7 + d).uniform(-0.45, 0.45, size=(48, d))
    k = kap @ lat.a_inv_t.T
    ctx = EpsteinContext(lat, nu, device=0)
    alphas, D = ctx.derivatives(k, order)
    assert alphas == O.multi_indices(d, order)
    Do, Sabs = O.derivatives(lat.a, nu, order, k, with_abs=True)
    scale = np.maximum(np.abs(Do).max(axis=1, keepdims=True), 1.0)
    # 1e-12 of the point's scale plus the rounding floor of the method (16 eps x sum |terms|,
    # the same bound as the high orders below)
    bound = ZETA_TOL * scale + 16 * np.finfo(float).eps * Sabs
    assert (np.abs(D - Do) <= bound).all(), (np.abs(D - Do) / bound).max()
    if order == 2 and d > 1:
        H = ctx.zeta_hessian(k)
        for j, a in enumerate(alphas):
            i0, i1 = [i for i, v in enumerate(a) for _ in range(v)]
            assert np.abs(D[:, j] - H[:, i0, i1]).max() <= 1e-11 * scale.max()


def test_derivative_laplacian_identity_and_poly_weights():
    """sum_a d_a d_a d_b Z_5 = -4 pi^2 d_b Z_3 (third order from the Laplacian identity), and the
    general polynomial-weighted zeta reduces to M_ab for |alpha| = 2."""
    fcc = named_lattice("fcc")
    kap = np.random.default_rng(5).uniform(-0.45, 0.45, size=(64, 3))
    k = kap @ fcc.a_inv_t.T
    al3, D3 = EpsteinContext(fcc, 5.0, device=0).derivatives(k, 3)
    al1, D1 = EpsteinContext(fcc, 3.0, device=0).derivatives(k, 1)
    for b in range(3):
        lap = sum(D3[:, al3.index(tuple(2 * (i == a) + (i == b) for i in range(3)))] for a in range(3))
        ref = -4.0 * math.pi ** 2 * D1[:, al1.index(tuple(int(i == b) for i in range(3)))]
        assert np.abs(lap - ref).max() <= 1e-11 * max(1.0, np.abs(ref).max())
    M = polynomial_weighted_zeta(fcc, 5.0, k)
    M01 = polynomial_weighted_zeta(fcc, 5.0, k, alpha=(1, 1, 0))
    assert np.abs(M01.imag).max() == 0.0
    assert np.abs(M01.real - M[:, 0, 1]).max() <= 1e-11 * max(1.0, np.abs(M).max())
    with pytest.raises(PoleError):
        EpsteinContext(fcc, 5.0, device=0).derivatives(np.zeros(3), 2)


# --------------------------------------------------------------------------------------------
# Any order <= 12, any d <= 4: the moment form of the derivative kernel (deriv.cu)

LAT4 = [[1.0, 0.2, 0.0, 0.1], [0.0, 1.1, 0.3, 0.0], [0.0, 0.0, 0.9, 0.2], [0.1, 0.0, 0.0, 1.0]]


def _lat(name):
    from paper_2504_11989_b200 import Lattice
    return Lattice(np.array(LAT4)) if name == "lat4" else named_lattice(name)


@pytest.mark.gpu
@pytest.mark.parametrize("name,nu,order,npts", [
    ("square", 3.5, 5, 32), ("square", 3.5, 8, 32), ("square", 4.0, 12, 24), ("hexagonal", 4.5, 10, 24),
    ("integer_1d", 2.5, 12, 32), ("fcc", 5.0, 6, 16), ("fcc", 3.0, 8, 12), ("bcc", 6.5, 12, 8),
    ("lat4", 6.0, 1, 16), ("lat4", 5.0, 2, 16), ("lat4", 6.5, 4, 12), ("lat4", 7.0, 6, 6)])
def test_high_order_derivatives_vs_oracle(name, nu, order, npts):
    """d^alpha Z(k) for orders 5..12 and d = 4 (the reference's limits, L/epstein.py:347-353 and
    L/lattice.py:20) at random k in the cell vs the long-double oracle.

    High-order Ewald derivatives cancel: the direct and reciprocal terms grow like
    (2 pi m / e)^{m/2} while the value does not, so no double-precision evaluation (the reference's
    fsum tables included) gets below eps x sum|terms|.  The bound is therefore 1e-12 of the point's
    largest derivative plus 16 eps of the oracle's sum of |terms| for that value."""
    lat = _lat(name)
    d = lat.d
    kap = np.random.default_rng(order * 11 + d).uniform(-0.45, 0.45, size=(npts, d))
    k = kap @ lat.a_inv_t.T
    alphas, D = EpsteinContext(lat, nu, device=0).derivatives(k, order)
    assert alphas == O.multi_indices(d, order)
    Do, Sabs = O.derivatives(lat.a, nu, order, k, with_abs=True)
    scale = np.maximum(np.abs(Do).max(axis=1, keepdims=True), 1.0)
    bound = ZETA_TOL * scale + 16 * np.finfo(float).eps * Sabs
    assert (np.abs(D - Do) <= bound).all(), (np.abs(D - Do) / bound).max()


@pytest.mark.gpu
def test_high_order_laplacian_identity():
    """sum_a d_a^2 d^beta Z_5 = -4 pi^2 d^beta Z_3 for every |beta| = 6 (order 8 of nu = 5 against
    order 6 of nu = 3): ties the high orders together without the oracle."""
    fcc = named_lattice("fcc")
    k = np.random.default_rng(9).uniform(-0.4, 0.4, size=(24, 3)) @ fcc.a_inv_t.T
    al8, D8 = EpsteinContext(fcc, 5.0, device=0).derivatives(k, 8)
    al6, D6 = EpsteinContext(fcc, 3.0, device=0).derivatives(k, 6)
    scale = max(1.0, np.abs(D8).max())
    for j, beta in enumerate(al6):
        lap = sum(D8[:, al8.index(tuple(beta[i] + 2 * (i == a) for i in range(3)))] for a in range(3))
        assert np.abs(lap + 4.0 * math.pi ** 2 * D6[:, j]).max() <= 1e-12 * scale, beta


@pytest.mark.gpu
def test_device_taylor_tables_vs_reference_and_host(golden):
    """EpsteinContext.reg_derivatives builds the k = 0 tables on the device (moment kernel in Taylor
    mode): vs the reference's fsum tables (orders up to 12, d up to 4) at 1e-10 of each order's
    scale, and vs the host long-double restatement."""
    import json
    import os
    from test_host import taylor_scales
    from paper_2504_11989_b200.taylor import build_reg_derivatives_host
    with open(os.path.join(os.path.dirname(__file__), "golden", "golden_taylor.json")) as f:
        cases = list(golden["taylor"]) + json.load(f)["taylor"]
    for t in cases:
        ctx = EpsteinContext(_lat(t["lattice"]), t["nu"], device=0)
        tab = ctx.reg_derivatives(t["order"])
        host = build_reg_derivatives_host(ctx, t["order"])
        sc = taylor_scales(t["derivs"])
        assert len(tab.derivs) == len(t["derivs"])
        for alpha, ref in t["derivs"]:
            got = tab.derivs[tuple(alpha)]
            s = sc[sum(alpha)]
            assert abs(got - ref) <= 1e-10 * s, (t["lattice"], t["nu"], alpha, got, ref)
            assert abs(got - host.derivs[tuple(alpha)]) <= 1e-12 * s, (t["lattice"], t["nu"], alpha)
