"""Property tests of the GPU path on random lattices and exponents (hypothesis)."""
import numpy as np
import pytest
from hypothesis import HealthCheck, given, settings
from hypothesis import strategies as st

from conftest import emetric
from oracle import oracle as O
from paper_2504_11989_b200 import Lattice
from paper_2504_11989_b200.epstein import EpsteinContext
from paper_2504_11989_b200.quadrature import QuadratureConfig, integrate_product

pytestmark = pytest.mark.gpu
# derandomize: the same examples on every run (reproducible round-end runs; widen by hand with
# --hypothesis-seed when exploring)
SETTINGS = settings(max_examples=25, deadline=None, derandomize=True, suppress_health_check=list(HealthCheck))


@st.composite
def lattices(draw, dims=(2, 3)):
    d = draw(st.sampled_from(dims))
    a = np.eye(d) + np.array(draw(st.lists(st.floats(-0.3, 0.3), min_size=d * d, max_size=d * d))).reshape(d, d)
    a *= draw(st.floats(0.7, 1.5))
    return Lattice(a)


exponents = st.floats(0.6, 9.0).filter(lambda v: min(abs(v - round(v)), 1.0) > 1e-3 or v == round(v))


@SETTINGS
@given(lat=lattices(), nu=exponents, seed=st.integers(0, 2 ** 31 - 1))
def test_even_periodic_decomposed(lat, nu, seed):
    ctx = EpsteinContext(lat, nu, device=0)
    if ctx.branch == "trivial":
        return
    rng = np.random.default_rng(seed)
    k = rng.uniform(-0.45, 0.45, size=(16, lat.d)) @ lat.a_inv_t.T
    z = ctx.zeta(k)
    scale = max(1.0, float(np.abs(z).max()))
    assert np.abs(ctx.zeta(-k) - z).max() <= 1e-12 * scale
    shift = rng.integers(-2, 3, size=lat.d) @ lat.a_inv_t.T
    assert np.abs(ctx.zeta(k + shift) - z).max() <= 1e-11 * scale
    assert np.abs(ctx.reg_zeta(k) + ctx.singular(k) / ctx.vol - z).max() <= 1e-12 * scale
    assert emetric(z, O.zeta(lat.a, nu, k)).max() <= 1e-12 * scale


@SETTINGS
@given(lat=lattices(), nu=exponents, s=st.floats(0.5, 2.0), seed=st.integers(0, 2 ** 31 - 1))
def test_lattice_scaling(lat, nu, s, seed):
    """Z_{s Lambda, nu}(k / s) = s^-nu Z_{Lambda, nu}(k)."""
    ctx = EpsteinContext(lat, nu, device=0)
    if ctx.branch == "trivial":
        return
    k = np.random.default_rng(seed).uniform(-0.45, 0.45, size=(8, lat.d)) @ lat.a_inv_t.T
    z1 = ctx.zeta(k)
    z2 = EpsteinContext(lat.scaled(s), nu, device=0).zeta(k / s)
    assert emetric(z2, s ** -nu * z1).max() <= 1e-11 * max(1.0, float(np.abs(z1).max()))


@SETTINGS
@given(lat=lattices((3,)), t=st.floats(0.3, 2.0), seed=st.integers(0, 2 ** 31 - 1))
def test_hessian_trace_identity_any_split(lat, t, seed):
    """tr(-Hess Z_5 / 4 pi^2) = Z_3 for any theta split."""
    tt = t * lat.volume ** (-2.0 / 3.0)
    k = np.random.default_rng(seed).uniform(-0.45, 0.45, size=(8, 3)) @ lat.a_inv_t.T
    M = EpsteinContext(lat, 5.0, splitting=tt, device=0).polynomial_weighted(k)
    z3 = EpsteinContext(lat, 3.0, device=0).zeta(k)
    assert emetric(np.trace(M, axis1=1, axis2=2), z3).max() <= 1e-11 * max(1.0, float(np.abs(z3).max()))


@settings(max_examples=6, deadline=None, derandomize=True, suppress_health_check=list(HealthCheck))
@given(lat=lattices((2,)), nus=st.lists(st.floats(2.3, 6.0), min_size=3, max_size=3))
def test_exponent_permutation_symmetry(lat, nus):
    """zeta^(3) is invariant under cyclic shifts and reversal of the exponent vector."""
    cfg = QuadratureConfig(grid_u=64, grid_v=64, estimate_error=False)
    v = integrate_product(lat, nus, cfg)[0]
    for perm in ([nus[1], nus[2], nus[0]], nus[::-1]):
        w = integrate_product(lat, perm, cfg)[0]
        assert abs(w - v) <= 1e-12 * abs(v)


@settings(max_examples=12, deadline=None, derandomize=True, suppress_health_check=list(HealthCheck))
@given(lat=lattices(), nu=st.floats(2.5, 8.0), order=st.integers(1, 4), seed=st.integers(0, 2 ** 31 - 1))
def test_derivative_parity_and_periodicity(lat, nu, order, seed):
    """d^alpha Z(-k) = (-1)^|alpha| d^alpha Z(k) and d^alpha Z(k + G) = d^alpha Z(k)."""
    ctx = EpsteinContext(lat, nu, device=0)
    if ctx.branch == "trivial":
        return
    rng = np.random.default_rng(seed)
    k = rng.uniform(-0.45, 0.45, size=(8, lat.d)) @ lat.a_inv_t.T
    k = k[np.linalg.norm(k, axis=1) > 0.05]
    _, D = ctx.derivatives(k, order)
    _, Dm = ctx.derivatives(-k, order)
    scale = max(1.0, float(np.abs(D).max()))
    assert np.abs(Dm - (-1) ** order * D).max() <= 1e-11 * scale
    shift = rng.integers(-2, 3, size=lat.d) @ lat.a_inv_t.T
    _, Ds = ctx.derivatives(k + shift, order)
    assert np.abs(Ds - D).max() <= 1e-10 * scale
