"""Host-side logic of the drop-in (CPU only): C-ABI exports, lattice geometry, exponent
classification, the native context/table builder vs the reference's point sets, configs,
Duffy layout and the phase-scan arithmetic."""
import ctypes as C
import math
import os
import re

import numpy as np
import pytest

from paper_2504_11989_b200 import LatticeError, Lattice, named_lattice, parse_lattice_spec
from paper_2504_11989_b200 import _native as N
from paper_2504_11989_b200.epstein import EpsteinContext, classify_exponent
from paper_2504_11989_b200.quadrature import (QuadratureConfig, angular_nodes, duffy_cells,
                                              tail_primitive)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_cabi_exports_every_declared_symbol():
    hdr = open(os.path.join(ROOT, "include", "latsum_b200.h")).read()
    declared = set(re.findall(r"^\s*(?:int|double|const char\*)\s+(lz_\w+)\s*\(", hdr, re.M))
    assert len(declared) >= 20
    L = N.lib()
    for name in declared:
        assert hasattr(L, name), name
    assert declared == set(N.SIGNATURES), declared ^ set(N.SIGNATURES)
    assert "sm_100a" in L.lz_version().decode()


def test_lattice_geometry():
    assert named_lattice("sq").volume == 1.0
    assert abs(named_lattice("hex").volume - math.sqrt(3) / 2) < 1e-15
    assert abs(named_lattice("fcc").volume - 1 / math.sqrt(2)) < 1e-15
    for name in ("fcc", "bcc"):
        assert abs(named_lattice(name).min_distance() - 1.0) < 1e-12
    lat = named_lattice("hex", 2.5)
    assert abs(lat.volume - 2.5 ** 2 * math.sqrt(3) / 2) < 1e-13
    r = Lattice(np.diag([2.0, 1.0])).reciprocal()
    assert np.allclose(r.a, np.diag([0.5, 1.0]))
    assert np.allclose(named_lattice("hex").reciprocal().reciprocal().a, named_lattice("hex").a, atol=1e-14)
    assert abs(named_lattice("bcc").brillouin_zone().volume * named_lattice("bcc").volume - 1) < 1e-14
    assert parse_lattice_spec("hex:2.5") == lat
    assert parse_lattice_spec("d=2;A=1,0;0,1") == named_lattice("square")
    for bad in ("d=2;A=1,0", "nope", "d=x;A=1", "hex:abc"):
        with pytest.raises(LatticeError):
            parse_lattice_spec(bad)
    with pytest.raises(LatticeError):
        Lattice([[1.0, 2.0], [2.0, 4.0]])
    with pytest.raises(LatticeError):
        Lattice(np.eye(5))
    with pytest.raises(LatticeError):
        named_lattice("sq", -1.0)


def test_bz_reduce_half_open():
    bz = named_lattice("square").brillouin_zone()
    k = np.array([[0.5, -0.5], [1.25, 0.75], [-0.5, 0.49]])
    red = bz.reduce(k)
    assert np.allclose(red, [[-0.5, -0.5], [0.25, -0.25], [-0.5, 0.49]])
    assert bz.contains(red[0])


def test_classify_exponent(golden):
    for c in golden["cases"]:
        d = named_lattice(c["lattice"]).d
        branch, nu, m = classify_exponent(c["nu"], d)
        assert branch == c["branch"]
        assert nu == c["nu"]
        assert m == c["log_m"]
    assert classify_exponent(3.0 + 1e-13, 3)[0] == "log_case"
    with pytest.raises(ValueError):
        classify_exponent(101.0, 2)
    with pytest.raises(ValueError):
        classify_exponent(float("nan"), 2)


@pytest.mark.parametrize("idx", range(29))
def test_native_context_matches_reference(golden, idx):
    """Constants, point counts and (d <= 2) the exact point sets in the reference's order."""
    c = golden["cases"][idx]
    lat = named_lattice(c["lattice"])
    ctx = EpsteinContext(lat, c["nu"], device=-1)
    assert ctx.branch == c["branch"]
    if ctx.branch == "trivial":
        assert ctx.const_value == c["const_value"]
        return
    for key in ("s_rec", "pref", "rfac", "bconst", "kmax", "split", "vol"):
        assert abs(getattr(ctx, key) - c[key]) <= 2e-15 * abs(c[key]), key
    assert abs(ctx.singular_coef() - c["singular_coef"]) <= 2e-15 * abs(c["singular_coef"])
    assert (len(ctx.dir_w), len(ctx.rec_pts)) == (c["n_dir"], c["n_rec"])
    assert abs(math.fsum(ctx.dir_w) - c["dir_w_fsum"]) <= 1e-14 * abs(c["dir_w_fsum"])
    assert abs(math.fsum(ctx.rec_norm2) - c["rec_norm2_fsum"]) <= 1e-13 * c["rec_norm2_fsum"]
    if "dir_pts" in c:
        assert np.abs(ctx.dir_pts - np.array(c["dir_pts"]).reshape(-1, lat.d)).max() <= 1e-15
        assert np.abs(ctx.rec_pts - np.array(c["rec_pts"]).reshape(-1, lat.d)).max() <= 2e-15
        w = np.array(c["dir_w"])
        assert np.abs(ctx.dir_w - w).max() <= 1e-13 * np.abs(w).max()  # reference Gamma(s<0) recurrence
    # reciprocal-summand tables: Chebyshev-fitted pieces within 6e-16 relative of long double
    stats = ctx.table_stats(hessian=True)
    assert stats.table_max_rel_err < 6e-16
    assert stats.table_x_hi > 35.0  # terms below 1e-18 of the unit scale are dropped


def test_hessian_point_sets():
    for name, nu, hd, hr in (("fcc", 5.0, 171, 1330), ("bcc", 5.0, 364, 2196)):
        info = EpsteinContext(named_lattice(name), nu, device=-1).table_stats(hessian=True)
        assert (info.n_dir_h, info.n_rec_h) == (hd, hr)


def test_no_cpu_fallback():
    ctx = EpsteinContext(named_lattice("square"), 3.5, device=-1)
    with pytest.raises(RuntimeError):
        ctx.zeta(np.array([[0.1, 0.2]]))


def test_quadrature_config_roundtrip():
    cfg = QuadratureConfig(gauss_order=10, epsilon=0.05, grid_u=96, grading=3, splitting=1.25)
    assert QuadratureConfig.from_text(cfg.to_text()) == cfg
    with pytest.raises(ValueError):
        QuadratureConfig(epsilon=0.6)
    with pytest.raises(ValueError):
        QuadratureConfig(taylor_order=3)
    with pytest.raises(ValueError):
        QuadratureConfig.from_text("bogus=1")


def test_duffy_layout():
    for d in (1, 2, 3):
        cells = duffy_cells(d)
        assert len(cells) == 2 ** (d - 1) * d
        v, w = angular_nodes(d, 14)
        assert abs(w.sum() - 0.5 ** (d - 1)) < 1e-15
    assert duffy_cells(3)[1].pyramid == 1 and duffy_cells(3)[3].signs == (1.0, -1.0)


def test_tail_primitive_examples():
    assert tail_primitive(2.0, 0, 1.0 / 16.0, 1.0) == -128.0
    # log^1 closed form of PAPER.md:282
    nu, eps, w2 = 1.5, 0.1, 0.7
    ell = math.log(math.pi * eps * eps * w2)
    assert abs(tail_primitive(nu, 1, eps, w2) + eps ** -nu * (2 + nu * ell) / nu ** 2) < 1e-12


def test_phase_scan_from_reference_constants(golden, golden_integrals):
    """lambda_c(p) from the reference's own constants (SURVEY 8(d) C5 values)."""
    from paper_2504_11989_b200.phase import LatticeConstants, LJParams, critical_coupling, phase_scan
    z = golden["zeta_at_zero"]
    fcc = LatticeConstants("fcc", z["fcc_12"], z["fcc_6"], golden_integrals["fcc"]["atm"],
                           named_lattice("fcc").volume)
    bcc = LatticeConstants("bcc", z["bcc_12"], z["bcc_6"], golden_integrals["bcc"]["atm"],
                           named_lattice("bcc").volume)
    lj = LJParams()
    expect = {0.0: 0.6347989463554651, 0.5: 0.6736514573960529, 1.0: 0.7088057861542634,
              2.0: 0.7706881159724265}
    for p, lc in expect.items():
        got = critical_coupling(fcc, bcc, lj, p)
        assert abs(got - lc) < 1e-9, (p, got, lc)
    vec = critical_coupling(fcc, bcc, lj, list(expect))   # vectorised over pressures
    assert np.allclose(vec, list(expect.values()), rtol=0, atol=1e-9)
    pts = phase_scan(fcc, bcc, lj, [0.0], np.linspace(0, 2, 64))
    assert pts[0].winner == "fcc"      # fcc wins at lambda = 0
    winners = [p.winner for p in pts]
    assert winners.count("bcc") > 0 and winners[-1] == "bcc"
    flips = sum(1 for a, b in zip(winners, winners[1:]) if a != b)
    assert flips == 1


def _taylor_cases(golden):
    import json
    import os
    with open(os.path.join(os.path.dirname(__file__), "golden", "golden_taylor.json")) as f:
        high = json.load(f)["taylor"]
    return list(golden["taylor"]) + high


# the 4-dimensional lattice of tests/golden/make_golden.py (LAT4)
LAT4 = [[1.0, 0.2, 0.0, 0.1], [0.0, 1.1, 0.3, 0.0], [0.0, 0.0, 0.9, 0.2], [0.1, 0.0, 0.0, 1.0]]


def _taylor_lattice(name):
    return Lattice(np.array(LAT4)) if name == "lat4" else named_lattice(name)


def taylor_scales(derivs):
    """Per-order error scale of a Taylor table: the largest |entry| of that order, or (when a whole
    order vanishes by symmetry, e.g. order 10 of the hexagonal nu = 4 table, whose reference entries
    are all ~1e-7 of rounding noise) the geometric mean of the neighbouring orders' scales."""
    mx = {}
    for a, v in derivs:
        o = sum(a)
        mx[o] = max(mx.get(o, 0.0), abs(v))
    sc = {}
    for o, v in mx.items():
        nb = [mx[o - 2], mx[o + 2]] if (o - 2 in mx and o + 2 in mx) else []
        sc[o] = max(v, math.sqrt(nb[0] * nb[1]) if nb else 0.0, 1.0)
    return sc


def test_taylor_tables_match_reference(golden):
    """Host long-double Hermite expansion (the cross-check of the device tables) vs the
    reference's fsum Taylor tables at k = 0, orders up to 12 and d up to 4.  The reference combines
    heavily cancelling Hermite terms in double, so its own error grows with the order: the bound is
    1e-10 of the order's scale (taylor_scales)."""
    from paper_2504_11989_b200.taylor import build_reg_derivatives_host
    for t in _taylor_cases(golden):
        ctx = EpsteinContext(_taylor_lattice(t["lattice"]), t["nu"], device=-1)
        tab = build_reg_derivatives_host(ctx, t["order"])
        assert len(tab.derivs) == len(t["derivs"])
        sc = taylor_scales(t["derivs"])
        for alpha, ref in t["derivs"]:
            got = tab.derivs[tuple(alpha)]
            assert abs(got - ref) <= 1e-10 * sc[sum(alpha)], (t["lattice"], t["nu"], alpha, got, ref)


def test_native_upper_gamma(golden):
    for row in golden["upper_gamma"]:
        s = row["s"]
        if 1e-12 < abs(s - round(s)) < 1e-3:
            continue
        for x, ref in zip(row["x"], row["g"]):
            got = N.lib().lz_upper_gamma(s, x)
            tol = 1e-12 * abs(ref)
            if s < 0:
                tol += 1e-14 * x ** (s + math.ceil(-s) - 1) * math.exp(-x)
            assert abs(got - ref) <= tol, (s, x)


def test_host_only_plans():
    """Fused plans build without a GPU (host tables only) and report their layout."""
    import ctypes as C
    from paper_2504_11989_b200.quadrature import Plan
    fcc = named_lattice("fcc")
    t = 0.65 * fcc.volume ** (-2.0 / 3.0)
    z3 = EpsteinContext(fcc, 3.0, splitting=t, device=-1)
    z5 = EpsteinContext(fcc, 5.0, splitting=t, device=-1)
    h = C.c_void_p()
    N.check(N.lib().lz_plan_create_atm(z3.handle, z5.handle, C.byref(h)))
    plan = Plan(h, 3, 2, (z3, z5))
    info = plan.info()
    assert info.kind == 1 and info.alias == 1 and info.n_funcs == 2   # Z_3's E_1 table serves F'_5
    assert 0 < info.n_dir <= 364 and info.n_runs < info.n_dir       # ball-truncated half cube, runs
    assert info.n_rec >= 728 and info.table_max_rel_err < 6e-16
    assert abs(info.split - t) < 1e-15 and info.smem_bytes < 200_000
    with pytest.raises(RuntimeError):
        plan.integrate(8, 4, 3)
    sq = named_lattice("square")
    c3 = EpsteinContext(sq, 3.0, device=-1)
    c4 = EpsteinContext(sq, 4.0, device=-1)
    arr = (C.c_void_p * 2)(c3.handle, c4.handle)
    mult = (C.c_int * 2)(2, 1)
    h2 = C.c_void_p()
    N.check(N.lib().lz_plan_create_product(arr, mult, 2, C.byref(h2)))
    p2 = Plan(h2, 2, 1, (c3, c4)).info()
    assert p2.kind == 0 and p2.nctx == 2 and p2.n_funcs == 2 and p2.alias == 0
    # ATM plans need nu and nu + 2
    h3 = C.c_void_p()
    assert N.lib().lz_plan_create_atm(c3.handle, c3.handle, C.byref(h3)) != 0


def test_directional_coeff_matches_term_loop():
    """RegZetaTaylor.directional_coeff (one gather over power ladders per order) against the plain
    loop over multi-indices, multinomial(alpha) w^alpha D^alpha / (2k)! (L/epstein.py:449-466), on a
    synthetic table in d = 3 up to order 12, for a batch of directions and a single one."""
    import itertools
    import math
    from paper_2504_11989_b200.epstein import RegZetaTaylor
    rng = np.random.default_rng(5)
    d, order = 3, 12
    derivs = {a: float(rng.normal()) for a in itertools.product(range(order + 1), repeat=d)
              if sum(a) <= order and sum(a) % 2 == 0}
    derivs[(2, 0, 0)] = 0.0   # zero entries are skipped
    tab = RegZetaTaylor(named_lattice("fcc"), 3.0, order, derivs)
    w = rng.normal(size=(9, d))
    w[0, 1] = 0.0             # 0^0 = 1
    for k in range(order // 2 + 1):
        ref = np.zeros(len(w))
        for alpha, val in derivs.items():
            if sum(alpha) != 2 * k:
                continue
            mult = math.factorial(2 * k)
            for a in alpha:
                mult //= math.factorial(a)
            ref += mult * np.prod(w ** np.array(alpha), axis=1) * val
        ref /= math.factorial(2 * k)
        got = tab.directional_coeff(w, k)
        scale = np.max(np.abs(ref)) + 1e-300
        assert np.max(np.abs(got - ref)) <= 1e-12 * scale, k
        assert abs(tab.directional_coeff(w[3], k) - got[3]) <= 1e-15 * scale
    with pytest.raises(ValueError):
        tab.directional_coeff(w, order // 2 + 1)


def test_atm_plan_row_block_host_only():
    """The default d = 3 ATM plan at the low split is the row-factorised one: no slab or line block
    in the shared-memory image (tables only) although the direct set is large; LATSUM_LINE=0
    brings the slab block back; a cell too flat for the row block's plane limit keeps a slab."""
    import ctypes as C
    import os
    from paper_2504_11989_b200 import Lattice
    from paper_2504_11989_b200.quadrature import Plan

    def host_plan(lat, scale):
        t = scale * lat.volume ** (-2.0 / 3.0)
        z3 = EpsteinContext(lat, 3.0, splitting=t, deriv_order=-1, device=-1)
        z5 = EpsteinContext(lat, 5.0, splitting=t, deriv_order=-2, device=-1)
        h = C.c_void_p()
        N.check(N.lib().lz_plan_create_atm(z3.handle, z5.handle, C.byref(h)))
        return Plan(h, 3, 2, (z3, z5)).info()

    for name in ("fcc", "bcc"):
        info = host_plan(named_lattice(name), 0.05)
        assert 5000 < info.n_dir < 7000 and info.smem_bytes < 70_000, (name, info.n_dir, info.smem_bytes)
    os.environ["LATSUM_LINE"] = "0"
    try:
        slab = host_plan(named_lattice("fcc"), 0.13)
    finally:
        del os.environ["LATSUM_LINE"]
    row = host_plan(named_lattice("fcc"), 0.13)
    assert slab.n_dir == row.n_dir and slab.smem_bytes > row.smem_bytes + 30_000
    flat = host_plan(Lattice(np.diag([1.0, 1.0, 0.3])), 0.05)
    assert flat.smem_bytes > 120_000   # slab walk: quadrature.atm_plan then re-plans at the larger split


def test_allreduce_partials_argument_errors():
    """The C-ABI all-reduce validates its arguments before touching CUDA or NCCL."""
    assert N.lib().lz_allreduce_partials(None, 0, None, None) == N.LZ_EINVAL
    assert "communicator" in N.last_error()
    assert N.lib().lz_allreduce_partials(None, 8, C.c_void_p(1), None) == N.LZ_EINVAL


def _bz_even_integrands(lat):
    """Same integrands as tests/golden/make_golden.py:bz_even_cases (restated, not imported:
    the golden script needs the reference)."""
    z1 = lat.a[:, 0]
    z2 = lat.a @ np.ones(lat.d)
    return {
        "one": lambda k: np.ones(len(k)),
        "cos_a1": lambda k: np.cos(2 * np.pi * k @ z1),
        "cos_a1_sq": lambda k: np.cos(2 * np.pi * k @ z1) ** 2,
        "gauss3": lambda k: np.exp(-3.0 * np.einsum("ij,ij->i", k, k)),
        "mix": lambda k: (1.0 + np.einsum("ij,ij->i", k, k)) ** -1.5 * np.cos(2 * np.pi * k @ z2),
    }


def test_integrate_bz_even_matches_reference(golden_near_d):
    """integrate_bz_even (L/quadrature.py:493-515): the reference's adaptive rule, cells in lock
    step; host integrand, so this runs without a GPU.  Lemma 2.5 identities on top: the plane
    wave of a nonzero lattice vector integrates to 0, the constant to 1, cos^2 to 1/2."""
    from paper_2504_11989_b200.quadrature import integrate_bz_even
    for rec in golden_near_d["bz_even"]:
        lat = named_lattice(rec["lattice"])
        v = integrate_bz_even(lat, _bz_even_integrands(lat)[rec["f"]])
        ref = rec["value"]
        assert abs(v - ref) <= 1e-13 * max(1.0, abs(ref)), (rec, v)
        exact = {"one": 1.0, "cos_a1": 0.0, "cos_a1_sq": 0.5}.get(rec["f"])
        if exact is not None:
            assert abs(v - exact) <= 1e-13, (rec, v)


def test_endpoint_exponent_and_auto_grading():
    """The auto rule's grading choice: analytic integrands keep the configured grid (C2, C4 fast
    paths unchanged), exponents just above d get graded."""
    from paper_2504_11989_b200.epstein import EpsteinContext
    from paper_2504_11989_b200.quadrature import auto_grading, endpoint_exponent

    class _C:  # context stand-in: only the branch data is read
        def __init__(self, branch, nu, log_m=None, coef=1.0):
            self.branch, self.nu, self.log_m, self._c = branch, nu, log_m, coef

        def singular_coef(self):
            return self._c

    g, lg, tr = "generic", "log_case", "trivial"
    assert endpoint_exponent([_C(g, 3.0)] * 3, 2) == math.inf          # C2: |k|^1 along rays
    assert endpoint_exponent([_C(lg, 4.0, 1)] * 51, 2) == 3.0          # C4: u^2 log u times u
    assert abs(endpoint_exponent([_C(g, 2.05)], 2) - 1.05) < 1e-12
    assert abs(endpoint_exponent([_C(g, 3.3), _C(lg, 5.0, 1)], 3) - 2.3) < 1e-12
    assert endpoint_exponent([_C(tr, -2.0)], 2) == math.inf
    assert auto_grading(math.inf, 64) == 1
    assert auto_grading(3.0, 256) == 1      # C4 keeps its plain 256-point rule
    assert auto_grading(1.05, 64) == 3
    assert auto_grading(0.3, 64) == 4
    assert auto_grading(1.05, 64, base=5) == 5
