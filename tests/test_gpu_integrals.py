"""GPU parity of the fused Duffy-grid integral kernels (product of zetas, ATM integrand)."""
import numpy as np
import pytest

from oracle import oracle as O
from paper_2504_11989_b200 import named_lattice
from paper_2504_11989_b200.epstein import EpsteinContext
from paper_2504_11989_b200.manybody import ATMGrid, atm_cohesive_energy, atm_integrals, many_body_zeta
from paper_2504_11989_b200.quadrature import Plan, QuadratureConfig, atm_plan, fixed_grid_integral, integrate_product

pytestmark = pytest.mark.gpu
SUM_TOL = 1e-10  # BASELINE north_star: <= 1e-10 relative on each lattice sum


def test_fixed_grids_vs_reference_nodes(golden):
    """Same node set as the reference zeta evaluated on it (golden): node-sum parity."""
    for fg in golden["fixed_grid"]:
        lat = named_lattice(fg["lattice"])
        v = fixed_grid_integral(lat, fg["nus"], fg["n_u"], fg["n_v"], fg["grading"])
        assert abs(v - fg["value"]) <= 1e-12 * abs(fg["value"]), (fg, v)


def test_c2_three_body_square(golden):
    """Config 2: zeta^(3)(3,3,3) on Z^2, Duffy 64 x 64 per cell, vs the reference's adaptive value."""
    cfg = QuadratureConfig(grid_u=64, grid_v=64)
    v, err = integrate_product(named_lattice("square"), (3, 3, 3), cfg)
    ref = golden["c2"]["value"]
    assert abs(v - ref) <= SUM_TOL * abs(ref), (v, ref)
    assert err < 1e-9 * abs(v)


def test_c2_direct_sum_crosscheck():
    """Truncated direct summation |x|,|y| <= R by FFT convolution (BASELINE C2 cross-check)."""
    R = 200
    n = np.arange(-R, R + 1)
    X, Y = np.meshgrid(n, n, indexing="ij")
    r2 = (X * X + Y * Y).astype(float)
    f = np.zeros_like(r2)
    f[r2 > 0] = r2[r2 > 0] ** -1.5
    size = 2 * (2 * R + 1)
    F = np.fft.rfft2(f, s=(size, size))
    conv = np.fft.irfft2(F * F, s=(size, size))
    # sum_{x,y} f(x) f(y-x) f(y): conv[y] = sum_x f(x) f(y - x), shifted by 2R
    g = conv[R:R + 2 * R + 1, R:R + 2 * R + 1]
    direct = float(np.sum(g * f))
    v, _ = integrate_product(named_lattice("square"), (3, 3, 3), QuadratureConfig(grid_u=64, grid_v=64))
    assert abs(direct - v) / v < 2e-9  # truncation error of R = 200 (measured 1.35e-9)


def test_c4_51_body_chain(golden_integrals):
    """Config 4: 51-fold product of Z_4 on Z^2, Duffy 256 x 256."""
    cfg = QuadratureConfig(grid_u=256, grid_v=256, estimate_error=False)
    v, _ = integrate_product(named_lattice("square"), [4.0] * 51, cfg)
    ref = golden_integrals["c4"]["value"]
    assert abs(v - ref) <= SUM_TOL * abs(ref), (v, ref)


def test_hex51_paper_case(golden_integrals):
    cfg = QuadratureConfig(grid_u=256, grid_v=256, estimate_error=False)
    v, _ = integrate_product(named_lattice("hex"), [3.0] * 51, cfg)
    ref = golden_integrals["hex51"]["value"]
    assert abs(v - ref) <= SUM_TOL * abs(ref), (v, ref)


def test_small_products(golden):
    for rec in golden["integrals_small"]:
        lat = named_lattice(rec["lattice"])
        cfg = QuadratureConfig(grid_u=96, grid_v=96, force_integral=True)
        v, _ = integrate_product(lat, rec["nus"], cfg)
        assert abs(v - rec["value"]) <= SUM_TOL * abs(rec["value"]), (rec, v)


def test_two_body_identity():
    lat = named_lattice("hex")
    cfg = QuadratureConfig(grid_u=96, grid_v=96, force_integral=True)
    res = many_body_zeta(lat, (4, 5), cfg)
    ref = many_body_zeta(lat, (4, 5)).value  # Cor. 2.7 short-circuit Z(9, 0)
    assert abs(res.value - ref) <= 1e-12 * abs(ref)
    assert many_body_zeta(lat, (5,)).value == 0.0


def test_atm_grid_vs_oracle():
    """The fused ATM kernel against the long-double oracle on the same small grid."""
    for name in ("fcc", "bcc", "square", "integer_1d"):
        lat = named_lattice(name)
        g = ATMGrid(8, 6, 3)
        res = atm_integrals(lat, g)
        s = O.atm_grid(lat.a, 8, 6, 3)
        sc = 2.0 ** lat.d
        assert abs(res.zeta333 - sc * s[0]) <= 1e-12 * abs(sc * s[0]), name
        assert abs(res.dot_term - sc * s[1]) <= 1e-12 * max(1.0, abs(sc * s[1])), name


@pytest.mark.parametrize("name,key", [("fcc", "fcc"), ("bcc", "bcc")])
def test_c3_atm_energy(golden_integrals, name, key):
    """Config 3 (fcc; bcc for the phase scan): 12 x 128 x 128^2 graded Duffy nodes."""
    res = atm_integrals(named_lattice(name), ATMGrid(128, 128, 3))
    ref = golden_integrals[key]
    assert abs(res.energy - ref["atm"]) <= SUM_TOL * abs(ref["atm"]), (res.energy, ref["atm"])
    assert abs(res.zeta333 - ref["z333"]) <= SUM_TOL * abs(ref["z333"])


@pytest.mark.parametrize("name,key", [("integer_1d", "integer_1d"), ("square", "square")])
def test_atm_low_dimensions(golden_integrals, name, key):
    lat = named_lattice(name)
    g = ATMGrid(256, 256, 3)
    e = atm_cohesive_energy(lat, grid=g)
    ref = golden_integrals[key]["atm"]
    assert abs(e - ref) <= SUM_TOL * abs(ref), (e, ref)


def test_atm_scaling_homogeneity():
    lat = named_lattice("fcc")
    g = ATMGrid(48, 24, 3)
    e1 = atm_cohesive_energy(lat, grid=g)
    e2 = atm_cohesive_energy(lat.scaled(1.3), grid=g)
    assert abs(e2 * 1.3 ** 9 - e1) <= 1e-12 * abs(e1)


def test_nccl_allreduce_through_cabi():
    """lz_allreduce_partials on a one-rank NCCL group (the box has one GPU): the C-ABI all-reduce
    is the identity for W = 1 and the sharded ATM sum through it matches the local one."""
    import socket

    import torch
    import torch.distributed as dist

    from paper_2504_11989_b200 import _native as N
    from paper_2504_11989_b200.distributed import (ShardedIntegral, allreduce_partials,
                                                   nccl_comm_ptr)
    if dist.is_initialized():
        pytest.skip("a process group already exists")
    with socket.socket() as sock:
        sock.bind(("127.0.0.1", 0))
        port = sock.getsockname()[1]
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    try:
        t = torch.arange(1000, dtype=torch.float64, device="cuda")
        dist.all_reduce(t)  # connects the communicator
        comm = nccl_comm_ptr()
        assert comm != 0
        x = torch.linspace(-1.0, 1.0, 4097, dtype=torch.float64, device="cuda")
        y = x.clone()
        allreduce_partials(y)
        torch.cuda.synchronize()
        assert torch.equal(x, y)
        st = torch.cuda.current_stream().cuda_stream
        assert N.lib().lz_allreduce_partials(y.data_ptr(), y.numel(), None, st) == N.LZ_EINVAL
        s = ShardedIntegral(atm_plan(named_lattice("fcc")), 32, 16, 3)
        s.world = 2  # force the collective path (this rank still owns every tile: W = 1 sum)
        out = s.run().cpu().numpy()
        res = atm_integrals(named_lattice("fcc"), ATMGrid(32, 16, 3))
        assert out[0] * 8 == res.zeta333
    finally:
        dist.destroy_process_group()


# (n_u, n_v): 16 -> a tile holds 4 line pairs (atomic tile protocol); 128 -> a line pair is one
# tile, owned by its warp; 96 -> tiles cut line pairs (ranks share a pair's plane sums); 256 -> a
# line pair spans two tiles
@pytest.mark.parametrize("n_u,n_v", [(32, 16), (6, 128), (4, 96), (3, 256)])
def test_tile_sharding_bit_identical(n_u, n_v):
    """Slot-disjoint partials: any split of the tile range gives bit-identical tile partials, and
    the chunked reduction of every world size's shards gives the same bits as the one-call API."""
    import torch

    from paper_2504_11989_b200.distributed import ShardedIntegral
    lat = named_lattice("fcc")
    plan = atm_plan(lat)
    nn, nt = plan.tiles(n_u, n_v, 3)
    full = torch.zeros(nt * 2, dtype=torch.float64, device="cuda")
    plan.integrate_device(full, n_u, n_v, 3)
    for world in (2, 3, 8):
        parts = torch.zeros(nt * 2, dtype=torch.float64, device="cuda")
        for r in range(world):
            lo, hi = nt * r // world, nt * (r + 1) // world
            buf = torch.zeros(nt * 2, dtype=torch.float64, device="cuda")
            plan.integrate_device(buf, n_u, n_v, 3, lo, hi)
            parts += buf  # exact: disjoint slots
        assert torch.equal(parts, full)
    res = atm_integrals(lat, ATMGrid(n_u, n_v, 3))
    for world in (1, 2, 3, 4, 8):
        # each rank's chunks on this GPU in turn; the all-reduce of disjoint chunk slots is a sum
        # with zeros, emulated exactly by adding the per-rank chunk vectors
        chunks = None
        for r in range(world):
            s = ShardedIntegral(plan, n_u, n_v, 3, world=world, rank=r)
            s.world = 1  # no collective: this process is every rank in turn
            s.chunks.zero_()
            s.integrate()
            from paper_2504_11989_b200 import _native as N
            N.check(N.lib().lz_reduce_chunks(s.partials.data_ptr(), s.n_tiles, 2, s.layout.chunk_tiles,
                                             s.chunk_lo, s.chunk_hi, s.chunks.data_ptr(),
                                             torch.cuda.current_stream().cuda_stream))
            chunks = s.chunks.clone() if chunks is None else chunks + s.chunks
        o = torch.zeros(2, dtype=torch.float64, device="cuda")
        Plan.reduce_device(chunks, s.layout.n_chunks, 2, o)
        assert float(o[0]) * 8 == res.zeta333 and float(o[1]) * 8 == res.dot_term, world


@pytest.mark.parametrize("name", ["fcc", "bcc"])
def test_atm_line_kernel_partial_patches_vs_oracle(name):
    """n_v = 40: the second 32-node patch of every line has 24 padding lanes (they repeat the
    line's last node with weight 0, keeping the warp on one line); against the oracle."""
    lat = named_lattice(name)
    res = atm_integrals(lat, ATMGrid(2, 40, 3))
    s = O.atm_grid(lat.a, 2, 40, 3)
    assert abs(res.zeta333 - 8 * s[0]) <= 1e-12 * abs(8 * s[0])
    assert abs(res.dot_term - 8 * s[1]) <= 1e-12 * max(1.0, abs(8 * s[1]))


@pytest.mark.parametrize("name", ["integer_1d", "square", "fcc", "bcc"])
def test_meromorphic_continuation_path(golden_integrals, name):
    """zeta(-1,5,5) and zeta(1,3,5) (some nu <= d): analytic tail on (0, eps) from the native
    Taylor tables + device grid on (eps, 1/2); vs the reference's integrate_product."""
    lat = named_lattice(name)
    ref = golden_integrals[name]
    cfg = QuadratureConfig(grid_u=64, grid_v=48 if lat.d == 3 else 64, method="grid")
    vals = {}
    for key, nus in (("zm155", (-1, 5, 5)), ("z135", (1, 3, 5))):
        v, err = integrate_product(lat, nus, cfg)
        vals[key] = v
        assert abs(v - ref[key]) <= SUM_TOL * abs(ref[key]), (name, key, v, ref[key])
    # Prop. 2.4 recombination vs the Hessian-form ATM energy
    z333 = integrate_product(lat, (3, 3, 3), QuadratureConfig(grid_u=128, grid_v=64, grading=3))[0] \
        if lat.d == 3 else ref["z333"]
    e24 = z333 / 24 - 3 * vals["zm155"] / 16 + 3 * vals["z135"] / 8
    assert abs(e24 - ref["atm"]) <= SUM_TOL * abs(ref["atm"])


def test_table_square_and_normalized(golden_integrals, golden):
    from paper_2504_11989_b200.manybody import normalized_many_body, table_square
    rows = {(n, nu): v for n, nu, v, _ in table_square(n_list=(2, 3, 5), nu_list=(3.0,))}
    sq_z6 = [c for c in golden["cases"] if c["lattice"] == "square" and c["nu"] == 6.0][0]["zeta_at_zero"]
    assert abs(rows[(2, 3.0)] - sq_z6) <= 1e-12 * abs(sq_z6)          # Cor. 2.7
    assert abs(rows[(3, 3.0)] - golden["c2"]["value"]) <= 1e-10 * golden["c2"]["value"]
    five = [r for r in golden["integrals_small"] if r["lattice"] == "square" and len(r["nus"]) == 5][0]
    assert abs(rows[(5, 3.0)] - five["value"]) <= 1e-10 * abs(five["value"])
    hexl = named_lattice("hex")
    assert abs(normalized_many_body(hexl, 3.0, 4)) <= 1.0                # PAPER section 4.3 bound


@pytest.mark.parametrize("name,nus,key", [("square", (3, 3, 3), None), ("square", (1, 3, 5), "z135"),
                                          ("integer_1d", (-1, 5, 5), "zm155"), ("fcc", (-1, 5, 5), "zm155")])
def test_adaptive_method_matches_reference(golden, golden_integrals, name, nus, key):
    """method='adaptive': the reference's GK15/G7 refinement with GPU panels (drop-in fidelity)."""
    lat = named_lattice(name)
    cfg = QuadratureConfig(method="adaptive")
    v, err = integrate_product(lat, nus, cfg)
    ref = golden["c2"]["value"] if key is None else golden_integrals[name][key]
    ref_err = golden["c2"]["err"] if key is None else golden_integrals[name][key + "_err"]
    assert abs(v - ref) <= max(1e-12 * abs(ref), 2 * ref_err), (v, ref)
    assert 0.0 < err < 1e-9 * abs(v)


def test_c5_phase_scan_from_gpu_constants(golden, golden_integrals):
    """Config 5: LJ(12,6) + lambda ATM, fcc vs bcc; constants Z(6,0), Z(12,0), K_ATM on the GPU."""
    from paper_2504_11989_b200.phase import LJParams, critical_coupling, lattice_constants, phase_scan
    lj = LJParams()
    fcc = lattice_constants("fcc", lj, ATMGrid(128, 128, 3))
    bcc = lattice_constants("bcc", lj, ATMGrid(128, 128, 3))
    z = golden["zeta_at_zero"]
    assert abs(fcc.z_n - z["fcc_12"]) <= 1e-12 * z["fcc_12"] and abs(bcc.z_m - z["bcc_6"]) <= 1e-12 * z["bcc_6"]
    assert abs(fcc.k_atm - golden_integrals["fcc"]["atm"]) <= 1e-10 * golden_integrals["fcc"]["atm"]
    assert abs(bcc.k_atm - golden_integrals["bcc"]["atm"]) <= 1e-10 * golden_integrals["bcc"]["atm"]
    expect = {0.0: 0.6347989463554651, 0.5: 0.6736514573960529, 1.0: 0.7088057861542634,
              2.0: 0.7706881159724265}
    for p, lc in expect.items():
        assert abs(critical_coupling(fcc, bcc, lj, p) - lc) < 1e-8, p
    pts = phase_scan(fcc, bcc, lj, [0.0, 1.0], np.linspace(0.0, 2.0, 64), np.linspace(0.9, 1.7, 64))
    assert pts[0].winner == "fcc" and pts[63].winner == "bcc"


def test_direct_sums_reproduce_paper_and_epstein(golden, golden_integrals):
    """GPU direct summation (SPEC oracle module): the paper's own direct-sum values, and the
    algebraic convergence of direct sums to the Epstein-method results."""
    from paper_2504_11989_b200.direct import direct_sum_atm, direct_sum_zeta
    # 1D ATM by direct summation at L = 5000
    e1 = direct_sum_atm(named_lattice("Z"), 5000)
    assert abs(e1 - (-0.2723018495076886)) <= 2e-15
    # 2D square-lattice ATM at L = 250 ("over 10^10 summands", ~6 h on one core)
    e2 = direct_sum_atm(named_lattice("square"), 250)
    assert abs(e2 - 0.7700936511489661) <= 1e-13 * abs(e2)
    # the truncated sums approach the Epstein values
    ref2 = golden_integrals["square"]["atm"]
    assert abs(e2 - ref2) < 1e-8 * ref2
    z = direct_sum_zeta(named_lattice("square"), (3, 3, 3), 200)
    assert abs(z - golden["c2"]["value"]) < 3e-9 * golden["c2"]["value"]
    fcc = named_lattice("fcc")
    errs = [abs(direct_sum_atm(fcc, L) - golden_integrals["fcc"]["atm"]) for L in (4, 8, 16)]
    assert errs[0] > errs[1] > errs[2] and errs[2] < 5e-4 * golden_integrals["fcc"]["atm"]


@pytest.mark.parametrize("scale", [0.17, 0.3, 0.6, 1.0])
def test_atm_energy_split_invariance(scale):
    """The fused ATM sum does not depend on the theta split (0.17 makes the direct block too large
    for the parameter-space variant, exercising the shared-memory fallback)."""
    lat = named_lattice("fcc")
    grid = ATMGrid(32, 16, 3)
    ref = atm_integrals(lat, grid)
    t = scale * lat.volume ** (-2.0 / 3.0)
    res = atm_integrals(lat, grid, splitting=t)
    assert abs(res.energy - ref.energy) <= 1e-12 * abs(ref.energy)
    assert abs(res.dot_term - ref.dot_term) <= 1e-12 * abs(ref.dot_term)
    if scale == 0.17:
        info = atm_plan(lat, t).info()
        assert info.n_dir * 4 > 3584  # direct block exceeds the 28 KB parameter block


@pytest.mark.parametrize("seed", [3, 11])
def test_atm_line_kernel_skewed_lattice_vs_oracle(seed):
    """Line-factorised ATM kernel on a generic (skewed, anisotropic) 3D lattice: its line block
    (plane grouping per pyramid axis, step codes, v = sqrt|w| z) against the long-double oracle."""
    from paper_2504_11989_b200 import Lattice
    rng = np.random.default_rng(seed)
    a = (np.eye(3) + rng.uniform(-0.25, 0.25, (3, 3))) * rng.uniform(0.8, 1.3)
    lat = Lattice(a)
    res = atm_integrals(lat, ATMGrid(2, 8, 3))
    s = O.atm_grid(lat.a, 2, 8, 3)
    assert abs(res.zeta333 - 8 * s[0]) <= 1e-12 * abs(8 * s[0])
    assert abs(res.dot_term - 8 * s[1]) <= 1e-12 * max(1.0, abs(8 * s[1]))
    assert atm_plan(lat).info().n_dir > 0


@pytest.mark.parametrize("u", [[[1, 1, 0], [0, 1, 0], [0, 0, 1]], [[1, 0, 0], [1, 1, 0], [-1, 0, 1]]])
def test_atm_energy_basis_invariance(u):
    """The ATM energy is a property of the lattice, not of its basis: fcc with a unimodular change
    of basis (different line blocks, pyramid axes and reciprocal bookkeeping) gives the same sum
    to the quadrature/rounding level (the Duffy cells follow the basis, so the grids differ)."""
    from paper_2504_11989_b200 import Lattice
    fcc = named_lattice("fcc")
    other = Lattice(fcc.a @ np.array(u, dtype=float))
    e0 = atm_cohesive_energy(fcc, grid=ATMGrid(64, 64, 3))
    e1 = atm_cohesive_energy(other, grid=ATMGrid(64, 64, 3))
    assert abs(e1 - e0) <= 1e-8 * abs(e0), (e0, e1)


def test_near_d_products_meet_reference_contract(golden_near_d):
    """integrate_product's default for exponents just above d: the reference's
    whole-range adaptive value (L/quadrature.py:421-423) within max(1e-10 |ref|, 2 ref_err).
    The one-body case (nu = 2.01) is exactly 0 (SPEC one-body identity); the reference itself
    misses 0 by 1.5e-13 against its own 2e-14 estimate, so that case checks we are at least as
    close to 0."""
    for rec in golden_near_d["cases"]:
        lat = named_lattice(rec["lattice"])
        v, err = integrate_product(lat, rec["nus"])
        ref = rec["value"]
        if len(rec["nus"]) == 1:
            assert abs(v) <= max(abs(ref), 1e-14), (rec, v)
            continue
        tol = max(SUM_TOL * abs(ref), 2.0 * rec["err"])
        assert abs(v - ref) <= tol, (rec, v, err)
        assert err <= 1e-11 * abs(v), (rec, err)


def test_near_d_escalation_to_adaptive(golden_near_d):
    """A grid too coarse for its own error check escalates (doubled grid, then the reference's
    adaptive rule) instead of returning an unconverged value."""
    rec = next(r for r in golden_near_d["cases"] if r["nus"] == [2.05, 2.05, 2.05])
    lat = named_lattice(rec["lattice"])
    v, err = integrate_product(lat, rec["nus"], QuadratureConfig(grid_u=6, grid_v=6))
    assert abs(v - rec["value"]) <= max(SUM_TOL * abs(rec["value"]), 2.0 * rec["err"]), (v, err)
    # method="grid" is the literal grid: no escalation, and its estimate shows the gap
    vg, eg = integrate_product(lat, rec["nus"], QuadratureConfig(grid_u=64, grid_v=64, method="grid"))
    assert abs(vg - rec["value"]) > 1e-6 * abs(rec["value"]) and eg > 1e-6 * abs(vg)


@pytest.mark.gpu
def test_product_at_matches_zeta_products():
    """lz_plan_product_at (one fused kernel for prod_j Z_j^{m_j} at arbitrary k, the adaptive
    path's integrand) against the single-context zeta kernels on the same points."""
    import torch
    from paper_2504_11989_b200.quadrature import product_plan
    for name, groups in [("fcc", ((3.0, 1), (5.0, 2))), ("square", ((3.5, 3),)),
                         ("bcc", ((-1.0, 1), (5.0, 1), (1.0, 1), (3.0, 2)))]:
        lat = named_lattice(name)
        k = np.random.default_rng(4).uniform(-0.5, 0.5, size=(2000, lat.d)) @ lat.a_inv_t.T
        got = product_plan(lat, groups).product_at(torch.tensor(k, device="cuda")).cpu().numpy()
        ref = np.ones(len(k))
        for nu, m in groups:
            ref = ref * EpsteinContext(lat, nu, device=0).zeta(k) ** m
        assert np.abs(got - ref).max() <= 1e-12 * np.abs(ref).max(), name


@pytest.mark.gpu
def test_product_at_edge_cases():
    """Empty batches, pole detection at k in the reciprocal lattice (nu = d), and the ATM plan
    rejected by lz_plan_product_at."""
    import ctypes as C
    import torch
    from paper_2504_11989_b200 import _native as N
    from paper_2504_11989_b200.quadrature import product_plan
    sq = named_lattice("square")
    plan = product_plan(sq, ((3.0, 2),))
    assert plan.product_at(torch.zeros((0, 2), dtype=torch.float64, device="cuda")).numel() == 0
    pole = product_plan(sq, ((2.0, 1), (3.0, 1)))   # nu = d: pole at k in the reciprocal lattice
    k = torch.tensor([[0.1, 0.2], [1.0, 0.0]], dtype=torch.float64, device="cuda")
    out = torch.empty(2, dtype=torch.float64, device="cuda")
    st = torch.zeros(1, dtype=torch.int32, device="cuda")
    N.check(N.lib().lz_plan_product_at(pole.handle, k.data_ptr(), 2, out.data_ptr(), st.data_ptr(),
                                       torch.cuda.current_stream().cuda_stream), "product at")
    torch.cuda.synchronize()
    assert int(st.item()) & 1
    with pytest.raises(ValueError):
        atm_plan(named_lattice("fcc")).product_at(k[:, :1].repeat(1, 3).contiguous())


@pytest.mark.gpu
def test_derivatives_device_matches_host_path():
    """EpsteinContext.derivatives_device (device pointers, stream-ordered) equals the host-buffer
    entry point bit for bit, for the compile-time (order 3) and moment (order 7, d = 4) kernels."""
    import torch
    from paper_2504_11989_b200 import Lattice
    lat4 = Lattice(np.array([[1.0, 0.2, 0.0, 0.1], [0.0, 1.1, 0.3, 0.0], [0.0, 0.0, 0.9, 0.2],
                             [0.1, 0.0, 0.0, 1.0]]))
    for lat, nu, m in ((named_lattice("fcc"), 5.0, 3), (lat4, 6.0, 7)):
        k = np.random.default_rng(5).uniform(-0.4, 0.4, size=(300, lat.d)) @ lat.a_inv_t.T
        ctx = EpsteinContext(lat, nu, device=0)
        _, host = ctx.derivatives(k, m)
        dev = ctx.derivatives_device(torch.tensor(k, device="cuda"), m).cpu().numpy()
        assert np.array_equal(host, dev)
        assert ctx.derivatives_device(torch.zeros((0, lat.d), dtype=torch.float64, device="cuda"), m).shape[0] == 0


@pytest.mark.gpu
def test_device_taylor_table_trivial_branch():
    """Trivial branch (nu in -2N0): Z_reg is the constant Z(nu, 0) (L/epstein.py:371-375)."""
    ctx = EpsteinContext(named_lattice("square"), -2.0, device=0)
    tab = ctx.reg_derivatives(6)
    assert tab.derivs[(0, 0)] == ctx.const_value
    assert all(v == 0.0 for a, v in tab.derivs.items() if sum(a) > 0)


def _golden_atm_generic():
    import json
    import os
    with open(os.path.join(os.path.dirname(__file__), "golden", "golden_atm_generic.json")) as f:
        return json.load(f)


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["hexagonal", "oblique", "triclinic"])
def test_atm_generic_lattices(name):
    """The fused ATM kernels (d = 2 tile kernel, d = 3 line kernel) on lattices without the
    catalog's symmetry, and the Prop. 2.4 adaptive route, against the reference's own Prop. 2.4
    energies (tests/golden/make_golden.py --atm-generic)."""
    from paper_2504_11989_b200 import Lattice
    g = _golden_atm_generic()[name]
    mats = {"oblique": [[1.0, 0.35], [0.0, 0.9]],
            "triclinic": [[1.0, 0.15, 0.25], [0.0, 1.1, 0.3], [0.05, 0.0, 0.95]]}
    lat = named_lattice(name) if name == "hexagonal" else Lattice(np.array(mats[name]))
    res = atm_integrals(lat, ATMGrid(128, 128, 3))
    assert abs(res.energy - g["atm"]) <= 1e-10 * abs(g["atm"]), (res.energy, g["atm"])
    cfg = QuadratureConfig(method="adaptive")
    for key, nus in (("z333", (3, 3, 3)), ("zm155", (-1, 5, 5)), ("z135", (1, 3, 5))):
        v, _ = integrate_product(lat, nus, cfg)
        assert abs(v - g[key]) <= max(1e-12 * abs(g[key]), 2 * g[key + "_err"]), (key, v, g[key])


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["fcc", "bcc", "triclinic"])
@pytest.mark.parametrize("grid", [(4, 128, 3), (3, 64, 3), (2, 96, 3), (2, 40, 3), (1, 288, 3)])
def test_atm_kernel_forms_agree(name, grid, monkeypatch):
    """The three ATM kernel forms -- row-factorised direct space (D table per axis and radial node,
    the default), the shared-memory line block (LATSUM_LINE=1) and the slab walk (LATSUM_LINE=0)
    -- give the same sums on the same split.  Grids: whole patch pairs (the row kernel's
    four-node fast path), two patches per line, an odd patch count and a partial last patch
    (its per-patch path), and more angular nodes than the row kernel stages in shared memory."""
    from paper_2504_11989_b200 import Lattice
    lat = named_lattice(name) if name != "triclinic" else \
        Lattice(np.array([[1.0, 0.15, 0.25], [0.0, 1.1, 0.3], [0.05, 0.0, 0.95]]))
    t = 0.13 * lat.volume ** (-2.0 / 3.0)
    out = {}
    for form in ("2", "1", "0"):
        monkeypatch.setenv("LATSUM_LINE", form)
        atm_plan.cache_clear()
        out[form] = atm_integrals(lat, ATMGrid(*grid), splitting=t)
    monkeypatch.delenv("LATSUM_LINE")
    atm_plan.cache_clear()
    for form in ("1", "0"):
        assert abs(out[form].zeta333 - out["2"].zeta333) <= 2e-13 * abs(out["2"].zeta333), form
        assert abs(out[form].dot_term - out["2"].dot_term) <= 2e-13 * abs(out["2"].dot_term), form


@pytest.mark.gpu
def test_atm_default_plan_uses_row_block():
    """The default fcc / bcc ATM plans take the row-factorised block (no slab or line block staged:
    the shared-memory image is the tables only) at the low split, and a very flat cell that does
    not fit it falls back to the slab walk at the larger split."""
    from paper_2504_11989_b200 import Lattice
    for name in ("fcc", "bcc"):
        lat = named_lattice(name)
        info = atm_plan(lat).info()
        assert info.smem_bytes < 70_000 and info.n_dir > 4000
        assert abs(info.split - 0.05 * lat.volume ** (-2.0 / 3.0)) < 1e-15
    flat = Lattice(np.diag([1.0, 1.0, 0.3]))
    info = atm_plan(flat).info()
    assert abs(info.split - 0.13 * flat.volume ** (-2.0 / 3.0)) < 1e-15
    res = atm_integrals(flat, ATMGrid(2, 8, 3))
    s = O.atm_grid(flat.a, 2, 8, 3)
    assert abs(res.zeta333 - 8 * s[0]) <= 1e-12 * abs(8 * s[0])
    assert abs(res.dot_term - 8 * s[1]) <= 1e-12 * max(1.0, abs(8 * s[1]))


@pytest.mark.gpu
def test_atm_row_kernel_candidate_overflow(monkeypatch):
    """A line pair whose reciprocal candidates overflow the per-warp list makes every node test all
    points within reach itself (fast-path kernel) or takes the per-patch culling (general kernel):
    forced with a zero-capacity list, both give the default result bit for bit (the same terms in
    the same order; the rest contribute exact zeros)."""
    lat = named_lattice("fcc")
    grid = ATMGrid(6, 128, 3)
    ref = atm_integrals(lat, grid)
    monkeypatch.setenv("LATSUM_ROW_CAND_MAX", "0")
    atm_plan.cache_clear()
    res = atm_integrals(lat, grid)
    monkeypatch.delenv("LATSUM_ROW_CAND_MAX")
    atm_plan.cache_clear()
    assert res.zeta333 == ref.zeta333 and res.dot_term == ref.dot_term
