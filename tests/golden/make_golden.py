#!/usr/bin/env python3
"""Generate golden fixtures by running the UNMODIFIED reference ``latsum`` package.

Test infrastructure only.  This script imports the reference from
``/root/reference/pkg/src/latsum`` under the alias ``latsum_ref`` (so it can
coexist with the new package) and writes small JSON fixtures next to itself:

* ``golden.json``           quick items (seconds): contexts, zeta values,
                            incomplete gamma, fixed-grid node sums, C1, C2.
* ``golden_integrals.json`` slow items (minutes): the reference's adaptive
                            ``integrate_product`` for C4 and the fcc/bcc
                            three-body integrals behind the ATM energies.
* ``golden_near_d.json``    ``--near-d``: the reference's whole-range adaptive
                            ``integrate_product`` for exponents just above the
                            dimension (slowly converging algebraic endpoint
                            singularities) and ``integrate_bz_even`` on smooth
                            even integrands.

The GPU box has no ``/root/reference``; the fixtures travel instead.
Usage:  python tests/golden/make_golden.py [--slow | --near-d] [--threads N]
"""
from __future__ import annotations

import argparse
import importlib.util
import json
import math
import os
import sys
import time

import numpy as np

REF_SRC = "/root/reference/pkg/src/latsum"
HERE = os.path.dirname(os.path.abspath(__file__))


def load_reference():
    spec = importlib.util.spec_from_file_location(
        "latsum_ref", os.path.join(REF_SRC, "__init__.py"),
        submodule_search_locations=[REF_SRC])
    mod = importlib.util.module_from_spec(spec)
    sys.modules["latsum_ref"] = mod
    spec.loader.exec_module(mod)
    import latsum_ref.epstein  # noqa: F401
    import latsum_ref.incgamma  # noqa: F401
    import latsum_ref.quadrature  # noqa: F401
    return mod


def fl(x):
    return [float(v) for v in np.ravel(x)]


# (lattice name, nu) pairs whose contexts and zeta values are pinned.
CASES = [
    ("integer_1d", 2.0), ("integer_1d", 3.0), ("integer_1d", 0.5), ("integer_1d", 5.0),
    ("square", 3.5), ("square", 3.0), ("square", 4.0), ("square", 8.0),
    ("square", 2.0), ("square", 1.5), ("square", 5.0), ("square", 9.0),
    ("square", -1.0), ("square", 6.0),
    ("hexagonal", 3.0), ("hexagonal", 9.0),
    ("fcc", 3.0), ("fcc", 5.0), ("fcc", 6.0), ("fcc", 12.0), ("fcc", 1.0), ("fcc", -1.0),
    ("fcc", 4.2),
    ("bcc", 3.0), ("bcc", 5.0), ("bcc", 6.0), ("bcc", 12.0),
    ("square", 3.0005),  # near-integer incomplete-gamma order (Lentz branch)
    ("square", -2.0),    # trivial branch
]


def context_record(ref, lat, nu):
    ctx = ref.epstein.epstein_context(lat, nu)
    rec = {"branch": ctx.branch, "nu": ctx.nu, "log_m": ctx.log_m, "vol": ctx.vol,
           "split": ctx.split}
    if ctx.branch == "trivial":
        rec["const_value"] = ctx.const_value
        return ctx, rec
    rec.update({
        "s_rec": ctx.s_rec, "pref": ctx.pref, "rfac": ctx.rfac, "bconst": ctx.bconst,
        "kmax": ctx.kmax, "n_dir": int(len(ctx.dir_pts)), "n_rec": int(len(ctx.rec_pts)),
        "dir_w_fsum": math.fsum(ctx.dir_w), "rec_norm2_fsum": math.fsum(ctx.rec_norm2),
        "singular_coef": ctx.singular_coef(),
    })
    # exact point sets for the small 1D/2D cases (lattice coordinates, Cartesian)
    if lat.d <= 2:
        rec["dir_pts"] = fl(ctx.dir_pts)
        rec["dir_w"] = fl(ctx.dir_w)
        rec["rec_pts"] = fl(ctx.rec_pts)
    return ctx, rec


def sample_points(d, rng, n):
    """Seeded k points: inside the BZ box, on its boundary, and outside it."""
    kap = rng.uniform(-0.5, 0.5, size=(n, d))
    kap[0] = 0.5                      # corner
    kap[1, 0] = -0.5                  # face
    kap[2] = 1e-3                     # near the singularity
    kap[3] = rng.uniform(-3.0, 3.0, size=d)   # outside: exercises reduction
    kap[4] = 0.25
    return kap


def quick(ref):
    out = {"generator": "tests/golden/make_golden.py", "reference": REF_SRC,
           "numpy": np.__version__}
    import scipy
    out["scipy"] = scipy.__version__
    E = ref.epstein
    # ---- C1 ----------------------------------------------------------------
    sq = ref.named_lattice("square")
    k1 = np.random.default_rng(0).uniform(-0.5, 0.5, size=(4096, 2))
    z1 = E.epstein_context(sq, 3.5).zeta(k1)
    out["c1"] = {"lattice": "square", "nu": 3.5, "seed": 0, "n": 4096,
                 "k_fsum": math.fsum(k1.ravel()), "k0": fl(k1[0]),
                 "zeta": fl(z1), "zeta_fsum": math.fsum(z1)}
    # ---- contexts + zeta/reg/singular at sample points ---------------------
    cases = []
    rng = np.random.default_rng(1234)
    for name, nu in CASES:
        lat = ref.named_lattice(name)
        ctx, rec = context_record(ref, lat, nu)
        kap = sample_points(lat.d, rng, 12)
        kk = kap @ lat.a_inv_t.T
        rec["lattice"] = name
        rec["k"] = fl(kk)
        rec["zeta"] = fl(ctx.zeta(kk))
        rec["reg_zeta"] = fl(ctx.reg_zeta(kk))
        if ctx.branch != "trivial":
            try:
                rec["zeta_at_zero"] = ctx.zeta_at_zero()
            except ref.PoleError:
                rec["zeta_at_zero"] = "pole"
        cases.append(rec)
    out["cases"] = cases
    # ---- incomplete gamma --------------------------------------------------
    ug = []
    xs = np.array([0.003, 0.05, 0.3, 0.785, 1.0, 1.5, 2.0, 3.7, 7.5, 15.0, 30.0, 45.0])
    for s in [2.5, 1.5, 1.0, 0.5, 0.25, 0.0, -0.5, -0.75, -1.0, -1.5, -2.0, -2.5,
              -3.0, -4.5, -0.9995, 3.0, 6.0, 0.0005]:
        ug.append({"s": s, "x": fl(xs), "g": fl(ref.incgamma.upper_gamma(s, xs))})
    out["upper_gamma"] = ug
    xe = np.array([1e-6, 0.01, 0.3, 0.99, 1.0, 2.5, 10.0, 40.0])
    out["exp1_plus_log"] = {"x": fl(xe), "v": fl(ref.incgamma.exp1_plus_log(xe))}
    # ---- fixed Duffy grids: reference zeta on exactly our node sets ---------
    out["fixed_grid"] = [fixed_grid_sum(ref, "square", [3, 3, 3], 8, 8, 1),
                         fixed_grid_sum(ref, "square", [4] * 51, 8, 8, 1),
                         fixed_grid_sum(ref, "square", [3.5, 5.0], 6, 5, 2),
                         fixed_grid_sum(ref, "hexagonal", [3, 3, 3], 6, 6, 1),
                         fixed_grid_sum(ref, "fcc", [3, 3, 3], 4, 3, 3),
                         fixed_grid_sum(ref, "bcc", [3, 4.5], 3, 3, 3)]
    # ---- quick adaptive integrals ----------------------------------------
    Q = ref.quadrature
    t = time.time()
    v, e = Q.integrate_product(sq, (3, 3, 3))
    out["c2"] = {"lattice": "square", "nus": [3, 3, 3], "value": v, "err": e,
                 "seconds_1thread": time.time() - t}
    two = []
    for name, nus in [("square", (4, 5)), ("hexagonal", (4, 5)), ("square", (3.5, 6.0)),
                      ("square", (3, 3, 3, 3, 3)), ("hexagonal", (3, 3, 3, 3, 3))]:
        lat = ref.named_lattice(name)
        v, e = Q.integrate_product(lat, nus)
        two.append({"lattice": name, "nus": list(nus), "value": v, "err": e})
    out["integrals_small"] = two
    # ---- phase constants (Z(nu, 0)) -----------------------------------------
    pc = {}
    for name in ("fcc", "bcc"):
        lat = ref.named_lattice(name)
        for nu in (6.0, 12.0, 5.0, 4.0):
            pc[f"{name}_{nu:g}"] = E.epstein_context(lat, nu).zeta_at_zero()
    out["zeta_at_zero"] = pc
    # ---- finite-difference Hessians of Z_5 (loose check of the new M(k)) ------
    fd = []
    for name in ("fcc", "bcc"):
        lat = ref.named_lattice(name)
        c5 = E.epstein_context(lat, 5.0)
        c3 = E.epstein_context(lat, 3.0)
        for kap in ([0.11, -0.23, 0.31], [0.4, 0.05, -0.2], [-0.02, 0.03, 0.045]):
            k = np.array(kap) @ lat.a_inv_t.T
            h = 2e-4
            H = np.zeros((3, 3))
            for a in range(3):
                for b in range(3):
                    ea = np.eye(3)[a] * h
                    eb = np.eye(3)[b] * h
                    pts = np.array([k + ea + eb, k + ea - eb, k - ea + eb, k - ea - eb])
                    f = c5.zeta(pts)
                    H[a, b] = (f[0] - f[1] - f[2] + f[3]) / (4 * h * h)
            M = -H / (4 * math.pi ** 2)
            fd.append({"lattice": name, "k": fl(k), "M_fd": fl(M),
                       "z3": float(c3.zeta(k)), "z5": float(c5.zeta(k))})
    out["hessian_fd"] = fd
    # ---- Taylor tables at k = 0 (for the tail path) ---------------------------
    tay = []
    for name, nu, order in [("square", 2.0, 8), ("square", 1.0, 6), ("fcc", 5.0, 4),
                            ("integer_1d", -1.0, 8)]:
        lat = ref.named_lattice(name)
        tab = E.reg_zeta_derivatives(lat, nu, order)
        tay.append({"lattice": name, "nu": nu, "order": order,
                    "derivs": [[list(a), float(v)] for a, v in sorted(tab.derivs.items())]})
    out["taylor"] = tay
    return out


def duffy_nodes(lat, n_u, n_v, grading):
    """Fixed Duffy grid in the reference's coordinates (L/quadrature.py:136-177)
    with Gauss-Legendre in u on (0,1/2), graded u = t^q / 2."""
    x, w = np.polynomial.legendre.leggauss(n_u)
    tt = (x + 1.0) / 2.0
    wt = w / 2.0
    u = 0.5 * tt ** grading
    wu = wt * 0.5 * grading * tt ** (grading - 1)
    Q = sys.modules["latsum_ref.quadrature"]
    d = lat.d
    v, wv = Q.angular_nodes(d, n_v)
    ks, ws = [], []
    for cell in Q.duffy_cells(d):
        wdir = cell.directions(lat, v)
        k = (u[:, None, None] * wdir[None, :, :]).reshape(-1, d)
        wt2 = (wu[:, None] * u[:, None] ** (d - 1) * wv[None, :]).ravel()
        ks.append(k)
        ws.append(wt2)
    return np.concatenate(ks), np.concatenate(ws)


def fixed_grid_sum(ref, name, nus, n_u, n_v, grading):
    lat = ref.named_lattice(name)
    d = lat.d
    k, w = duffy_nodes(lat, n_u, n_v, grading)
    prod = np.ones(len(k))
    for nu in nus:
        prod = prod * ref.epstein.epstein_context(lat, float(nu)).zeta(k)
    val = 2.0 ** d * math.fsum(w * prod)
    return {"lattice": name, "nus": [float(v) for v in nus], "n_u": n_u, "n_v": n_v,
            "grading": grading, "n_nodes": int(len(k)), "value": val}


def slow(ref, threads):
    Q = ref.quadrature
    out = {"generator": "tests/golden/make_golden.py --slow", "threads": threads}
    sq = ref.named_lattice("square")
    t = time.time()
    v, e = Q.integrate_product(sq, [4.0] * 51, threads=threads)
    out["c4"] = {"lattice": "square", "nus": "[4]*51", "value": v, "err": e,
                 "z0": ref.epstein.epstein_context(sq, 4.0).zeta_at_zero(),
                 "seconds": time.time() - t}
    hexl = ref.named_lattice("hex")
    v, e = Q.integrate_product(hexl, [3.0] * 51, threads=threads)
    out["hex51"] = {"value": v, "err": e}
    for name in ("integer_1d", "square", "fcc", "bcc"):
        lat = ref.named_lattice(name)
        rec = {}
        for key, nus in (("z333", (3, 3, 3)), ("zm155", (-1, 5, 5)), ("z135", (1, 3, 5))):
            t = time.time()
            v, e = Q.integrate_product(lat, nus, threads=threads)
            rec[key] = v
            rec[key + "_err"] = e
            rec[key + "_seconds"] = time.time() - t
            print(name, key, v, e, time.time() - t, flush=True)
        rec["atm"] = rec["z333"] / 24 - 3 * rec["zm155"] / 16 + 3 * rec["z135"] / 8
        out[name] = rec
    return out


# products with every exponent above d whose integrand u^(d-1) prod Z(u w) carries a
# non-analytic u^eta (eta = d-1 + min(nu)-d) or u^eta log u endpoint term
NEAR_D = [("square", (2.05, 2.05, 2.05)), ("square", (2.2, 3.0, 3.0)), ("square", (2.5, 2.5)),
          ("square", (2.01,)), ("square", (3.5, 4.0)), ("hexagonal", (2.1, 2.1, 2.1)),
          ("integer_1d", (1.3, 2.0)), ("fcc", (3.3, 4.0, 4.0)), ("bcc", (3.5, 3.5))]


def bz_even_cases(ref):
    """Smooth even integrands for integrate_bz_even, as (lattice, label, callable)."""
    out = []
    for name in ("integer_1d", "square", "hexagonal", "fcc"):
        lat = ref.named_lattice(name)
        d = lat.d
        z1 = lat.a[:, 0]
        z2 = lat.a @ np.ones(d)
        out.append((name, "one", lambda k: np.ones(len(k))))
        out.append((name, "cos_a1", lambda k, z=z1: np.cos(2 * np.pi * k @ z)))
        out.append((name, "cos_a1_sq", lambda k, z=z1: np.cos(2 * np.pi * k @ z) ** 2))
        out.append((name, "gauss3", lambda k: np.exp(-3.0 * np.einsum("ij,ij->i", k, k))))
        out.append((name, "mix", lambda k, z=z2: (1.0 + np.einsum("ij,ij->i", k, k)) ** -1.5
                    * np.cos(2 * np.pi * k @ z)))
    return out


def near_d(ref, threads):
    Q = ref.quadrature
    out = {"generator": "tests/golden/make_golden.py --near-d", "threads": threads,
           "cases": [], "bz_even": []}
    for name, nus in NEAR_D:
        lat = ref.named_lattice(name)
        t = time.time()
        v, e = Q.integrate_product(lat, nus, threads=threads)
        rec = {"lattice": name, "nus": list(nus), "value": v, "err": e,
               "seconds": time.time() - t}
        print(rec, flush=True)
        out["cases"].append(rec)
    for name, label, f in bz_even_cases(ref):
        lat = ref.named_lattice(name)
        v = Q.integrate_bz_even(lat, f)
        out["bz_even"].append({"lattice": name, "f": label, "value": v})
    return out


# the 4-dimensional test lattice of tests/test_gpu_zeta.py (L/lattice.py:20 allows d <= 4)
LAT4 = [[1.0, 0.2, 0.0, 0.1], [0.0, 1.1, 0.3, 0.0], [0.0, 0.0, 0.9, 0.2], [0.1, 0.0, 0.0, 1.0]]


def taylor_high(ref):
    """Taylor tables of Z_reg at k = 0 up to the reference's maximum order 12 (L/epstein.py:347-353),
    d = 2, 3 and 4, every branch (generic, log case)."""
    E = sys.modules["latsum_ref.epstein"]
    out = {"taylor": []}
    cases = [("square", 3.5, 12), ("hexagonal", 4.0, 12), ("fcc", 3.0, 8), ("bcc", 5.0, 8),
             ("fcc", 6.0, 12), ("lat4", 6.0, 6), ("lat4", 3.0, 4)]
    for name, nu, order in cases:
        lat = ref.Lattice(np.array(LAT4)) if name == "lat4" else ref.named_lattice(name)
        t0 = time.time()
        tab = E.reg_zeta_derivatives(lat, nu, order)
        out["taylor"].append({"lattice": name, "nu": nu, "order": order, "seconds": time.time() - t0,
                              "derivs": [[list(a), float(v)] for a, v in sorted(tab.derivs.items())]})
        print(name, nu, order, "%.1f s" % (time.time() - t0), flush=True)
    return out


# lattices without the catalog's symmetry for the ATM goldens (line kernel on a generic cell)
TRICLINIC = [[1.0, 0.15, 0.25], [0.0, 1.1, 0.3], [0.05, 0.0, 0.95]]
OBLIQUE = [[1.0, 0.35], [0.0, 0.9]]


def atm_generic(ref, threads):
    """ATM energies (Prop. 2.4: the three continued integrals of the reference's own adaptive
    route) on the hexagonal lattice and on lattices without symmetry (triclinic 3D, oblique 2D)."""
    Q = ref.quadrature
    out = {"generator": "tests/golden/make_golden.py --atm-generic", "threads": threads}
    for name, lat in (("hexagonal", ref.named_lattice("hexagonal")),
                      ("oblique", ref.Lattice(np.array(OBLIQUE))),
                      ("triclinic", ref.Lattice(np.array(TRICLINIC)))):
        rec = {}
        for key, nus in (("z333", (3, 3, 3)), ("zm155", (-1, 5, 5)), ("z135", (1, 3, 5))):
            t = time.time()
            v, e = Q.integrate_product(lat, nus, threads=threads)
            rec[key] = v
            rec[key + "_err"] = e
            rec[key + "_seconds"] = time.time() - t
            print(name, key, v, e, time.time() - t, flush=True)
        rec["atm"] = rec["z333"] / 24 - 3 * rec["zm155"] / 16 + 3 * rec["z135"] / 8
        out[name] = rec
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--slow", action="store_true")
    ap.add_argument("--near-d", action="store_true")
    ap.add_argument("--taylor", action="store_true")
    ap.add_argument("--atm-generic", action="store_true")
    ap.add_argument("--threads", type=int, default=os.cpu_count() or 1)
    args = ap.parse_args()
    ref = load_reference()
    if args.slow:
        res = slow(ref, args.threads)
        path = os.path.join(HERE, "golden_integrals.json")
    elif args.atm_generic:
        res = atm_generic(ref, args.threads)
        path = os.path.join(HERE, "golden_atm_generic.json")
    elif args.taylor:
        res = taylor_high(ref)
        path = os.path.join(HERE, "golden_taylor.json")
    elif args.near_d:
        res = near_d(ref, args.threads)
        path = os.path.join(HERE, "golden_near_d.json")
    else:
        res = quick(ref)
        path = os.path.join(HERE, "golden.json")
    with open(path, "w") as f:
        json.dump(res, f, indent=1)
    print("wrote", path)


if __name__ == "__main__":
    main()
