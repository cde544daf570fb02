"""Lennard-Jones + ATM stability of fcc vs bcc (PAPER §5).

Host arithmetic on a handful of lattice constants that the GPU produces once
per lattice: Z_{Lambda,n}(0), Z_{Lambda,m}(0) (zeta_at_zero) and the ATM
constant K_Lambda = E_ATM(Lambda_unit) (the fused ATM integral).  The enthalpy
per particle at nearest-neighbour distance R is

    H(R) = nm/(2(n-m)) (Z_n(0)/(n R^n) - Z_m(0)/(m R^m)) + lambda K / R^9 + p V_unit R^3

with Z_m(0) in the second term (the paper prints Z_n there).
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

_GOLD = (math.sqrt(5.0) - 1.0) / 2.0


@dataclass(frozen=True)
class LJParams:
    n: float = 12.0
    m: float = 6.0


@dataclass(frozen=True)
class LatticeConstants:
    """Per-structure constants of the scan (unit nearest-neighbour distance)."""

    name: str
    z_n: float       # Z_{Lambda,n}(0)
    z_m: float       # Z_{Lambda,m}(0)
    k_atm: float     # E_ATM(Lambda_unit)
    v_unit: float    # volume per particle at R = 1


@dataclass(frozen=True)
class PhasePoint:
    p: float
    lam: float
    winner: str
    r_fcc: float
    r_bcc: float
    h_fcc: float
    h_bcc: float


def lj_cohesive(c: LatticeConstants, lj: LJParams, r):
    n, m = lj.n, lj.m
    r = np.asarray(r, dtype=float)
    return n * m / (2.0 * (n - m)) * (c.z_n / (n * r ** n) - c.z_m / (m * r ** m))


def total_enthalpy(c: LatticeConstants, lj: LJParams, lam: float, p: float, r):
    r = np.asarray(r, dtype=float)
    return lj_cohesive(c, lj, r) + lam * c.k_atm / r ** 9 + p * c.v_unit * r ** 3


def _enthalpy_derivs(c, lj, lam, p, r):
    """dH/dR and d2H/dR2 of total_enthalpy (closed form)."""
    n, m = lj.n, lj.m
    pre = n * m / (2.0 * (n - m))
    a_, b_ = pre * c.z_n / n, pre * c.z_m / m        # H = a R^-n - b R^-m + lam K R^-9 + p V R^3
    k_, v_ = lam * c.k_atm, p * c.v_unit
    d1 = -n * a_ * r ** (-n - 1) + m * b_ * r ** (-m - 1) - 9.0 * k_ * r ** -10 + 3.0 * v_ * r ** 2
    d2 = (n * (n + 1) * a_ * r ** (-n - 2) - m * (m + 1) * b_ * r ** (-m - 2) + 90.0 * k_ * r ** -11
          + 6.0 * v_ * r)
    return d1, d2


def _golden_min(c, lj, lam, p, r_grid, tol=1e-13, iters=12):
    """Vectorised global minimum of H(R) over R for arrays of (lambda, p): best point of the R grid,
    then safeguarded Newton on dH/dR = 0 inside the bracketing grid cells (quadratic convergence;
    a golden-section step replaces any Newton step that leaves the bracket)."""
    lam = np.asarray(lam, dtype=float)
    p = np.asarray(p, dtype=float)
    lam, p = np.broadcast_arrays(lam, p)
    r_grid = np.asarray(r_grid, dtype=float)
    h = total_enthalpy(c, lj, lam[..., None], p[..., None], r_grid)
    i = np.argmin(h, axis=-1)
    if np.any((i == 0) | (i == len(r_grid) - 1)):
        raise ValueError("enthalpy minimum hits the R bracket boundary")
    lo, hi = r_grid[i - 1], r_grid[i + 1]
    r = r_grid[i].astype(float)
    active = np.ones(r.shape, dtype=bool)
    for _ in range(iters + 40):
        d1, d2 = _enthalpy_derivs(c, lj, lam, p, r)
        step = np.where(d2 > 0.0, d1 / np.where(d2 > 0.0, d2, 1.0), 0.0)
        rn = r - step
        bad = (d2 <= 0.0) | (rn <= lo) | (rn >= hi)
        rn = np.where(bad, np.where(d1 > 0.0, lo + _GOLD * (r - lo), r + (1.0 - _GOLD) * (hi - r)), rn)
        # shrink the bracket around the root of dH/dR (converged entries are frozen)
        lo = np.where(active & (d1 <= 0.0), np.maximum(lo, r), lo)
        hi = np.where(active & (d1 > 0.0), np.minimum(hi, r), hi)
        done = np.abs(rn - r) <= tol * np.abs(r)
        r = np.where(active, rn, r)
        active &= ~done
        if not np.any(active):
            break
    return r, total_enthalpy(c, lj, lam, p, r)


def optimize_scale(c: LatticeConstants, lj: LJParams, lam: float, p: float,
                   r_grid=None, tol: float = 1e-13):
    """Global minimum of H(R): best point of a coarse grid, then golden-section refinement
    (SPEC.md: optimize_scale).  Returns (R*, H*)."""
    if r_grid is None:
        r_grid = np.linspace(0.5, 3.0, 200)
    r, h = _golden_min(c, lj, lam, p, r_grid, tol)
    return float(r), float(h)


def phase_scan(fcc: LatticeConstants, bcc: LatticeConstants, lj: LJParams, p_grid, lam_grid,
               r_grid=None):
    """Winner of min_R H for every (p, lambda) of the grids, ordered by (p, lambda)."""
    if r_grid is None:
        r_grid = np.linspace(0.5, 3.0, 200)
    P, L = np.meshgrid(np.asarray(p_grid, float), np.asarray(lam_grid, float), indexing="ij")
    rf, hf = _golden_min(fcc, lj, L, P, r_grid)
    rb, hb = _golden_min(bcc, lj, L, P, r_grid)
    pts = []
    for idx in np.ndindex(P.shape):
        pts.append(PhasePoint(float(P[idx]), float(L[idx]), "fcc" if hf[idx] <= hb[idx] else "bcc",
                              float(rf[idx]), float(rb[idx]), float(hf[idx]), float(hb[idx])))
    return pts


def critical_coupling(fcc: LatticeConstants, bcc: LatticeConstants, lj: LJParams, p,
                      lam_grid=None, r_grid=None, tol: float = 1e-14):
    """lambda_c(p): first fcc -> bcc sign change of min_R H_fcc - min_R H_bcc on the lambda grid,
    refined inside the bracketing points (SPEC.md: 'bisection on lambda ... between bracketing
    points') by safeguarded Newton with the envelope-theorem slope K_fcc/R_fcc^9 - K_bcc/R_bcc^9,
    falling back to bisection.
    ``p`` may be a scalar or an array (vectorised over pressures)."""
    if lam_grid is None:
        lam_grid = np.linspace(0.0, 2.0, 64)
    if r_grid is None:
        r_grid = np.linspace(0.5, 3.0, 200)
    scalar = np.ndim(p) == 0
    p = np.atleast_1d(np.asarray(p, float))
    lam_grid = np.asarray(lam_grid, float)

    def delta(lam, pp):
        return _golden_min(fcc, lj, lam, pp, r_grid)[1] - _golden_min(bcc, lj, lam, pp, r_grid)[1]

    def delta_d(lam, pp):
        # envelope theorem: d/dlambda min_R H(R; lambda) = K / R*^9 at the minimiser
        rf, hf = _golden_min(fcc, lj, lam, pp, r_grid)
        rb, hb = _golden_min(bcc, lj, lam, pp, r_grid)
        return hf - hb, fcc.k_atm / rf ** 9 - bcc.k_atm / rb ** 9

    dv = delta(lam_grid[None, :], p[:, None])
    out = np.full(len(p), np.nan)
    flip = (dv[:, :-1] <= 0.0) & (dv[:, 1:] > 0.0)
    has = flip.any(axis=1)
    first = np.argmax(flip, axis=1)
    a = lam_grid[first].astype(float)
    b = lam_grid[np.minimum(first + 1, len(lam_grid) - 1)].astype(float)
    # safeguarded Newton on delta(lambda) = 0 inside the sign-change bracket (bisection fallback)
    lam = 0.5 * (a + b)
    for _ in range(100):
        fm, dm = delta_d(lam, p)
        a = np.where(fm <= 0.0, lam, a)
        b = np.where(fm <= 0.0, b, lam)
        step = np.where(dm != 0.0, fm / np.where(dm != 0.0, dm, 1.0), 0.0)
        nxt = lam - step
        bad = ~((nxt > a) & (nxt < b)) | (dm == 0.0)
        nxt = np.where(bad, 0.5 * (a + b), nxt)
        done = (np.abs(nxt - lam) <= tol) | (b - a <= tol)
        lam = nxt
        if np.all(done):
            break
    a = b = lam
    out[has] = 0.5 * (a + b)[has]
    return float(out[0]) if scalar else out


def lattice_constants(name: str, lj: LJParams = LJParams(), atm_grid=None) -> LatticeConstants:
    """Compute a structure's constants on the GPU (two zeta_at_zero + one fused ATM integral)."""
    from .epstein import epstein_context
    from .lattice import named_lattice
    from .manybody import atm_integrals
    lat = named_lattice(name)
    z_n = epstein_context(lat, lj.n).zeta_at_zero()
    z_m = epstein_context(lat, lj.m).zeta_at_zero()
    k = atm_integrals(lat, atm_grid).energy
    return LatticeConstants(name, z_n, z_m, k, lat.volume)
