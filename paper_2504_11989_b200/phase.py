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


def optimize_scale(c: LatticeConstants, lj: LJParams, lam: float, p: float,
                   r_grid=None, tol: float = 1e-13):
    """Global minimum of H(R): best point of a coarse grid, then golden-section refinement."""
    if r_grid is None:
        r_grid = np.linspace(0.5, 3.0, 200)
    r_grid = np.asarray(r_grid, dtype=float)
    h = total_enthalpy(c, lj, lam, p, r_grid)
    i = int(np.argmin(h))
    if i == 0 or i == len(r_grid) - 1:
        raise ValueError("enthalpy minimum hits the R bracket boundary")
    a, b = r_grid[i - 1], r_grid[i + 1]
    x1 = b - _GOLD * (b - a)
    x2 = a + _GOLD * (b - a)
    f1 = float(total_enthalpy(c, lj, lam, p, x1))
    f2 = float(total_enthalpy(c, lj, lam, p, x2))
    while b - a > tol * max(1.0, abs(a)):
        if f1 < f2:
            b, x2, f2 = x2, x1, f1
            x1 = b - _GOLD * (b - a)
            f1 = float(total_enthalpy(c, lj, lam, p, x1))
        else:
            a, x1, f1 = x1, x2, f2
            x2 = a + _GOLD * (b - a)
            f2 = float(total_enthalpy(c, lj, lam, p, x2))
    r = 0.5 * (a + b)
    return r, float(total_enthalpy(c, lj, lam, p, r))


def _delta_h(fcc, bcc, lj, lam, p, r_grid):
    return optimize_scale(fcc, lj, lam, p, r_grid)[1] - optimize_scale(bcc, lj, lam, p, r_grid)[1]


def phase_scan(fcc: LatticeConstants, bcc: LatticeConstants, lj: LJParams, p_grid, lam_grid,
               r_grid=None):
    """Winner of min_R H for every (p, lambda) of the grids, ordered by (p, lambda)."""
    pts = []
    for p in p_grid:
        for lam in lam_grid:
            rf, hf = optimize_scale(fcc, lj, float(lam), float(p), r_grid)
            rb, hb = optimize_scale(bcc, lj, float(lam), float(p), r_grid)
            pts.append(PhasePoint(float(p), float(lam), "fcc" if hf <= hb else "bcc", rf, rb, hf, hb))
    return pts


def critical_coupling(fcc: LatticeConstants, bcc: LatticeConstants, lj: LJParams, p: float,
                      lam_grid=None, r_grid=None, tol: float = 1e-14):
    """lambda_c(p): first fcc -> bcc sign change of min_R H_fcc - min_R H_bcc on the lambda
    grid, refined by bisection (SPEC.md: 'bisection on lambda ... between bracketing points')."""
    if lam_grid is None:
        lam_grid = np.linspace(0.0, 2.0, 64)
    vals = [_delta_h(fcc, bcc, lj, float(l), p, r_grid) for l in lam_grid]
    for i in range(len(lam_grid) - 1):
        if vals[i] <= 0.0 < vals[i + 1]:
            a, b = float(lam_grid[i]), float(lam_grid[i + 1])
            fa = vals[i]
            while b - a > tol:
                mid = 0.5 * (a + b)
                fm = _delta_h(fcc, bcc, lj, mid, p, r_grid)
                if (fm <= 0.0) == (fa <= 0.0):
                    a, fa = mid, fm
                else:
                    b = mid
            return 0.5 * (a + b)
    return math.nan


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
