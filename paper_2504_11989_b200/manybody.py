"""Many-body zeta functions and the ATM cohesive energy.

The reference package declares these in its SPEC but does not ship them; the
reference's nearest code is ``integrate_product`` (L/quadrature.py:455-490)
plus the Prop. 2.4 recombination

    E_ATM = zeta(3,3,3)/24 - 3 zeta(-1,5,5)/16 + 3 zeta(1,3,5)/8 .

The B200 path evaluates the same energy without meromorphic continuation, as
one absolutely convergent BZ integral of zeta values and polynomial-weighted
zetas (the north star's "dot-product term via polynomial-weighted zeta"):

    E_ATM = (V/6) int_BZ [ Z_3(k)^3 - 3 tr(M(k)^3) ] dk,
    M_ab(k) = sum'_z z_a z_b |z|^-5 e^{-2 pi i z.k} = -d_a d_b Z_5(k) / (4 pi^2),

because sum_{x+y+z=0} (x.y)(y.z)(z.x) |x|^-5|y|^-5|z|^-5 = V int tr(M^3) and the
ATM cosine product equals -(d1.d2)(d2.d3)(d3.d1)/(r1^2 r2^2 r3^2) for the
three side vectors of a triangle.  One fused kernel produces both integrands
per node (csrc/kernels.cu, tile_kernel MODE 1).
"""
from __future__ import annotations

import time
from dataclasses import dataclass, field

from .epstein import epstein_context
from .lattice import Lattice
from .quadrature import QuadratureConfig, atm_plan, integrate_product


@dataclass
class ManyBodyResult:
    value: float
    error_estimate: float
    n: int
    lattice: Lattice
    nu: tuple
    config: QuadratureConfig
    wall_time: float = 0.0


def many_body_zeta(lattice: Lattice, nus, cfg: QuadratureConfig | None = None) -> ManyBodyResult:
    """zeta^(n)(nu) = V int_BZ prod Z (Theorem 2.6), with the Cor. 2.7 short-circuits."""
    cfg = cfg or QuadratureConfig()
    nus = tuple(float(x) for x in nus)
    n = len(nus)
    if n < 1:
        raise ValueError("need at least one exponent")
    t0 = time.perf_counter()
    if n == 1 and not cfg.force_integral:
        value, err = 0.0, 0.0
    elif n == 2 and not cfg.force_integral:
        value, err = epstein_context(lattice, nus[0] + nus[1], cfg.splitting).zeta_at_zero(), 0.0
    else:
        value, err = integrate_product(lattice, nus, cfg)
    return ManyBodyResult(value, err, n, lattice, nus, cfg, time.perf_counter() - t0)


def normalized_many_body(lattice: Lattice, nu: float, n: int, cfg: QuadratureConfig | None = None) -> float:
    """zeta^(n)(nu, ..., nu) / Z_nu(0)^n (PAPER §4.3); |value| <= 1 for nu > d."""
    if nu <= lattice.d:
        raise ValueError("normalized many-body zeta requires nu > d")
    z0 = epstein_context(lattice, float(nu)).zeta_at_zero()
    return many_body_zeta(lattice, [nu] * n, cfg).value / z0 ** n


def table_square(n_list=(2, 3, 4, 5, 6, 7, 8), nu_list=(2.0, 3.0), cfg: QuadratureConfig | None = None):
    """Table 1 of the paper (SPEC.md: table_square): zeta^(n)(nu, ..., nu) on the square lattice.

    Rows (n, nu, value, error_estimate); nu = 2 = d runs through the continuation path."""
    from .lattice import named_lattice
    sq = named_lattice("square")
    rows = []
    for nu in nu_list:
        for n in n_list:
            res = many_body_zeta(sq, [nu] * n, cfg)
            rows.append((n, float(nu), res.value, res.error_estimate))
    return rows


@dataclass(frozen=True)
class ATMGrid:
    """Fixed Duffy grid of the ATM integral: n_u radial (graded u = t^q/2) x n_v^(d-1) angular."""

    n_u: int = 128
    n_v: int = 128
    grading: int = 3


@dataclass
class ATMResult:
    energy: float        # E_ATM = (V/6) int [Z3^3 - 3 tr M^3]
    zeta333: float       # zeta^(3)(3,3,3) = V int Z3^3
    dot_term: float      # D = V int tr(M^3)
    grid: ATMGrid = field(default_factory=ATMGrid)
    nodes: int = 0
    wall_time: float = 0.0


def atm_integrals(lattice: Lattice, grid: ATMGrid | None = None, splitting: float | None = None) -> ATMResult:
    """Both ATM integrands on the fixed Duffy grid in one GPU pass."""
    grid = grid or ATMGrid()
    d = lattice.d
    if d not in (1, 2, 3):
        raise ValueError("the ATM sum converges absolutely only for d in {1, 2, 3}")
    t0 = time.perf_counter()
    plan = atm_plan(lattice, splitting)
    s = plan.integrate(grid.n_u, grid.n_v, grid.grading)
    scale = 2.0 ** d
    z333 = scale * s[0]
    dot = scale * s[1]
    nodes, _ = plan.tiles(grid.n_u, grid.n_v, grid.grading)
    return ATMResult((z333 - 3.0 * dot) / 6.0, z333, dot, grid, nodes, time.perf_counter() - t0)


def atm_cohesive_energy(lattice: Lattice, cfg: QuadratureConfig | None = None,
                        grid: ATMGrid | None = None) -> float:
    """ATM three-body cohesive energy (Def. 1.1 / Prop. 2.4)."""
    if cfg is not None and grid is None:
        grid = ATMGrid(n_u=cfg.grid_u, n_v=cfg.grid_v, grading=max(cfg.grading, 3))
    return atm_integrals(lattice, grid, cfg.splitting if cfg else None).energy


def atm_energy_scaled(lattice: Lattice, scale: float, **kw) -> float:
    """Homogeneity check helper: E_ATM(s Lambda) = E_ATM(Lambda) / s^9."""
    return atm_cohesive_energy(lattice.scaled(scale), **kw)


__all__ = ["ManyBodyResult", "many_body_zeta", "normalized_many_body", "table_square", "ATMGrid", "ATMResult",
           "atm_integrals", "atm_cohesive_energy", "atm_energy_scaled"]
