"""Meromorphic-continuation path of integrate_product for exponents nu <= d.

Reference algorithm (L/quadrature.py:274-452): split the radial
integral at epsilon.  Near u = 0 every factor is its explicit singularity plus
the Taylor polynomial of Z_reg along the ray, so u^(d-1) prod_i Z(nu_i, u w) is
a finite sum of monomials c(w) u^eta log^m(pi u^2 |w|^2) whose integrals over
(0, epsilon) have closed forms -- for eta <= -1 these closed forms ARE the
analytic continuation.  The outer part (epsilon, 1/2) is a regular integral.

B200 split of the work:
  * outer part: the fused product kernel on a device-generated Gauss-Legendre
    grid with u in (epsilon, 1/2) (lz_grid.u_lo); the integrand is analytic on
    the closed interval (its singularity sits at u = 0, a distance epsilon
    away), so the fixed rule converges geometrically and needs none of the
    reference's monomial subtraction, which only served its adaptive error
    control;
  * inner part: closed-form host algebra per direction (tiny: a few hundred
    monomials times the number of directions), from the native Taylor tables.
"""
from __future__ import annotations

import math
import warnings

import numpy as np

from .epstein import GENERIC, LOG_CASE, TRIVIAL
from .errors import ConvergenceError, TruncationWarning

_KEY_DIGITS = 9
_PRUNE = 1e-20
_EXTRA_ORDER = 2
_TERM_BUDGET = 200_000


def _ray_expansion(ctx, taylor, w, wsq, ell):
    """Monomials of Z(nu, u w) for small u: {(exponent, log power): coefficients over rows of w}."""
    d = ctx.d
    out = {}
    if ctx.branch == GENERIC and ctx.singular_coef() != 0.0:
        out[(round(ctx.nu - d, _KEY_DIGITS), 0)] = ctx.singular_coef() * wsq ** ((ctx.nu - d) / 2.0) / ctx.vol
    elif ctx.branch == LOG_CASE:
        m = ctx.log_m
        out[(float(2 * m), 1)] = ctx.singular_coef() * wsq ** m / ctx.vol
    for j in range(ell // 2 + 1):
        key = (float(2 * j), 0)
        c = taylor.directional_coeff(w, j)
        out[key] = out[key] + c if key in out else c
    return out


def _multiply(a, b, cap):
    """Truncated product of two monomial expansions (exponents above ``cap`` dropped)."""
    prod = {}
    for (ea, ma), ca in a.items():
        for (eb, mb), cb in b.items():
            e = round(ea + eb, _KEY_DIGITS)
            if e > cap:
                continue
            key = (e, ma + mb)
            if key in prod:
                prod[key] = prod[key] + ca * cb
            else:
                prod[key] = ca * cb
    if not prod:
        return prod
    scale = max(float(np.max(np.abs(c))) for c in prod.values())
    kept = {k: c for k, c in prod.items() if float(np.max(np.abs(c))) > _PRUNE * scale}
    if len(kept) > _TERM_BUDGET:
        raise ConvergenceError("tail product expansion exploded; reduce taylor_order")
    return kept


def _tail_primitive(nu, m, eps, wsq, allow_high):
    from .quadrature import tail_primitive
    return tail_primitive(nu, m, eps, wsq, allow_high)


def ray_series(contexts, taylors, w, cfg):
    """Monomials of prod_i Z(nu_i, u w) near u = 0 (above the u^(d-1) factor), per row of w."""
    ell = cfg.taylor_order
    wsq = np.einsum("ij,ij->i", w, w)
    series = {(0.0, 0): np.ones(len(w))}
    for ctx, tab in zip(contexts, taylors):
        series = _multiply(series, _ray_expansion(ctx, tab, w, wsq, ell), ell + _EXTRA_ORDER)
    return series


def tail_values(contexts, taylors, w, cfg, series=None):
    """Continuation value of int_0^eps u^(d-1) prod Z(nu_i, u w) du for every row of w."""
    d = contexts[0].d
    ell = cfg.taylor_order
    wsq = np.einsum("ij,ij->i", w, w)
    if series is None:
        series = ray_series(contexts, taylors, w, cfg)
    total = np.zeros(len(w))
    top = np.zeros(len(w))
    for (e, m), c in sorted(series.items()):
        piece = c * _tail_primitive(-(d + e), m, cfg.epsilon, wsq, cfg.allow_high_log_power)
        total += piece
        if e >= ell:
            top += np.abs(piece)
    if np.any(top > cfg.adaptive_rel_tol * np.maximum(np.abs(total), 1e-300) * 1e3):
        warnings.warn("highest retained Taylor order still contributes noticeably; increase "
                      "taylor_order or decrease epsilon", TruncationWarning, stacklevel=3)
    return total


def integrate_product_continued(lattice, contexts, cfg):
    """V int_BZ prod Z (value, error estimate) when some exponent is <= d."""
    from .quadrature import _distinct, angular_nodes, duffy_cells, product_plan
    d = lattice.d
    groups, const = _distinct(contexts)
    if const == 0.0:
        return 0.0, 0.0
    if not groups:
        return const, 0.0  # V int_BZ 1 dk = 1
    live = [c for c in contexts if c.branch != TRIVIAL]
    taylors = [c.reg_derivatives(cfg.taylor_order) for c in live]
    # inner part: closed forms per direction, weighted with the angular rule
    v, wv = angular_nodes(d, cfg.grid_v)
    inner = []
    for cell in duffy_cells(d):
        w = cell.directions(lattice, v)
        inner.append(math.fsum(wv * tail_values(live, taylors, w, cfg)))
    inner_sum = math.fsum(inner)
    # outer part on the GPU: u in (epsilon, 1/2), no grading needed
    if len(groups) > 4:
        raise ValueError("at most 4 distinct exponents per product kernel")
    plan = product_plan(lattice, tuple(groups), cfg.splitting)

    def outer(n_u, n_v):
        return plan.integrate(n_u, n_v, 1, u_lo=cfg.epsilon)[0]

    value = const * 2.0 ** d * (outer(cfg.grid_u, cfg.grid_v) + inner_sum)
    err = 0.0
    if cfg.estimate_error:
        coarse = const * 2.0 ** d * (outer(max(2, 3 * cfg.grid_u // 4), cfg.grid_v) + inner_sum)
        err = abs(value - coarse)
    return value, err
