"""Brillouin-zone quadrature of zeta products — drop-in for L/quadrature.py.

``V int_BZ prod_i Z(nu_i, k) dk = 2^d sum_cells int u^(d-1) prod_i Z(nu_i, u w(v)) du dv``
with the reference's Duffy decomposition (L/quadrature.py:1-27, 136-177):
2^(d-1) d cells, directions ``w = A^{-T} sigma^j (2 p v, 1)^T`` and tensor
Gauss-Legendre angular nodes on [0, 1/2]^(d-1).

B200 design: instead of the reference's host-driven adaptive Gauss-Kronrod
rounds (each a small batch of zeta calls), the radial integral uses a fixed
Gauss-Legendre rule in ``t`` with optional grading ``u = t^q / 2`` (q = 3 tames
the log^3 singularities of 3-D products).  The whole node set is generated on
the device; every distinct exponent is evaluated once per node and raised to
its multiplicity; 256-node tiles reduce to slot-disjoint partials that shard
across GPUs with one all-reduce (see distributed.py).  Results agree with the
reference's adaptive values to ~1e-14 at the BASELINE grid sizes.
"""
from __future__ import annotations

import ctypes as C
import math
import os
from collections import Counter
from dataclasses import dataclass
from functools import lru_cache

import numpy as np

from . import _native as N
from .epstein import TRIVIAL, EpsteinContext, epstein_context
from .errors import PoleError
from .lattice import Lattice

_POLE_TOL = 1e-10


@dataclass(frozen=True)
class QuadratureConfig:
    """Tuning knobs (L/quadrature.py:82-133) plus the fixed-grid fields of the B200 path."""

    gauss_order: int = 14
    epsilon: float = 1.0 / 16.0
    taylor_order: int = 8
    adaptive_rel_tol: float = 1e-13
    adaptive_max_depth: int = 40
    force_integral: bool = False
    allow_high_log_power: bool = False
    splitting: float | None = None
    # fixed Duffy grid of the device path
    grid_u: int = 64
    grid_v: int = 64
    grading: int = 1
    estimate_error: bool = True
    # "auto": fixed device grid when every exponent exceeds d, else the adaptive path;
    # "grid": fixed device grid (continuation tail on the host for nu <= d);
    # "adaptive": the reference's GK15/G7 strategy with GPU panel evaluation
    method: str = "auto"

    def __post_init__(self):
        if not 0.0 < self.epsilon < 0.5:
            raise ValueError("epsilon must lie in (0, 1/2)")
        if self.gauss_order < 2:
            raise ValueError("gauss_order must be at least 2")
        if self.taylor_order % 2 != 0 or self.taylor_order < 0:
            raise ValueError("taylor_order must be a nonnegative even integer")
        if self.grid_u < 2 or self.grid_v < 1 or self.grading < 1:
            raise ValueError("grid_u >= 2, grid_v >= 1 and grading >= 1 required")
        if self.method not in ("auto", "grid", "adaptive"):
            raise ValueError("method must be 'auto', 'grid' or 'adaptive'")

    _INT = ("gauss_order", "taylor_order", "adaptive_max_depth", "grid_u", "grid_v", "grading")
    _FLOAT = ("epsilon", "adaptive_rel_tol", "splitting")
    _BOOL = ("force_integral", "allow_high_log_power", "estimate_error")
    _STR = ("method",)

    def to_text(self) -> str:
        keys = ("gauss_order", "epsilon", "taylor_order", "adaptive_rel_tol", "adaptive_max_depth",
                "force_integral", "allow_high_log_power", "grid_u", "grid_v", "grading",
                "estimate_error", "method")
        out = []
        for k in keys:
            v = getattr(self, k)
            out.append(f"{k}={v!r}" if isinstance(v, float) else f"{k}={v}")
        if self.splitting is not None:
            out.append(f"splitting={self.splitting!r}")
        return "\n".join(out)

    @classmethod
    def from_text(cls, text: str) -> "QuadratureConfig":
        kwargs = {}
        for line in text.replace(",", "\n").splitlines():
            line = line.strip()
            if not line or line.startswith("#"):
                continue
            key, _, value = line.partition("=")
            key, value = key.strip(), value.strip()
            if key in cls._INT:
                kwargs[key] = int(value)
            elif key in cls._FLOAT:
                kwargs[key] = float(value)
            elif key in cls._BOOL:
                kwargs[key] = value.lower() in ("1", "true", "yes")
            elif key in cls._STR:
                kwargs[key] = value
            else:
                raise ValueError(f"unknown config key {key!r}")
        return cls(**kwargs)


@dataclass(frozen=True)
class DuffyCell:
    """One sign pattern and pyramid of the Duffy decomposition (L/quadrature.py:136-152)."""

    signs: tuple
    pyramid: int

    def directions(self, lattice: Lattice, v: np.ndarray) -> np.ndarray:
        d = lattice.d
        v = np.atleast_2d(v)
        t = np.empty((max(len(v), 1), d))
        if d > 1:
            t[:, :-1] = 2.0 * np.asarray(self.signs) * v
        t[:, -1] = 1.0
        return np.roll(t, self.pyramid, axis=1) @ lattice.a_inv_t.T


def duffy_cells(d: int):
    """All 2^(d-1) d cells, signs outer and pyramid inner (L/quadrature.py:155-162)."""
    cells = []
    for signs in np.ndindex(*([2] * (d - 1))):
        p = tuple(1.0 if s == 0 else -1.0 for s in signs)
        cells.extend(DuffyCell(p, j) for j in range(d))
    return cells


def angular_nodes(d: int, order: int):
    """Tensor Gauss-Legendre nodes and weights on [0, 1/2]^(d-1) (L/quadrature.py:165-177)."""
    if d == 1:
        return np.zeros((1, 0)), np.ones(1)
    x, w = np.polynomial.legendre.leggauss(order)
    v1, w1 = (x + 1.0) / 4.0, w / 4.0
    v = np.stack([g.ravel() for g in np.meshgrid(*([v1] * (d - 1)), indexing="ij")], axis=-1)
    wts = np.ones(len(v))
    for g in np.meshgrid(*([w1] * (d - 1)), indexing="ij"):
        wts = wts * g.ravel()
    return v, wts


def tail_primitive(nu: float, m: int, eps: float, wsq, allow_high_log_power: bool = False):
    """Continuation value of int_0^eps u^(-nu-1) log^m(pi u^2 w^2) du (L/quadrature.py:274-296)."""
    if m < 0:
        raise ValueError("log power must be nonnegative")
    if m > 3 and not allow_high_log_power:
        raise NotImplementedError("log powers above 3 require allow_high_log_power (general recurrence)")
    if abs(nu) < _POLE_TOL:
        raise PoleError(f"tail integral diverges: net power u^-1 with log^{m}")
    wsq = np.asarray(wsq, dtype=float)
    ell = np.log(math.pi * eps * eps * wsq)
    epow = eps ** (-nu)
    acc = -epow / nu * np.ones_like(wsq)
    for j in range(1, m + 1):
        acc = -epow * ell ** j / nu + (2.0 * j / nu) * acc
    return acc


# ---------------------------------------------------------------------------------
# Device plans

class Plan:
    """A fused device plan (product of distinct zetas, or the ATM integrand)."""

    def __init__(self, handle, d: int, ncomp: int, keepalive):
        self._h = handle
        self.d = d
        self.ncomp = ncomp
        self._keep = keepalive  # contexts must outlive the plan

    def __del__(self):
        try:  # also reached at interpreter shutdown, when module globals may be gone
            h = getattr(self, "_h", None)
            if h is not None and N is not None and N._lib is not None:
                N._lib.lz_plan_destroy(h)
        except Exception:
            pass

    @property
    def handle(self):
        return self._h

    def info(self) -> "N.PlanInfo":
        out = N.PlanInfo()
        N.check(N.lib().lz_plan_get_info(self._h, C.byref(out)), "plan info")
        return out

    def tiles(self, n_u: int, n_v: int, grading: int):
        g = N.Grid(n_u, n_v, grading, 0, 0)
        nn, nt = C.c_int64(0), C.c_int64(0)
        N.check(N.lib().lz_grid_tiles(self.d, C.byref(g), C.byref(nn), C.byref(nt)), "grid")
        return nn.value, nt.value

    def integrate(self, n_u: int, n_v: int, grading: int, u_lo: float = 0.0) -> np.ndarray:
        """Sum over all nodes (before the 2^d factor), through host memory."""
        N.require_cuda("BZ quadrature")
        g = N.Grid(n_u, n_v, grading, 0, 0, float(u_lo))
        out = np.zeros(self.ncomp, dtype=np.float64)
        N.check(N.lib().lz_plan_integrate_host(self._h, C.byref(g), N.dptr(out)), "integral")
        return out

    def integrate_device(self, partials, n_u: int, n_v: int, grading: int, tile_lo: int = 0,
                         tile_hi: int = 0, stream=None, grid_blocks: int = 0, u_lo: float = 0.0):
        """Write the tile partials of [tile_lo, tile_hi) into a CUDA tensor (n_tiles x ncomp)."""
        import torch
        g = N.Grid(n_u, n_v, grading, tile_lo, tile_hi, float(u_lo))
        st = stream if stream is not None else torch.cuda.current_stream(partials.device).cuda_stream
        N.check(N.lib().lz_plan_integrate(self._h, C.byref(g), partials.data_ptr(), grid_blocks, st),
                "integral")

    @staticmethod
    def reduce_device(partials, n_tiles: int, ncomp: int, out, stream=None):
        import torch
        st = stream if stream is not None else torch.cuda.current_stream(partials.device).cuda_stream
        N.check(N.lib().lz_reduce_partials(partials.data_ptr(), n_tiles, ncomp, out.data_ptr(), st),
                "reduce")


@lru_cache(maxsize=256)
def product_plan(lattice: Lattice, nus_key: tuple, splitting: float | None = None) -> Plan:
    """Plan for prod_j Z_{nu_j}^{m_j}; ``nus_key`` = ((nu, m), ...) of distinct exponents."""
    ctxs = [epstein_context(lattice, nu, splitting) for nu, _ in nus_key]
    arr = (C.c_void_p * len(ctxs))(*[c.handle for c in ctxs])
    mult = (C.c_int * len(ctxs))(*[m for _, m in nus_key])
    h = C.c_void_p()
    N.check(N.lib().lz_plan_create_product(arr, mult, len(ctxs), C.byref(h)), "product plan")
    return Plan(h, lattice.d, 1, ctxs)


# Theta-split used by the fused ATM plan, as a multiple of the reference's V^(-2/d)
# (L/epstein.py:107).  The lattice sum is split-invariant; a smaller split moves work from the
# reciprocal sum (table lookups, ~64 instructions per term) to the direct sum (phase rotations,
# ~18 per point).  Measured on B200: see DESIGN.md section 3.2.
ATM_SPLIT_SCALE = float(os.environ.get("LATSUM_ATM_SPLIT_SCALE", "0.13"))


@lru_cache(maxsize=64)
def atm_plan(lattice: Lattice, splitting: float | None = None) -> Plan:
    """Plan for the ATM integrand [Z_3^3, tr(M_5^3)], M_5 = polynomial-weighted zeta at nu = 5."""
    if splitting is None and ATM_SPLIT_SCALE != 1.0:
        splitting = ATM_SPLIT_SCALE * lattice.volume ** (-2.0 / lattice.d)
    # the two contexts' host enumerations are independent native calls (GIL released): overlap them
    from concurrent.futures import ThreadPoolExecutor
    # Both contexts are private to this (cached) plan and enumerate only what it reads: Z_3 lends
    # its constants and reciprocal set (the kernel takes Z_3 = tr M_5), Z_5 its constants and the
    # Hessian's widened point sets
    with ThreadPoolExecutor(max_workers=2) as pool:
        f5 = pool.submit(EpsteinContext, lattice, 5.0, splitting, -2)
        z3 = EpsteinContext(lattice, 3.0, splitting, deriv_order=-1)
        z5 = f5.result()
    h = C.c_void_p()
    N.check(N.lib().lz_plan_create_atm(z3.handle, z5.handle, C.byref(h)), "atm plan")
    return Plan(h, lattice.d, 2, (z3, z5))


def _distinct(contexts):
    """Group identical exponents: [(nu, multiplicity)] in first-appearance order, plus the
    constant factor of trivial-branch exponents."""
    const = 1.0
    counts = Counter()
    order = []
    for ctx in contexts:
        if ctx.branch == TRIVIAL:
            const *= ctx.const_value
            continue
        if ctx.nu not in counts:
            order.append(ctx.nu)
        counts[ctx.nu] += 1
    return [(nu, counts[nu]) for nu in order], const


def fixed_grid_integral(lattice: Lattice, nus, n_u: int, n_v: int, grading: int = 1,
                        splitting: float | None = None) -> float:
    """2^d * sum over the fixed Duffy grid of u^(d-1) prod Z (all exponents must exceed d)."""
    contexts = [epstein_context(lattice, float(nu), splitting) for nu in nus]
    groups, const = _distinct(contexts)
    if const == 0.0:
        return 0.0
    if not groups:
        return const * float(2.0 ** lattice.d * _grid_weight_sum(lattice.d, n_u, n_v, grading))
    if len(groups) > 4:
        raise ValueError("at most 4 distinct exponents per product kernel")
    plan = product_plan(lattice, tuple(groups), splitting)
    s = plan.integrate(n_u, n_v, grading)[0]
    return const * (2.0 ** lattice.d) * s


def _grid_weight_sum(d, n_u, n_v, grading):
    # integral of u^(d-1) over the Duffy cells = V * |BZ box| / 2^d in fractional coords = 1/2^d
    return 1.0 / 2.0 ** d


def integrate_product(lattice: Lattice, nus, cfg: QuadratureConfig | None = None, threads: int = 1):
    """Duffy-decomposed ``V int_BZ prod_i Z(nu_i, k) dk`` (L/quadrature.py:455-490).

    Returns (value, error_estimate).  All exponents above the dimension: fixed
    graded Gauss-Legendre grid on the GPU; the error estimate is the difference
    to a 3/4-resolution grid.  Exponents at or below the dimension need the
    meromorphic-continuation tail path (next rows).
    ``threads`` is accepted for signature compatibility; the GPU does the work.
    """
    cfg = cfg or QuadratureConfig()
    nus = [float(x) for x in nus]
    d = lattice.d
    contexts = [epstein_context(lattice, nu, cfg.splitting) for nu in nus]
    min_nu = min(ctx.nu for ctx in contexts if ctx.branch != TRIVIAL) if any(
        c.branch != TRIVIAL for c in contexts) else math.inf
    if cfg.method == "adaptive" or (cfg.method == "auto" and min_nu <= d):
        N.require_cuda("BZ quadrature")
        from .adaptive import integrate_product_adaptive
        return integrate_product_adaptive(lattice, contexts, cfg)
    if min_nu <= d:
        from .tail import integrate_product_continued
        return integrate_product_continued(lattice, contexts, cfg)
    value = fixed_grid_integral(lattice, nus, cfg.grid_u, cfg.grid_v, cfg.grading, cfg.splitting)
    err = 0.0
    if cfg.estimate_error:
        coarse = fixed_grid_integral(lattice, nus, max(2, (3 * cfg.grid_u) // 4),
                                     max(1, (3 * cfg.grid_v) // 4), cfg.grading, cfg.splitting)
        err = abs(value - coarse)
    return value, err


def integrate_bz_even(lattice: Lattice, fvec, cfg: QuadratureConfig | None = None):
    """``V int_BZ f(k) dk`` for an even integrand given as a k-batch callable (L/quadrature.py:493-515).

    Test utility: ``fvec`` is a host callable, so the node weights are formed on the host.
    """
    cfg = cfg or QuadratureConfig()
    d = lattice.d
    x, w = np.polynomial.legendre.leggauss(cfg.grid_u)
    t = (x + 1.0) / 2.0
    u = 0.5 * t ** cfg.grading
    wu = (w / 2.0) * 0.5 * cfg.grading * t ** (cfg.grading - 1) * u ** (d - 1)
    v, wv = angular_nodes(d, cfg.grid_v if d > 1 else 1)
    total = []
    for cell in duffy_cells(d):
        wdir = cell.directions(lattice, v)
        k = (u[:, None, None] * wdir[None, :, :]).reshape(-1, d)
        f = np.asarray(fvec(k), dtype=float).reshape(len(u), len(wdir))
        total.append(math.fsum((wu[:, None] * f * wv[None, :]).ravel()))
    return 2.0 ** d * math.fsum(total)
