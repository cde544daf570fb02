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
import itertools
import math
import os
from collections import Counter
from dataclasses import dataclass
from functools import lru_cache

import numpy as np

from . import _native as N
from .epstein import LOG_CASE, TRIVIAL, EpsteinContext, epstein_context
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
    """One (sign pattern, pyramid) piece of the Duffy decomposition of the BZ box
    (semantics of L/quadrature.py:136-152).

    In fractional coordinates the pyramid with apex axis ``a = (pyramid - 1) mod d``
    holds the points ``u * (2 s_0 v_0, ..., 1, ...)`` whose coordinate on axis ``a``
    is ``u`` and whose angular coordinate ``v_i`` sits on axis ``(i + pyramid) mod d``.
    """

    signs: tuple
    pyramid: int

    def directions(self, lattice: Lattice, v: np.ndarray) -> np.ndarray:
        """Cartesian ray directions ``w = A^{-T} f`` for angular rows ``v`` in [0, 1/2]^(d-1)."""
        d = lattice.d
        v = np.asarray(v, dtype=float)
        rows = len(v) if v.ndim == 2 else 1
        frac = np.zeros((max(rows, 1), d))
        frac[:, (self.pyramid - 1) % d] = 1.0
        if d > 1:
            vv = v.reshape(rows, d - 1)
            for i, s in enumerate(self.signs):
                frac[:, (i + self.pyramid) % d] = (2.0 * s) * vv[:, i]
        return frac @ lattice.a_inv_t.T


def duffy_cells(d: int):
    """The 2^(d-1) d cells: sign patterns (+ before -, last sign fastest) outer, pyramids inner
    (ordering of L/quadrature.py:155-162)."""
    return [DuffyCell(tuple(signs), apex)
            for signs in itertools.product((1.0, -1.0), repeat=d - 1)
            for apex in range(d)]


def angular_nodes(d: int, order: int):
    """Tensor Gauss-Legendre rule on [0, 1/2]^(d-1), first axis slowest (L/quadrature.py:165-177)."""
    if d == 1:
        return np.zeros((1, 0)), np.ones(1)
    x, w = np.polynomial.legendre.leggauss(order)
    nodes1, weights1 = 0.25 * (x + 1.0), 0.25 * w
    idx = np.indices((order,) * (d - 1)).reshape(d - 1, -1).T
    v = nodes1[idx]
    wts = weights1[idx[:, 0]].copy()
    for axis in range(1, d - 1):
        wts = wts * weights1[idx[:, axis]]
    return v, wts


def tail_primitive(nu: float, m: int, eps: float, wsq, allow_high_log_power: bool = False):
    """Continuation value of ``int_0^eps u^(-nu-1) log^m(pi u^2 w^2) du`` (L/quadrature.py:274-296).

    Integrating by parts once per log power gives the closed sum
    ``-(eps^-nu / nu) * sum_j m!/(m-j)! (2/nu)^j L^(m-j)``, ``L = log(pi eps^2 w^2)``; the boundary
    term at ``u = 0`` is the part the continuation drops.  ``nu = 0`` is a genuine divergence.
    """
    if m < 0:
        raise ValueError(f"negative log power {m} in a tail monomial")
    if m > 3 and not allow_high_log_power:
        raise NotImplementedError(
            f"log power {m} > 3 in a tail monomial; pass allow_high_log_power=True")
    if abs(nu) < _POLE_TOL:
        raise PoleError(f"tail monomial u^-1 log^{m} has no continuation (nu = {nu!r})")
    ell = np.log(math.pi * eps * eps * np.asarray(wsq, dtype=float))
    # Horner over j: sum_j c_j L^(m-j) with c_j = m!/(m-j)! (2/nu)^j
    acc = np.ones_like(ell)
    coef = 1.0
    for j in range(1, m + 1):
        coef *= (m - j + 1) * 2.0 / nu
        acc = acc * ell + coef
    return -(eps ** (-nu) / nu) * acc


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

    def product_at(self, k):
        """prod_j Z_j(k)^{m_j} at a CUDA tensor of k points (n, d) -> CUDA tensor (n,) (product
        plans; one fused kernel for every factor)."""
        import torch
        k = k.contiguous()
        out = torch.empty(k.shape[0], dtype=torch.float64, device=k.device)
        st = torch.cuda.current_stream(k.device).cuda_stream
        N.check(N.lib().lz_plan_product_at(self._h, k.data_ptr(), k.shape[0], out.data_ptr(), None, st),
                "product at k")
        return out

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
# Round 2: the row-factorised direct space (d = 3) costs one complex multiply-add per (row, plane,
# channel) and line, so the split drops to 0.05 (fcc: 6,107 direct points, ~3 reciprocal terms per
# node); d <= 2 plans (slab walk) keep 0.13.
ATM_SPLIT_SCALE = float(os.environ.get("LATSUM_ATM_SPLIT_SCALE", "0.05"))
ATM_X_LO_MAX = 8.0
ATM_SPLIT_SCALE_LOW_D = float(os.environ.get("LATSUM_ATM_SPLIT_SCALE_2D", "0.13"))


_HELPER = None


def _helper():
    global _HELPER
    if _HELPER is None:
        from concurrent.futures import ThreadPoolExecutor
        _HELPER = ThreadPoolExecutor(max_workers=1, thread_name_prefix="latsum-plan")
    return _HELPER


@lru_cache(maxsize=64)
def atm_plan(lattice: Lattice, splitting: float | None = None) -> Plan:
    """Plan for the ATM integrand [Z_3^3, tr(M_5^3)], M_5 = polynomial-weighted zeta at nu = 5."""
    auto_split = splitting is None
    if splitting is None:
        scale = ATM_SPLIT_SCALE if lattice.d == 3 else ATM_SPLIT_SCALE_LOW_D
        if scale != 1.0:
            splitting = scale * lattice.volume ** (-2.0 / lattice.d)
            if lattice.d == 3:
                # the line kernel's q = 0 pieces cover x = c |k|^2 <= x_lo = c sigma_min(B)^2 / 4
                # (csrc/context.cpp table_x_lo) in bins of 0.25: keep x_lo <= 8 (32 bins, and the
                # rho series they are fitted from converges well inside its 64 terms)
                sig2 = 1.0 / float(np.linalg.eigvalsh(lattice.a.T @ lattice.a).max())
                splitting = max(splitting, math.pi * sig2 / (4.0 * ATM_X_LO_MAX))
    # the two contexts' host enumerations are independent native calls (GIL released): overlap them
    # (one helper thread, kept for the process)
    # Both contexts are private to this (cached) plan and enumerate only what it reads: Z_3 lends
    # its constants and reciprocal set (the kernel takes Z_3 = tr M_5), Z_5 its constants and the
    # Hessian's widened point sets
    f5 = _helper().submit(EpsteinContext, lattice, 5.0, splitting, -2)
    z3 = EpsteinContext(lattice, 3.0, splitting, deriv_order=-1)
    z5 = f5.result()
    h = C.c_void_p()
    N.check(N.lib().lz_plan_create_atm(z3.handle, z5.handle, C.byref(h)), "atm plan")
    plan = Plan(h, lattice.d, 2, (z3, z5))
    if auto_split and lattice.d == 3 and ATM_SPLIT_SCALE < ATM_SPLIT_SCALE_LOW_D and \
            plan.info().smem_bytes > 120_000:
        # the direct set did not fit the row-factorised block (very anisotropic cells): the slab
        # walk pays per direct point, so it gets the larger split
        return atm_plan(lattice, ATM_SPLIT_SCALE_LOW_D * lattice.volume ** (-2.0 / lattice.d))
    return plan


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


def endpoint_exponent(contexts, d: int) -> float:
    """Smallest non-analytic power ``eta`` of ``u`` in ``u^(d-1) prod Z(nu_i, u w)`` near ``u = 0``.

    Along a ray ``Z(nu, u w) = Z_reg(u w) + s(u w) / V`` with ``Z_reg`` analytic, so the
    integrand's only non-smooth terms come from the singular parts (L/epstein.py:202-231):
    ``u^(nu-d)`` (generic; analytic when ``nu - d`` is an odd integer, since ``|u w|^odd =
    u^odd |w|^odd``) or ``u^(2m) log u`` (log case).  Returns ``inf`` for an analytic integrand.
    """
    eta = math.inf
    for ctx in contexts:
        if ctx.branch == TRIVIAL:
            continue
        if ctx.branch == LOG_CASE:
            e = 2.0 * ctx.log_m
        else:
            if ctx.singular_coef() == 0.0:
                continue
            e = ctx.nu - d
            r = round(e)
            if abs(e - r) < 1e-12 and r % 2 == 1:
                continue
        eta = min(eta, d - 1 + e)
    return eta


# digits the graded radial rule is sized for: Gauss-Legendre on t^(q(eta+1)-1) loses
# n^(-2 q (eta+1)), so q is the smallest grading that pushes that below 10^-_GRADE_DIGITS
_GRADE_DIGITS = 18
_MAX_GRADING = 8


def auto_grading(eta: float, n_u: int, base: int = 1) -> int:
    """Radial grading ``u = t^q / 2`` for an endpoint term ``u^eta`` on an ``n_u``-point rule."""
    if not math.isfinite(eta) or n_u < 2:
        return base
    q = math.ceil(_GRADE_DIGITS * math.log(10.0) / (2.0 * (eta + 1.0) * math.log(n_u)))
    return max(base, min(q, _MAX_GRADING))


def integrate_product(lattice: Lattice, nus, cfg: QuadratureConfig | None = None, threads: int = 1):
    """Duffy-decomposed ``V int_BZ prod_i Z(nu_i, k) dk`` (L/quadrature.py:455-490).

    Returns (value, error_estimate), honouring the reference's accuracy contract
    ``cfg.adaptive_rel_tol`` (L/quadrature.py:421-423):

    * every exponent above d (``method="auto"``): a fixed Duffy grid on the GPU whose radial
      grading is chosen from the integrand's endpoint singularity (:func:`endpoint_exponent`),
      checked against a 3/4-resolution grid; if the two differ by more than
      ``10 * adaptive_rel_tol * |value|`` the grid is doubled once, and if that still fails the
      reference's own adaptive Gauss-Kronrod strategy runs with GPU panels;
    * some exponent at or below d: the adaptive path with the analytic tail (continuation);
    * ``method="grid"``: exactly the configured grid (``grading`` as given), no escalation;
    * ``method="adaptive"``: the reference's adaptive strategy for every exponent.

    ``threads`` is accepted for signature compatibility; the GPU does the work.
    """
    cfg = cfg or QuadratureConfig()
    nus = [float(x) for x in nus]
    d = lattice.d
    contexts = [epstein_context(lattice, nu, cfg.splitting) for nu in nus]
    live = [c for c in contexts if c.branch != TRIVIAL]
    min_nu = min(c.nu for c in live) if live else math.inf
    if cfg.method == "adaptive" or (cfg.method == "auto" and min_nu <= d):
        N.require_cuda("BZ quadrature")
        from .adaptive import integrate_product_adaptive
        return integrate_product_adaptive(lattice, contexts, cfg)
    if min_nu <= d:
        from .tail import integrate_product_continued
        return integrate_product_continued(lattice, contexts, cfg)
    if cfg.method == "grid":
        value = fixed_grid_integral(lattice, nus, cfg.grid_u, cfg.grid_v, cfg.grading, cfg.splitting)
        err = 0.0
        if cfg.estimate_error:
            err = abs(value - fixed_grid_integral(lattice, nus, max(2, (3 * cfg.grid_u) // 4),
                                                  max(1, (3 * cfg.grid_v) // 4), cfg.grading,
                                                  cfg.splitting))
        return value, err
    eta = endpoint_exponent(contexts, d)
    n_u, n_v = cfg.grid_u, cfg.grid_v
    for _ in range(2):
        q = auto_grading(eta, n_u, cfg.grading)
        value = fixed_grid_integral(lattice, nus, n_u, n_v, q, cfg.splitting)
        if not cfg.estimate_error:
            return value, 0.0
        coarse = fixed_grid_integral(lattice, nus, max(2, (3 * n_u) // 4), max(1, (3 * n_v) // 4),
                                     q, cfg.splitting)
        err = abs(value - coarse)
        if err <= 10.0 * cfg.adaptive_rel_tol * abs(value):
            return value, err
        n_u, n_v = 2 * n_u, 2 * n_v
    N.require_cuda("BZ quadrature")
    from .adaptive import integrate_product_adaptive
    return integrate_product_adaptive(lattice, contexts, cfg)


def integrate_bz_even(lattice: Lattice, fvec, cfg: QuadratureConfig | None = None):
    """``V int_BZ f(k) dk`` for an even integrand given as a k-batch callable (L/quadrature.py:493-515).

    The reference's rule: per Duffy cell, whole-range adaptive Gauss-Kronrod in ``u`` shared by
    the cell's ``gauss_order^(d-1)`` angular directions, weighted by the angular rule, cells
    summed exactly.  All cells advance in lock step so ``fvec`` sees one batch per refinement
    round (each cell's refinement decisions read only its own panels, so the trees, and hence
    the value, are those of the per-cell loop).  ``fvec`` is the caller's host function: this is
    a test utility, not the device path.
    """
    from .adaptive import NODES, _CellState, panel_sums
    cfg = cfg or QuadratureConfig()
    d = lattice.d
    v, wts = angular_nodes(d, cfg.gauss_order)
    dirs = [cell.directions(lattice, v) for cell in duffy_cells(d)]
    states = [_CellState(0.0, 0.5) for _ in dirs]
    while True:
        active = [i for i, st in enumerate(states) if st.pending is not None]
        if not active:
            break
        ks, shapes = [], []
        for i in active:
            a, b = states[i].pending
            u = ((0.5 * (a + b))[:, None] + (0.5 * (b - a))[:, None] * NODES[None, :]).ravel()
            ks.append((u[:, None, None] * dirs[i][None, :, :]).reshape(-1, d))
            shapes.append((u, len(a)))
        f_all = np.asarray(fvec(np.concatenate(ks)), dtype=float).ravel()
        off = 0
        for i, (u, m) in zip(active, shapes):
            nw = len(dirs[i])
            f = f_all[off:off + len(u) * nw].reshape(len(u), nw) * (u ** (d - 1))[:, None]
            off += len(u) * nw
            a, b = states[i].pending
            vals, errs, floors = panel_sums(f.reshape(m, 15, nw), a, b)
            states[i].absorb(vals, errs, floors, cfg.adaptive_rel_tol, cfg.adaptive_max_depth)
    return 2.0 ** d * math.fsum(float(wts @ st.result[0]) for st in states)
