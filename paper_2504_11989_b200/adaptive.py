"""Adaptive Gauss-Kronrod radial quadrature with GPU panel evaluation.

Drop-in fidelity mode of ``integrate_product`` (``QuadratureConfig(method="adaptive")``):
the reference's radial strategy (L/quadrature.py:183-268, 400-452) -- vector-valued
Kronrod-15 / Gauss-7 panels shared by all angular directions of a Duffy cell,
QUADPACK error scaling, refinement of every interval carrying at least a quarter
of the worst excess, deterministic interval order -- with the zeta products of
every panel evaluated on the GPU.  All Duffy cells advance in lock step, so one
round of refinement is one device batch (the per-cell refinement decisions only
read that cell's own panels, as in the reference, so results do not depend on
the batching).  For exponents <= d the inner part (0, epsilon) is the analytic
tail (tail.py) and the outer integrand has its growing monomials subtracted and
re-added in closed form, as the reference does.
"""
from __future__ import annotations

import math

import numpy as np

from .errors import ConvergenceError
from .tail import ray_series, tail_values

# Kronrod 15-point nodes (positive half, descending) with the embedded 7-point Gauss rule
# (QUADPACK qk15 constants).
_XK = np.array([0.991455371120812639206854697526329, 0.949107912342758524526189684047851,
                0.864864423359769072789712788640926, 0.741531185599394439863864773280788,
                0.586087235467691130294144838258730, 0.405845151377397166906606412076961,
                0.207784955007898467600689403773245, 0.0])
_WK = np.array([0.022935322010529224963732008058970, 0.063092092629978553290700663189204,
                0.104790010322250183839876322541518, 0.140653259715525918745189590510238,
                0.169004726639267902826583426598550, 0.190350578064785409913256402421014,
                0.204432940075298892414161999234649, 0.209482141084727828012999174891714])
_WG = np.array([0.129484966168869693270611432679082, 0.279705391489276667901467771423780,
                0.381830050505118944950369775488975, 0.417959183673469387755102040816327])

NODES = np.concatenate([-_XK[:-1], _XK[::-1]])          # 15 ascending abscissae on [-1, 1]
W_KRONROD = np.concatenate([_WK[:-1], _WK[::-1]])
W_GAUSS = np.zeros(15)
W_GAUSS[1::2] = np.concatenate([_WG[:-1], _WG[::-1]])   # Gauss points are the odd Kronrod ones

_MAX_INTERVALS = 60_000
_EPS = np.finfo(float).eps


def panel_sums(fv: np.ndarray, a: np.ndarray, b: np.ndarray):
    """Kronrod value, scaled error and roundoff floor of each interval; fv: (m, 15, W)."""
    half = (0.5 * (b - a))[:, None]
    ik = np.einsum("n,mnw->mw", W_KRONROD, fv) * half
    ig = np.einsum("n,mnw->mw", W_GAUSS, fv) * half
    resabs = np.einsum("n,mnw->mw", W_KRONROD, np.abs(fv)) * half
    mean = ik / (b - a)[:, None]
    resasc = np.einsum("n,mnw->mw", W_KRONROD, np.abs(fv - mean[:, None, :])) * half
    raw = np.abs(ik - ig)
    with np.errstate(divide="ignore", invalid="ignore"):
        ratio = np.where(resasc > 0.0, 200.0 * raw / np.where(resasc > 0.0, resasc, 1.0), 0.0)
        scaled = np.where(resasc > 0.0, resasc * np.minimum(1.0, ratio ** 1.5), raw)
    floor = 50.0 * _EPS * resabs
    return ik, np.maximum(scaled, floor), floor


class _CellState:
    """Subdivision tree of one Duffy cell (all W directions share it)."""

    def __init__(self, lo: float, hi: float):
        self.a = np.array([lo])
        self.b = np.array([hi])
        self.depth = np.array([0])
        self.vals = self.errs = self.floors = None
        self.pending = (self.a, self.b)   # intervals awaiting panel values
        self.result = None

    def absorb(self, vals, errs, floors, rtol, max_depth):
        """Merge the new panels, then either finish or pick the next intervals to split."""
        if self.vals is None:
            self.vals, self.errs, self.floors = vals, errs, floors
        else:
            keep = self._keep
            self.a = np.concatenate([self.a[keep], self._new_a])
            self.b = np.concatenate([self.b[keep], self._new_b])
            self.depth = np.concatenate([self.depth[keep], self._new_depth])
            self.vals = np.concatenate([self.vals[keep], vals])
            self.errs = np.concatenate([self.errs[keep], errs])
            self.floors = np.concatenate([self.floors[keep], floors])
            if len(self.a) > _MAX_INTERVALS:
                raise ConvergenceError("radial quadrature exceeded the interval budget")
            order = np.argsort(self.a, kind="stable")
            self.a, self.b, self.depth = self.a[order], self.b[order], self.depth[order]
            self.vals, self.errs, self.floors = self.vals[order], self.errs[order], self.floors[order]
        total = self.vals.sum(axis=0)
        target = np.maximum(rtol * np.maximum(np.abs(total), 0.1 * np.abs(self.vals).sum(axis=0)), 1e-300)
        etot = self.errs.sum(axis=0)
        if np.all(etot <= np.maximum(target, 1.25 * self.floors.sum(axis=0))):
            exact = np.array([math.fsum(self.vals[:, j]) for j in range(self.vals.shape[1])])
            self.result = (exact, etot)
            self.pending = None
            return
        bad = np.max(np.maximum(self.errs - self.floors, 0.0) / target[None, :], axis=1)
        can = self.depth < max_depth
        if not np.any(can & (bad > 0.0)):
            raise ConvergenceError(f"radial quadrature stalled at depth {max_depth}: error {etot.max():.2e}")
        worst = bad[can].max()
        sel = can & (bad >= 0.25 * worst) & (bad > 0.0)
        if not np.any(sel):
            sel = can & (bad > 0.0)
        idx = np.nonzero(sel)[0]
        mid = 0.5 * (self.a[idx] + self.b[idx])
        self._keep = ~sel
        self._new_a = np.concatenate([self.a[idx], mid])
        self._new_b = np.concatenate([mid, self.b[idx]])
        self._new_depth = np.concatenate([self.depth[idx] + 1, self.depth[idx] + 1])
        self.pending = (self._new_a, self._new_b)


class _DeviceProfile:
    """f(u, w) = const * u^(d-1) prod_j Z_j(u w)^{m_j} - subtracted monomials, with the zeta
    products of a whole refinement round evaluated in one GPU batch: one fused product kernel
    per group of <= 4 distinct exponents (lz_plan_product_at), contexts at cfg.splitting."""

    def __init__(self, lattice, groups, const, splitting=None):
        from .quadrature import product_plan
        self.d = lattice.d
        self.const = const
        self.plans = [product_plan(lattice, tuple(groups[i:i + 4]), splitting) for i in range(0, len(groups), 4)]

    def __call__(self, blocks, subs):
        import torch
        d = self.d
        k = np.concatenate([(u[:, None, None] * w[None, :, :]).reshape(-1, d) for u, w in blocks])
        kt = torch.from_numpy(k).pin_memory().to("cuda", non_blocking=True)
        prod = None
        for plan in self.plans:
            z = plan.product_at(kt)
            prod = z if prod is None else prod * z
        vals = prod.cpu().numpy() * self.const
        out, off = [], 0
        for (u, w), sub in zip(blocks, subs):
            n = len(u) * len(w)
            f = vals[off:off + n].reshape(len(u), len(w)) * (u ** (d - 1))[:, None]
            off += n
            if sub:
                wsq = np.einsum("ij,ij->i", w, w)
                for eta, m, c in sub:
                    mono = u[:, None] ** eta * c[None, :]
                    if m:
                        mono = mono * np.log(math.pi * u[:, None] ** 2 * wsq[None, :]) ** m
                    f = f - mono
            out.append(f)
        return out


def integrate_product_adaptive(lattice, contexts, cfg):
    """V int_BZ prod Z dk with the reference's adaptive radial strategy; (value, error)."""
    from .epstein import TRIVIAL
    from .quadrature import _distinct, angular_nodes, duffy_cells, tail_primitive
    d = lattice.d
    groups, const = _distinct(contexts)
    if const == 0.0:
        return 0.0, 0.0
    if not groups:
        return const, 0.0
    live = [c for c in contexts if c.branch != TRIVIAL]
    v, wts = angular_nodes(d, cfg.gauss_order)
    dirs = [cell.directions(lattice, v) for cell in duffy_cells(d)]
    min_nu = min(c.nu for c in live)
    continued = min_nu <= d
    lo = cfg.epsilon if continued else 0.0
    inner = [np.zeros(len(w)) for w in dirs]
    subtract = None
    if continued:
        taylors = [c.reg_derivatives(cfg.taylor_order) for c in live]
        subtract = []
        for ci, w in enumerate(dirs):
            series = ray_series(live, taylors, w, cfg)
            inner[ci] = tail_values(live, taylors, w, cfg, series) * const
            sub = []
            for (e, m), c in sorted(series.items()):
                eta = d - 1 + e
                if eta >= 0.5 or abs(eta + 1.0) < 1e-8 or (m > 3 and not cfg.allow_high_log_power):
                    continue
                sub.append((eta, m, c * const))
            subtract.append(sub)
    states = [_CellState(lo, 0.5) for _ in dirs]
    profile = _DeviceProfile(lattice, groups, const, cfg.splitting)
    while True:
        active = [ci for ci, s in enumerate(states) if s.pending is not None]
        if not active:
            break
        blocks = []
        for ci in active:
            a, b = states[ci].pending
            mid, half = 0.5 * (a + b), 0.5 * (b - a)
            blocks.append(((mid[:, None] + half[:, None] * NODES[None, :]).ravel(), dirs[ci]))
        subs = [subtract[ci] for ci in active] if subtract is not None else [None] * len(active)
        for ci, f in zip(active, profile(blocks, subs)):
            a, b = states[ci].pending
            vals, errs, floors = panel_sums(f.reshape(len(a), 15, len(dirs[ci])), a, b)
            states[ci].absorb(vals, errs, floors, cfg.adaptive_rel_tol, cfg.adaptive_max_depth)
    cell_vals, cell_errs = [], []
    for ci, w in enumerate(dirs):
        outer, err = states[ci].result
        if continued:
            wsq = np.einsum("ij,ij->i", w, w)
            for eta, m, c in subtract[ci]:
                nu_p = -(eta + 1.0)
                up = tail_primitive(nu_p, m, 0.5, wsq, cfg.allow_high_log_power)
                dn = tail_primitive(nu_p, m, cfg.epsilon, wsq, cfg.allow_high_log_power)
                outer = outer + c * (up - dn)
            outer = outer + inner[ci]
        cell_vals.append(float(wts @ outer))
        cell_errs.append(float(wts @ err))
    scale = 2.0 ** d
    return scale * math.fsum(cell_vals), scale * math.fsum(abs(e) for e in cell_errs)
