"""Epstein zeta functions on Bravais lattices — drop-in for L/epstein.py.

``Z(nu, k) = sum'_{z in Lambda} exp(-2 pi i z.k) |z|^-nu`` (meromorphically
continued), evaluated with the reference's theta split (L/epstein.py:1-29):
a direct sum of incomplete-gamma weights times phases, a reciprocal sum of
``|k+q|^(nu-d) Gamma((d-nu)/2, pi |k+q|^2 / t)`` and the explicit singularity
``shat``.  Context construction (point sets, constants, reciprocal-summand
tables) happens once in the native library; every evaluation runs on the GPU
through the C ABI (``lz_zeta*``).  The public names, signatures, branch
semantics, error classes and scalar/batch conventions follow the reference.

Beyond the reference: :meth:`EpsteinContext.zeta_hessian` and
:meth:`EpsteinContext.polynomial_weighted` give the Cartesian-derivative
(polynomial-weighted) zeta ``M_ab(k) = sum' z_a z_b |z|^-nu e^{-2 pi i z.k}
= -d_a d_b Z_nu(k) / (4 pi^2)`` needed for the ATM dot-product term.
"""
from __future__ import annotations

import ctypes as C
import math
import threading
from dataclasses import dataclass
from functools import lru_cache

import numpy as np

from . import _native as N
from .lattice import Lattice

GENERIC = "generic"
LOG_CASE = "log_case"
TRIVIAL = "trivial"
_BRANCHES = {0: GENERIC, 1: LOG_CASE, 2: TRIVIAL}

_BRANCH_TOL = 1e-12
TWO_PI = 2.0 * math.pi


def classify_exponent(nu: float, d: int):
    """(branch, snapped nu, log index m or None), as L/epstein.py:58-70."""
    if not np.isfinite(nu):
        raise ValueError("exponent must be finite")
    if abs(nu) > 100.0:
        raise ValueError("exponent magnitude above 100 is not supported")
    m = round((nu - d) / 2.0)
    if m >= 0 and abs(nu - (d + 2 * m)) < _BRANCH_TOL:
        return LOG_CASE, float(d + 2 * m), int(m)
    j = round(-nu / 2.0)
    if j >= 0 and abs(nu + 2 * j) < _BRANCH_TOL:
        return TRIVIAL, float(-2 * j), None
    return GENERIC, float(nu), None


def _as_batch(k, d):
    k = np.asarray(k, dtype=np.float64)
    single = k.ndim == 1
    k2 = np.ascontiguousarray(np.atleast_2d(k))
    if k2.shape[-1] != d:
        raise ValueError(f"k must have trailing dimension {d}, got shape {k.shape}")
    if not np.all(np.isfinite(k2)):
        raise ValueError("k contains non-finite entries")
    return k2.reshape(-1, d), single, k.shape[:-1] if k.ndim > 1 else ()


class EpsteinContext:
    """Per-(lattice, exponent) device-resident evaluation data (L/epstein.py:93-122).

    Construct through :func:`epstein_context`.  Immutable after construction;
    safe to share between threads.
    """

    def __init__(self, lattice: Lattice, nu: float, splitting: float | None = None,
                 deriv_order: int = 2, device: int | None = None):
        self.lattice = lattice
        d = lattice.d
        self.d = d
        p = N.CtxParams()
        p.d = d
        flat = np.ascontiguousarray(lattice.a, dtype=np.float64).ravel()
        for i, v in enumerate(flat):
            p.a[i] = float(v)
        p.nu = float(nu)
        p.splitting = float(splitting) if splitting is not None else -1.0
        p.deriv_order = int(deriv_order)
        self.device = N.current_device() if device is None else device
        h = C.c_void_p()
        N.check(N.lib().lz_ctx_create(C.byref(p), self.device, C.byref(h)), "epstein context")
        self._h = h
        info = N.CtxInfo()
        N.lib().lz_ctx_get_info(h, C.byref(info))
        self.info = info
        self.branch = _BRANCHES[info.branch]
        self.nu = info.nu
        self.log_m = info.log_m if info.branch == 1 else None
        self.vol = info.vol
        self.split = info.split
        self._lock = threading.Lock()
        self._taylor_cache: dict = {}
        self.has_hessian = False
        if self.branch == TRIVIAL:
            self.const_value = info.const_value
            return
        self.s_rec = info.s_rec
        self.pref = info.pref
        self.rfac = info.rfac
        self.bconst = info.bconst
        self.kmax = info.kmax
        # Hessian point sets and tables are built on first use; deriv_order < 0 marks the ATM
        # plan's private contexts (-1: reciprocal set only, -2: Hessian sets only)
        self.has_hessian = deriv_order >= 2 or deriv_order == -2

    def __del__(self):
        try:  # also reached at interpreter shutdown, when module globals may be gone
            h = getattr(self, "_h", None)
            if h is not None and N is not None and N._lib is not None:
                N._lib.lz_ctx_destroy(h)
        except Exception:
            pass

    def table_stats(self, hessian: bool = False) -> "N.CtxInfo":
        """Build the evaluation tables now (normally lazy) and return the context info with the
        table statistics (pieces, bins, x range, measured max relative fit error)."""
        N.check(N.lib().lz_ctx_prepare(self._h, 3 if (hessian and self.has_hessian) else 1), "prepare")
        info = N.CtxInfo()
        N.lib().lz_ctx_get_info(self._h, C.byref(info))
        return info

    # the reference's point-set attributes (L/epstein.py:126-198), fetched from the native
    # context on first access (plan-private contexts never need them)
    @property
    def dir_pts(self) -> np.ndarray:
        return self._cached("_dir_pts", lambda: self._points(0).reshape(-1, self.d))

    @property
    def dir_w(self) -> np.ndarray:
        return self._cached("_dir_w", lambda: self._points(1))

    @property
    def rec_pts(self) -> np.ndarray:
        return self._cached("_rec_pts", lambda: self._points(2).reshape(-1, self.d))

    @property
    def rec_norm2(self) -> np.ndarray:
        return self._cached("_rec_norm2", lambda: np.einsum("ij,ij->i", self.rec_pts, self.rec_pts))

    def _cached(self, name, make):
        v = self.__dict__.get(name)
        if v is None:
            v = make()
            self.__dict__[name] = v
        return v

    def _points(self, which):
        n = C.c_int64(0)
        N.lib().lz_ctx_get_points(self._h, which, None, 0, C.byref(n))
        out = np.empty(n.value, dtype=np.float64)
        if n.value:
            N.lib().lz_ctx_get_points(self._h, which, N.dptr(out), n.value, C.byref(n))
        return out

    @property
    def handle(self):
        return self._h

    # -- evaluation (GPU) -------------------------------------------------------------
    def _eval(self, k, flags):
        kb, single, shape = _as_batch(k, self.d)
        if self.branch == TRIVIAL:
            out = np.full(len(kb), self.const_value) if not (flags & N.SINGULAR_ONLY) else np.zeros(len(kb))
        else:
            N.require_cuda("Epstein zeta evaluation")
            out = np.empty(len(kb), dtype=np.float64)
            if len(kb):
                N.check(N.lib().lz_zeta_host(self._h, N.dptr(kb), len(kb), N.dptr(out), flags),
                        "zeta")
        if single:
            return float(out[0])
        return out.reshape(shape) if shape else out

    def _eval_into(self, k: np.ndarray, out: np.ndarray, flags: int = 0) -> np.ndarray:
        """Z into a caller-provided host buffer (no allocation; pinned buffers skip staging)."""
        N.require_cuda("Epstein zeta evaluation")
        assert k.dtype == np.float64 and k.flags.c_contiguous and out.dtype == np.float64
        n = k.shape[0]
        if n:
            N.check(N.lib().lz_zeta_host(self._h, N.dptr(k), n, N.dptr(out), flags), "zeta")
        return out

    def zeta_device(self, k, out=None, flags: int = 0, lanes_per_point: int = 0, stream=None):
        """Zero-copy path: ``k`` a CUDA torch tensor (n, d) float64; returns a CUDA tensor."""
        import torch
        N.require_cuda("Epstein zeta evaluation")
        k = k.contiguous()
        n = k.shape[0]
        if out is None:
            out = torch.empty(n, dtype=torch.float64, device=k.device)
        status = torch.zeros(1, dtype=torch.int32, device=k.device)
        st = stream if stream is not None else torch.cuda.current_stream(k.device).cuda_stream
        N.check(N.lib().lz_zeta(self._h, k.data_ptr(), n, out.data_ptr(), flags, lanes_per_point,
                                status.data_ptr(), st), "zeta")
        return out, status

    def singular_coef(self) -> float:
        """Coefficient of shat without the |k| powers (L/epstein.py:202-215)."""
        if self.branch == TRIVIAL:
            return 0.0
        return self.info.singular_coef

    def singular(self, k) -> np.ndarray:
        """shat(nu, k) (L/epstein.py:217-231); no BZ reduction, batch output."""
        kb = np.atleast_2d(np.asarray(k, dtype=float))
        rho = np.einsum("ij,ij->i", kb, kb)
        if self.branch == TRIVIAL:
            return np.zeros(len(rho))
        if self.branch == LOG_CASE and np.any(rho == 0.0):
            raise ValueError("singular part undefined at k = 0 in the log case")
        if self.branch == GENERIC and self.nu < self.d and np.any(rho == 0.0):
            raise ValueError("singular part diverges at k = 0 for nu < d")
        out = self._eval(kb, N.NO_REDUCE | N.SINGULAR_ONLY)
        return np.atleast_1d(out)

    def reg_zeta(self, k):
        """Z_reg(nu, k) on a batch (L/epstein.py:261-289); k is not reduced."""
        return self._eval(k, N.NO_REDUCE | N.REG_ONLY)

    def zeta(self, k):
        """Z(nu, k) = Z_reg + shat/V with the k = 0 continuation convention (L/epstein.py:291-320)."""
        return self._eval(k, 0)

    def zeta_at_zero(self) -> float:
        """Z(nu, 0) through the continuation in nu; pole at nu = d (L/epstein.py:322-324)."""
        return float(self.zeta(np.zeros(self.d)))

    # -- Cartesian-derivative (polynomial-weighted) zeta -----------------------------
    def zeta_hessian(self, k) -> np.ndarray:
        """d_a d_b Z_nu(k) as (..., d, d); k must not sit on the reciprocal lattice."""
        if self.branch == TRIVIAL:
            kb, single, shape = _as_batch(k, self.d)
            out = np.zeros((len(kb), self.d, self.d))
            return out[0] if single else out.reshape(shape + (self.d, self.d))
        if not self.has_hessian:
            raise ValueError("context built without Hessian tables (deriv_order < 2)")
        kb, single, shape = _as_batch(k, self.d)
        N.require_cuda("Epstein zeta Hessian")
        ns = self.d * (self.d + 1) // 2
        tri = np.empty((len(kb), ns), dtype=np.float64)
        if len(kb):
            N.check(N.lib().lz_zeta_hessian_host(self._h, N.dptr(kb), len(kb), N.dptr(tri)),
                    "zeta hessian")
        full = np.empty((len(kb), self.d, self.d))
        c = 0
        for a in range(self.d):
            for b in range(a, self.d):
                full[:, a, b] = tri[:, c]
                full[:, b, a] = tri[:, c]
                c += 1
        if single:
            return full[0]
        return full.reshape(shape + (self.d, self.d)) if shape else full

    def polynomial_weighted(self, k) -> np.ndarray:
        """M_ab(k) = sum' z_a z_b |z|^-nu e^{-2 pi i z.k} = -Hess Z_nu(k) / (4 pi^2)."""
        return -self.zeta_hessian(k) / (4.0 * math.pi ** 2)

    # -- order-m derivatives at arbitrary k (device kernel, deriv.cu)
    def derivatives(self, k, order: int):
        """All d^alpha Z_nu(k) with |alpha| = order (1..4, d <= 3): returns (alphas, values) with
        alphas a list of d-tuples in the reference's order (L/epstein.py:426-433) and values of
        shape (..., n_alpha).  k must avoid the reciprocal lattice (PoleError)."""
        alphas = multi_indices(self.d, order)
        kb, single, shape = _as_batch(k, self.d)
        if self.branch == TRIVIAL:
            out = np.zeros((len(kb), len(alphas)))
        else:
            N.require_cuda("Epstein zeta derivatives")
            out = np.empty((len(kb), len(alphas)), dtype=np.float64)
            if len(kb):
                N.check(N.lib().lz_zeta_derivatives_host(self._h, int(order), N.dptr(kb), len(kb),
                                                         N.dptr(out)), "zeta derivatives")
        if single:
            return alphas, out[0]
        return alphas, out.reshape(shape + (len(alphas),))

    def derivatives_device(self, k, order: int, out=None):
        """All d^alpha Z_nu(k), |alpha| = order, for a CUDA tensor of k points (n, d): returns the
        CUDA tensor (n, n_alpha) (stream-ordered, no host copies; pole points are not checked)."""
        import torch
        n = k.shape[0]
        na = len(multi_indices(self.d, order))
        if out is None:
            out = torch.empty((n, na), dtype=torch.float64, device=k.device)
        st = torch.cuda.current_stream(k.device).cuda_stream
        N.check(N.lib().lz_zeta_derivatives(self._h, int(order), k.contiguous().data_ptr(), n, out.data_ptr(),
                                            None, st), "zeta derivatives")
        return out

    def polynomial_weighted_general(self, k, alpha) -> np.ndarray:
        """M^alpha(k) = sum'_z z^alpha |z|^-nu e^{-2 pi i z.k} = d^alpha Z(k) / (-2 pi i)^|alpha|
        (complex; real for even |alpha|, imaginary for odd)."""
        alpha = tuple(int(a) for a in alpha)
        if len(alpha) != self.d or min(alpha) < 0:
            raise ValueError("alpha must be a d-tuple of nonnegative integers")
        m = sum(alpha)
        if m == 0:
            return self.zeta(k).astype(complex)
        alphas, vals = self.derivatives(k, m)
        j = alphas.index(alpha)
        return vals[..., j] / (-2j * math.pi) ** m

    # -- derivatives of the regularized part at k = 0 (host tables, L/epstein.py:347-415)
    def reg_derivatives(self, order: int) -> "RegZetaTaylor":
        if order % 2 != 0:
            raise ValueError("derivative order must be even")
        if order > 12:
            raise ValueError("derivative order above 12 is not supported")
        with self._lock:
            if order not in self._taylor_cache:
                from .taylor import build_reg_derivatives
                self._taylor_cache[order] = build_reg_derivatives(self, order)
            return self._taylor_cache[order]


@dataclass(frozen=True)
class RegZetaTaylor:
    """Partial derivatives of Z_reg at k = 0 up to an even total order (L/epstein.py:436-466)."""

    lattice: Lattice
    nu: float
    order: int
    derivs: dict

    def directional_coeff(self, w, k: int):
        """(w.grad)^{2k} Z_reg(0) / (2k)! for one direction or a batch of rows."""
        if 2 * k > self.order:
            raise ValueError(f"order {2 * k} exceeds table order {self.order}")
        w = np.asarray(w, dtype=float)
        single = w.ndim == 1
        w = np.atleast_2d(w)
        alphas, coef = self._order_terms(2 * k)
        if len(coef) == 0:
            acc = np.zeros(len(w))
        else:
            # all multi-indices of the order at once: power ladders w_a^0..w_a^total by repeated
            # multiplication, gathered per multi-index
            total = 2 * k
            acc = None
            for a in range(w.shape[1]):
                ladder = np.empty((len(w), total + 1))
                ladder[:, 0] = 1.0
                for e in range(1, total + 1):
                    ladder[:, e] = ladder[:, e - 1] * w[:, a]
                term = ladder[:, alphas[:, a]]
                acc = term if acc is None else acc * term
            acc = acc @ coef
        return acc[0] if single else acc

    def _order_terms(self, total: int):
        """Multi-indices of one total order with nonzero entries and their coefficients
        multinomial(alpha) D^alpha Z_reg(0) / total! (cached per table)."""
        cache = self.__dict__.setdefault("_terms", {})
        if total not in cache:
            al, cf = [], []
            for alpha, val in self.derivs.items():
                if sum(alpha) != total or val == 0.0:
                    continue
                mult = math.factorial(total)
                for a in alpha:
                    mult //= math.factorial(a)
                al.append(alpha)
                cf.append(mult * val / math.factorial(total))
            d = self.lattice.d
            cache[total] = (np.array(al, dtype=np.intp).reshape(len(al), d), np.array(cf, dtype=float))
        return cache[total]


@lru_cache(maxsize=4096)
def epstein_context(lattice: Lattice, nu: float, splitting: float | None = None) -> EpsteinContext:
    """Memoized evaluation context for (lattice, exponent) (L/epstein.py:469-472)."""
    return EpsteinContext(lattice, float(nu), splitting)


def epstein_zeta(lattice: Lattice, nu: float, k, reg: bool = False):
    """Z(nu, k), or its regularized part with ``reg=True`` (L/epstein.py:478-481)."""
    ctx = epstein_context(lattice, nu)
    return ctx.reg_zeta(k) if reg else ctx.zeta(k)


def singular_part(lattice: Lattice, nu: float, k):
    """shat(nu, k) (no 1/V factor) (L/epstein.py:484-486)."""
    return epstein_context(lattice, nu).singular(k)


def regularized_zeta(lattice: Lattice, nu: float, k):
    """Z_reg(nu, k) = Z(nu, k) - shat(nu, k)/V (L/epstein.py:489-491)."""
    return epstein_context(lattice, nu).reg_zeta(k)


def reg_zeta_derivatives(lattice: Lattice, nu: float, order: int) -> RegZetaTaylor:
    """Partial derivatives of Z_reg at k = 0 (L/epstein.py:494-496)."""
    return epstein_context(lattice, nu).reg_derivatives(order)


def directional_taylor_coeff(taylor: RegZetaTaylor, w, k: int):
    """Coefficient of u^(2k) in Z_reg(u w) around u = 0 (L/epstein.py:499-501)."""
    return taylor.directional_coeff(w, k)


def polynomial_weighted_zeta(lattice: Lattice, nu: float, k, alpha=None):
    """M_ab(k) = sum' z_a z_b |z|^-nu e^{-2 pi i z.k} (the ATM dot-product building block), or
    for a multi-index ``alpha`` the general M^alpha(k) = sum' z^alpha |z|^-nu e^{-2 pi i z.k}."""
    if alpha is None:
        return epstein_context(lattice, nu).polynomial_weighted(k)
    return epstein_context(lattice, nu).polynomial_weighted_general(k, alpha)


def multi_indices(d: int, order: int):
    """All d-tuples of nonnegative integers summing to ``order`` (L/epstein.py:426-433 order),
    as enumerated by the native library."""
    import ctypes as C
    n = C.c_int64(0)
    N.check(N.lib().lz_multi_indices(int(d), int(order), None, 0, C.byref(n)), "multi indices")
    buf = (C.c_int * (n.value * d))()
    N.check(N.lib().lz_multi_indices(int(d), int(order), buf, n.value, C.byref(n)), "multi indices")
    return [tuple(buf[i * d:(i + 1) * d]) for i in range(n.value)]
