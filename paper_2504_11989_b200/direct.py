"""Truncated direct summation on the GPU (the SPEC's oracle module).

Brute-force three-body sums over x, y in A{-L..L}^d -- an independent check of the
Epstein-zeta method that uses no special functions and no quadrature.  The
reference package does not ship this module; the paper's own direct sums
(1D ATM at L = 5000, 2D at L = 250 -- "over 10^10 summands")
take hours on a CPU and ~0.1 s here.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _native as N
from .lattice import Lattice

DEFAULT_MAX_PAIRS = 1e13   # ~100 s on one B200; the SPEC's CPU guard is 1e10


def _run(lattice: Lattice, L: int, kind: int, nus, max_pairs: float) -> float:
    if lattice.d > 3:
        raise ValueError("direct sums support d <= 3")
    N.require_cuda("direct summation")
    a = np.ascontiguousarray(lattice.a, dtype=np.float64)
    nu = np.ascontiguousarray(np.asarray(nus if nus is not None else (0.0, 0.0, 0.0), dtype=np.float64))
    out = C.c_double(0.0)
    N.check(N.lib().lz_direct_sum3(N.current_device(), lattice.d, N.dptr(a), int(L), kind, N.dptr(nu),
                                   float(max_pairs), C.byref(out)), "direct sum")
    return out.value


def direct_sum_zeta(lattice: Lattice, nus, L: int, max_pairs: float = DEFAULT_MAX_PAIRS) -> float:
    """sum' |x|^-nu1 |y - x|^-nu2 |y|^-nu3 over x, y, x - y != 0 in A{-L..L}^d (n = 3)."""
    nus = [float(v) for v in nus]
    if len(nus) != 3:
        raise ValueError("the GPU direct sum covers the three-body zeta function")
    if min(nus) <= lattice.d / 2.0:
        raise ValueError("direct summation needs convergent exponents (min nu > d/2 per factor)")
    return _run(lattice, L, 0, nus, max_pairs)


def direct_sum_atm(lattice: Lattice, L: int, max_pairs: float = DEFAULT_MAX_PAIRS) -> float:
    """(1/6) sum' U_ATM(x, y) over x, y, x - y != 0 in A{-L..L}^d (Def. 1.1)."""
    return _run(lattice, L, 1, None, max_pairs)
