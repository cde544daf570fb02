"""Taylor tables of Z_reg at k = 0 (host side, one-time per context).

Native: lz_ctx_reg_derivatives evaluates every partial derivative of even total
order <= ``order`` from the Hermite expansion of the Gaussian representation in
long double with compensated sums (reference: L/epstein.py:347-415).
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _native as N


def build_reg_derivatives(ctx, order: int):
    from .epstein import RegZetaTaylor
    n = C.c_int64(0)
    N.check(N.lib().lz_ctx_reg_derivatives(ctx.handle, order, None, None, 0, C.byref(n)), "reg_derivatives")
    al = np.zeros((n.value, ctx.d), dtype=np.int32)
    vals = np.zeros(n.value, dtype=np.float64)
    N.check(N.lib().lz_ctx_reg_derivatives(ctx.handle, order, al.ctypes.data_as(C.POINTER(C.c_int)),
                                           N.dptr(vals), n.value, C.byref(n)), "reg_derivatives")
    derivs = {tuple(int(x) for x in a): float(v) for a, v in zip(al, vals)}
    return RegZetaTaylor(ctx.lattice, ctx.nu, order, derivs)
