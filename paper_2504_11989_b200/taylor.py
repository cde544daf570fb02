"""Taylor tables of Z_reg at k = 0 (one-time per context), L/epstein.py:347-415.

The table is computed on the context's device: lz_ctx_reg_derivatives_device runs the moment
form of the derivative kernel (deriv.cu) at k = 0 for every even total order <= ``order`` over
the reference's widened point sets, with compensated sums (the reference combines the same
Hermite expansion with math.fsum).  ``build_reg_derivatives_host`` is the long-double host
restatement (lz_ctx_reg_derivatives), kept as a cross-check for the tests.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _native as N


def _table(ctx, order: int, fn_name: str):
    from .epstein import RegZetaTaylor
    fn = getattr(N.lib(), fn_name)
    n = C.c_int64(0)
    N.check(fn(ctx.handle, order, None, None, 0, C.byref(n)), "reg_derivatives")
    al = np.zeros((n.value, ctx.d), dtype=np.int32)
    vals = np.zeros(n.value, dtype=np.float64)
    N.check(fn(ctx.handle, order, al.ctypes.data_as(C.POINTER(C.c_int)), N.dptr(vals), n.value, C.byref(n)),
            "reg_derivatives")
    derivs = {tuple(int(x) for x in a): float(v) for a, v in zip(al, vals)}
    return RegZetaTaylor(ctx.lattice, ctx.nu, order, derivs)


def build_reg_derivatives(ctx, order: int):
    N.require_cuda("Taylor tables of Z_reg")
    return _table(ctx, order, "lz_ctx_reg_derivatives_device")


def build_reg_derivatives_host(ctx, order: int):
    return _table(ctx, order, "lz_ctx_reg_derivatives")
