"""ctypes wrapper of the CPU oracle (oracle/latsum_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and the
cpu_baseline / --impl reference legs of bench.py -- never by the product
package.  Parity of the oracle itself is pinned against golden vectors made by
running the reference (tests/golden/make_golden.py; tests/test_oracle.py).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "_build", "liblatsum_oracle.so")
_lib = None


def build(force: bool = False) -> str:
    src = os.path.join(HERE, "latsum_oracle.c")
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(src):
        subprocess.run(["make", "-s", "-C", HERE, "-B" if force else "_build/liblatsum_oracle.so"],
                       check=True)
    return LIB


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            build()
        L = C.CDLL(LIB)
        D = C.POINTER(C.c_double)
        L.orc_zeta.argtypes = [C.c_int, D, C.c_double, D, C.c_long, D, C.c_int]
        L.orc_hessian.argtypes = [C.c_int, D, C.c_double, D, C.c_long, D]
        L.orc_derivatives.argtypes = [C.c_int, D, C.c_double, C.c_int, D, C.c_long, D]
        L.orc_derivatives_abs.argtypes = [C.c_int, D, C.c_double, C.c_int, D, C.c_long, D, D]
        L.orc_multi_indices.argtypes = [C.c_int, C.c_int, C.POINTER(C.c_int)]
        L.orc_product_grid.argtypes = [C.c_int, D, D, C.c_int, C.c_int, C.c_int, C.c_int, C.c_long,
                                       C.c_long, D]
        L.orc_atm_grid.argtypes = [C.c_int, D, C.c_int, C.c_int, C.c_int, C.c_long, C.c_long, D]
        L.orc_upper_gamma.argtypes = [C.c_double, C.c_double]
        L.orc_upper_gamma.restype = C.c_double
        L.orc_context_counts.argtypes = [C.c_int, D, C.c_double, C.POINTER(C.c_long)]
        L.orc_grid_nodes.argtypes = [C.c_int, C.c_int, C.c_int]
        L.orc_grid_nodes.restype = C.c_long
        _lib = L
    return _lib


def _p(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _mat(lattice_a):
    return np.ascontiguousarray(np.asarray(lattice_a, dtype=np.float64))


def nthreads() -> int:
    return lib().orc_nthreads()


def zeta(a, nu, k, flags=0):
    """Z(nu, k) (flags 0) / Z_reg without reduction (flags 3); raises on a pole."""
    a = _mat(a)
    d = a.shape[0]
    k = np.ascontiguousarray(np.atleast_2d(np.asarray(k, dtype=np.float64)))
    out = np.empty(len(k))
    rc = lib().orc_zeta(d, _p(a), float(nu), _p(k), len(k), _p(out), flags)
    if rc == 2:
        raise ArithmeticError("pole")
    if rc:
        raise RuntimeError(f"oracle error {rc}")
    return out


def hessian(a, nu, k):
    a = _mat(a)
    d = a.shape[0]
    k = np.ascontiguousarray(np.atleast_2d(np.asarray(k, dtype=np.float64)))
    out = np.empty((len(k), d, d))
    rc = lib().orc_hessian(d, _p(a), float(nu), _p(k), len(k), _p(out))
    if rc:
        raise RuntimeError(f"oracle error {rc}")
    return out


def multi_indices(d, order):
    buf = (C.c_int * (512 * 4))()
    n = lib().orc_multi_indices(d, order, buf)
    return [tuple(buf[i * d:(i + 1) * d]) for i in range(n)]


def derivatives(a, nu, order, k, with_abs=False):
    """All d^alpha Z(k), |alpha| = order, in multi_indices(d, order) order (long double).
    with_abs: also the sum of |terms| of each value (direct + Hermite reciprocal terms), the
    cancellation scale that bounds the rounding error of any double-precision evaluation."""
    a = _mat(a)
    d = a.shape[0]
    k = np.ascontiguousarray(np.atleast_2d(np.asarray(k, dtype=np.float64)))
    na = len(multi_indices(d, order))
    out = np.empty((len(k), na))
    ab = np.empty((len(k), na))
    rc = lib().orc_derivatives_abs(d, _p(a), float(nu), int(order), _p(k), len(k), _p(out), _p(ab))
    if rc:
        raise RuntimeError(f"oracle error {rc}")
    return (out, ab) if with_abs else out


def product_grid(a, nus, n_u, n_v, grading=1, lo=0, hi=0):
    a = _mat(a)
    nus = np.ascontiguousarray(np.asarray(nus, dtype=np.float64))
    out = np.zeros(1)
    rc = lib().orc_product_grid(a.shape[0], _p(a), _p(nus), len(nus), n_u, n_v, grading, lo, hi, _p(out))
    if rc:
        raise RuntimeError(f"oracle error {rc}")
    return out[0]


def atm_grid(a, n_u, n_v, grading=3, lo=0, hi=0):
    a = _mat(a)
    out = np.zeros(2)
    rc = lib().orc_atm_grid(a.shape[0], _p(a), n_u, n_v, grading, lo, hi, _p(out))
    if rc:
        raise RuntimeError(f"oracle error {rc}")
    return out


def grid_nodes(d, n_u, n_v):
    return lib().orc_grid_nodes(d, n_u, n_v)


def upper_gamma(s, x):
    return lib().orc_upper_gamma(float(s), float(x))


def counts(a, nu):
    a = _mat(a)
    out = (C.c_long * 4)()
    rc = lib().orc_context_counts(a.shape[0], _p(a), float(nu), out)
    if rc:
        raise RuntimeError(f"oracle error {rc}")
    return tuple(out)
