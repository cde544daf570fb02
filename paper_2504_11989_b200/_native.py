"""ctypes binding of the C ABI in include/latsum_b200.h.

The shared library is built in-tree (``paper_2504_11989_b200/_lib``) by
``__graft_entry__.build()`` / :func:`build_library`.  There is no Python or CPU
fallback for any compute entry point: if the library is missing this module
raises on first use, and if no CUDA device is present every compute call
raises ``RuntimeError``.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading
import warnings

from .errors import LatticeError, PoleError

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_DIR = os.path.join(_HERE, "_lib")
LIB_PATH = os.path.join(LIB_DIR, "liblatsum_b200.so")
CSRC = os.path.join(_HERE, "csrc")
INCLUDE = os.path.join(os.path.dirname(_HERE), "include")
SOURCES = ["kernels.cu", "direct.cu", "deriv.cu", "context.cpp", "capi.cpp"]

NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo", "-O3", "-std=c++17",
              "-Xcompiler", "-fPIC", "-shared", "-ldl"]

LZ_OK, LZ_EINVAL, LZ_EPOLE, LZ_ENONFINITE, LZ_ECUDA, LZ_ENCCL, LZ_ESHELLS, LZ_ELATTICE, LZ_ESINGULAR = range(9)
NO_REDUCE, REG_ONLY, SINGULAR_ONLY = 1, 2, 4


class CtxParams(C.Structure):
    _fields_ = [("d", C.c_int), ("a", C.c_double * 16), ("nu", C.c_double),
                ("splitting", C.c_double), ("deriv_order", C.c_int)]


class CtxInfo(C.Structure):
    _fields_ = [("d", C.c_int), ("branch", C.c_int), ("log_m", C.c_int), ("pole", C.c_int),
                ("nu", C.c_double), ("vol", C.c_double), ("split", C.c_double),
                ("s_rec", C.c_double), ("pref", C.c_double), ("rfac", C.c_double),
                ("bconst", C.c_double), ("kmax", C.c_double), ("singular_coef", C.c_double),
                ("const_value", C.c_double),
                ("n_dir", C.c_int64), ("n_rec", C.c_int64), ("n_dir_h", C.c_int64),
                ("n_rec_h", C.c_int64),
                ("table_x_lo", C.c_double), ("table_x_hi", C.c_double),
                ("table_max_rel_err", C.c_double),
                ("table_pieces", C.c_int64), ("table_bins", C.c_int64)]


class Grid(C.Structure):
    _fields_ = [("n_u", C.c_int), ("n_v", C.c_int), ("grading", C.c_int),
                ("tile_lo", C.c_int64), ("tile_hi", C.c_int64), ("u_lo", C.c_double)]


class PlanInfo(C.Structure):
    _fields_ = [("d", C.c_int), ("kind", C.c_int), ("nctx", C.c_int), ("hess", C.c_int),
                ("alias", C.c_int), ("n_funcs", C.c_int),
                ("n_dir", C.c_int64), ("n_runs", C.c_int64), ("n_rec", C.c_int64),
                ("table_pieces", C.c_int64), ("table_bins", C.c_int64), ("n_t0", C.c_int64),
                ("smem_bytes", C.c_int64),
                ("table_x_lo", C.c_double), ("table_x_hi", C.c_double), ("table_max_rel_err", C.c_double),
                ("r_cut", C.c_double), ("split", C.c_double), ("t0_rho_max", C.c_double)]


# exported symbols and their signatures (every declaration of include/latsum_b200.h)
_P = C.c_void_p
_D = C.POINTER(C.c_double)
SIGNATURES = {
    "lz_ctx_create": (C.c_int, [C.POINTER(CtxParams), C.c_int, C.POINTER(_P)]),
    "lz_ctx_destroy": (C.c_int, [_P]),
    "lz_ctx_get_info": (C.c_int, [_P, C.POINTER(CtxInfo)]),
    "lz_ctx_prepare": (C.c_int, [_P, C.c_int]),
    "lz_ctx_get_points": (C.c_int, [_P, C.c_int, _D, C.c_int64, C.POINTER(C.c_int64)]),
    "lz_zeta": (C.c_int, [_P, _P, C.c_int64, _P, C.c_uint32, C.c_int, _P, _P]),
    "lz_zeta_host": (C.c_int, [_P, _D, C.c_int64, _D, C.c_uint32]),
    "lz_zeta_hessian": (C.c_int, [_P, _P, C.c_int64, _P, C.c_int, _P]),
    "lz_zeta_hessian_host": (C.c_int, [_P, _D, C.c_int64, _D]),
    "lz_grid_tiles": (C.c_int, [C.c_int, C.POINTER(Grid), C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
    "lz_plan_create_product": (C.c_int, [C.POINTER(_P), C.POINTER(C.c_int), C.c_int, C.POINTER(_P)]),
    "lz_plan_create_atm": (C.c_int, [_P, _P, C.POINTER(_P)]),
    "lz_plan_destroy": (C.c_int, [_P]),
    "lz_plan_get_info": (C.c_int, [_P, C.POINTER(PlanInfo)]),
    "lz_plan_product_at": (C.c_int, [_P, _P, C.c_int64, _P, _P, _P]),
    "lz_plan_integrate": (C.c_int, [_P, C.POINTER(Grid), _P, C.c_int, _P]),
    "lz_reduce_partials": (C.c_int, [_P, C.c_int64, C.c_int, _P, _P]),
    "lz_reduce_chunks": (C.c_int, [_P, C.c_int64, C.c_int, C.c_int64, C.c_int64, C.c_int64, _P, _P]),
    "lz_chunk_layout": (C.c_int, [C.c_int64, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
    "lz_transfer_stats": (C.c_int, [C.POINTER(C.c_int64), C.POINTER(C.c_int64), C.c_int]),
    "lz_release_caches": (C.c_int, [C.c_int]),
    "lz_plan_integrate_host": (C.c_int, [_P, C.POINTER(Grid), _D]),
    "lz_multi_indices": (C.c_int, [C.c_int, C.c_int, C.POINTER(C.c_int), C.c_int64, C.POINTER(C.c_int64)]),
    "lz_zeta_derivatives": (C.c_int, [_P, C.c_int, _P, C.c_int64, _P, _P, _P]),
    "lz_zeta_derivatives_host": (C.c_int, [_P, C.c_int, _D, C.c_int64, _D]),
    "lz_ctx_reg_derivatives": (C.c_int, [_P, C.c_int, C.POINTER(C.c_int), _D, C.c_int64,
                                          C.POINTER(C.c_int64)]),
    "lz_ctx_reg_derivatives_device": (C.c_int, [_P, C.c_int, C.POINTER(C.c_int), _D, C.c_int64,
                                                 C.POINTER(C.c_int64)]),
    "lz_upper_gamma": (C.c_double, [C.c_double, C.c_double]),
    "lz_direct_sum3": (C.c_int, [C.c_int, C.c_int, _D, C.c_int64, C.c_int, _D, C.c_double, _D]),
    "lz_fp64_peak": (C.c_int, [C.c_int, _D, _D]),
    "lz_allreduce_partials": (C.c_int, [_P, C.c_int64, _P, _P]),
    "lz_device_count": (C.c_int, [C.POINTER(C.c_int)]),
    "lz_strerror": (C.c_char_p, [C.c_int]),
    "lz_last_error": (C.c_char_p, []),
    "lz_version": (C.c_char_p, []),
}

_lib = None
_lock = threading.Lock()


def build_library(force: bool = False, verbose: bool = False) -> str:
    """Compile the sm_100a shared library in-tree with nvcc."""
    srcs = [os.path.join(CSRC, s) for s in SOURCES]
    hdrs = [os.path.join(CSRC, h) for h in ("special.cuh", "lz_internal.h")]
    hdrs.append(os.path.join(INCLUDE, "latsum_b200.h"))
    if not force and os.path.exists(LIB_PATH):
        newest = max(os.path.getmtime(p) for p in srcs + hdrs)
        if os.path.getmtime(LIB_PATH) >= newest:
            return LIB_PATH
    os.makedirs(LIB_DIR, exist_ok=True)
    nvcc = os.environ.get("NVCC", "nvcc")
    tmp = LIB_PATH + f".tmp{os.getpid()}"
    # one nvcc per translation unit, in parallel, then one link (same flags as a single call)
    from concurrent.futures import ThreadPoolExecutor
    compile_flags = [f for f in NVCC_FLAGS if f not in ("-shared", "-ldl")]
    objs = [os.path.join(LIB_DIR, os.path.basename(src) + f".{os.getpid()}.o") for src in srcs]

    def compile_one(pair):
        src, obj = pair
        cmd = [nvcc, *compile_flags, "-c", src, "-o", obj]
        return cmd, subprocess.run(cmd, capture_output=True, text=True)

    try:
        with ThreadPoolExecutor(max_workers=len(srcs)) as pool:
            results = list(pool.map(compile_one, zip(srcs, objs)))
        for cmd, res in results:
            if res.returncode != 0:
                raise RuntimeError("nvcc failed:\n" + " ".join(cmd) + "\n" + res.stdout + res.stderr)
            if verbose:
                print(res.stdout + res.stderr)
        cmd = [nvcc, *NVCC_FLAGS, *objs, "-o", tmp]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError("nvcc link failed:\n" + " ".join(cmd) + "\n" + res.stdout + res.stderr)
    finally:
        for o in objs:
            if os.path.exists(o):
                os.remove(o)
    os.replace(tmp, LIB_PATH)
    return LIB_PATH


def lib():
    """The loaded library (raises if it was never built: there is no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        # LATSUM_LIB: load another build of the library (A/B timing of kernel variants)
        path = os.environ.get("LATSUM_LIB") or LIB_PATH
        if not os.path.exists(path):
            raise RuntimeError(
                f"latsum_b200 native library not found at {path}; run "
                "`python -c 'import __graft_entry__ as g; g.build()'` (no CPU fallback exists)")
        L = C.CDLL(path)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def last_error() -> str:
    return lib().lz_last_error().decode()


def check(rc: int, what: str = ""):
    """Map C-ABI status codes onto the reference's exception classes."""
    if rc == LZ_OK:
        return
    msg = last_error() or lib().lz_strerror(rc).decode()
    if what:
        msg = f"{what}: {msg}"
    if rc == LZ_EPOLE:
        raise PoleError(msg)
    if rc == LZ_ELATTICE:
        raise LatticeError(msg)
    if rc in (LZ_EINVAL, LZ_ENONFINITE, LZ_ESINGULAR):
        raise ValueError(msg)
    if rc == LZ_ESHELLS:
        raise RuntimeError(msg)
    raise RuntimeError(msg)


_ndev = None


def device_count() -> int:
    global _ndev
    if _ndev is None:
        n = C.c_int(0)
        lib().lz_device_count(C.byref(n))
        _ndev = n.value
    return _ndev


def require_cuda(what: str):
    if device_count() < 1:
        raise RuntimeError(f"{what} needs a CUDA device: latsum_b200 has no CPU compute path")


def current_device() -> int:
    """Device of new contexts: torch's current device when torch has CUDA, else 0."""
    if device_count() < 1:
        return -1
    try:
        import torch
        if torch.cuda.is_available():
            return torch.cuda.current_device()
    except Exception:  # pragma: no cover - torch is optional for the API
        warnings.warn("torch unavailable; using CUDA device 0")
    return 0


def dptr(arr):
    return arr.ctypes.data_as(_D)
