"""TEST INFRASTRUCTURE ONLY: ctypes wrapper of the plain-C restatement
oracle/hyteg_oracle.c (built to oracle/_build/liboracle.so).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may use
it -- as the checker, never as the product."""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "_build", "liboracle.so")
_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            raise FileNotFoundError(f"{LIB} not built (make -C oracle restatement)")
        L = C.CDLL(LIB)
        p, i, d, u64, i64 = C.c_void_p, C.c_int, C.c_double, C.c_uint64, C.c_int64
        pd = C.POINTER(C.c_double)
        sig = {
            "og_last_error": (C.c_char_p, []),
            "og_create": (p, [C.c_char_p, i, i, C.POINTER(C.c_int), C.POINTER(C.c_ubyte), i, i]),
            "og_destroy": (None, [p]),
            "og_owned": (i64, [p, i]),
            "og_set": (i, [p, i, i, pd]),
            "og_get": (i, [p, i, i, pd]),
            "og_flags": (i, [p, i, C.POINTER(C.c_ubyte)]),
            "og_stencil": (i, [p, i64, i, pd, C.POINTER(C.c_int)]),
            "og_keyed_uniform": (i, [p, i, u64, u64, d, d, pd]),
            "og_sync": (i, [p, i, i]),
            "og_apply": (i, [p, i, i, i, i]),
            "og_residual": (i, [p, i, i, i, i]),
            "og_jacobi": (i, [p, i, i, d, i]),
            "og_gs": (i, [p, i, i, i]),
            "og_cgs": (i, [p, i, i, i]),
            "og_fmg": (i, [p, i, i, i, i, i, i, d, d, i, d, i, pd, C.POINTER(C.c_int)]),
            "og_pcg": (i, [p, i, i, i, i, i, d, d, i, pd]),
            "og_vcycle": (i, [p, i, i, i, i, i, i, d, d, i, pd]),
            "og_restrict": (i, [p, i, i, i, i]),
            "og_prolongate": (i, [p, i, i, i, i]),
            "og_assign": (i, [p, d, i, d, i, i, i, i]),
            "og_add_scaled": (i, [p, i, d, i, i, i]),
            "og_dot": (i, [p, i, i, i, pd]),
            "og_vcycle_jacobi": (i, [p, i, i, i, i, i, d, d, i, pd]),
            "og_coarse_solver": (None, [p, i, i]),
            "og_coarse_matrix": (i, [p, i, C.POINTER(i64), C.POINTER(i64), pd, i64, C.POINTER(i64)]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def _ck(code: int) -> None:
    if code != 0:
        raise RuntimeError(lib().og_last_error().decode(errors="replace"))


def _pd(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


class Session:
    """Single-rank restatement session: mesh, levels, nfuncs functions, LAPLACE."""

    def __init__(self, mesh: str, min_level: int, max_level: int, nfuncs: int = 4, bc: dict | None = None):
        bc = bc or {}
        m = (C.c_int * max(len(bc), 1))(*bc.keys())
        f = (C.c_ubyte * max(len(bc), 1))(*bc.values())
        h = lib().og_create(mesh.encode(), min_level, max_level, m, f, len(bc), nfuncs)
        if not h:
            raise RuntimeError(lib().og_last_error().decode())
        self.h = h
        self.mesh = mesh

    def __del__(self):
        if getattr(self, "h", None):
            lib().og_destroy(self.h)
            self.h = None

    def owned(self, level):
        return int(lib().og_owned(self.h, level))

    def set(self, fi, level, v):
        v = np.ascontiguousarray(v, dtype=np.float64)
        assert v.size == self.owned(level)
        _ck(lib().og_set(self.h, fi, level, _pd(v)))

    def get(self, fi, level):
        out = np.empty(self.owned(level))
        _ck(lib().og_get(self.h, fi, level, _pd(out)))
        return out

    def flags(self, level):
        out = np.zeros(self.owned(level), dtype=np.uint8)
        _ck(lib().og_flags(self.h, level, out.ctypes.data_as(C.POINTER(C.c_ubyte))))
        return out

    def stencil(self, pid, level):
        out = np.zeros(64)
        n = C.c_int()
        _ck(lib().og_stencil(self.h, pid, level, _pd(out), C.byref(n)))
        return out[: n.value].copy()

    def keyed_uniform(self, level, seed, stream=0, lo=-1.0, hi=1.0):
        out = np.empty(self.owned(level))
        _ck(lib().og_keyed_uniform(self.h, level, seed, stream, lo, hi, _pd(out)))
        return out

    def apply(self, src, dst, level, mask=7):
        _ck(lib().og_apply(self.h, src, dst, level, mask))

    def residual(self, rhs, x, r, level):
        _ck(lib().og_residual(self.h, rhs, x, r, level))

    def jacobi(self, rhs, x, omega, level):
        _ck(lib().og_jacobi(self.h, rhs, x, omega, level))

    def gs(self, rhs, x, level):
        _ck(lib().og_gs(self.h, rhs, x, level))

    def cgs(self, rhs, x, level):
        _ck(lib().og_cgs(self.h, rhs, x, level))

    def vcycle(self, rhs, x, level, smoother, nu1, nu2, omega, coarse_tol, ncycles):
        res = np.zeros(ncycles + 1)
        _ck(lib().og_vcycle(self.h, rhs, x, level, smoother, nu1, nu2, omega, coarse_tol, ncycles, _pd(res)))
        return res

    def fmg(self, rhs, x, level, smoother, nu1, nu2, omega, coarse_tol, per_level, tol, max_cycles):
        res = np.zeros(max_cycles + 2)
        n = C.c_int()
        _ck(lib().og_fmg(self.h, rhs, x, level, smoother, nu1, nu2, omega, coarse_tol, per_level, tol, max_cycles,
                         _pd(res), C.byref(n)))
        return res[: n.value]

    def pcg(self, rhs, x, level, nu1, nu2, omega, coarse_tol, iters):
        res = np.zeros(iters + 1)
        _ck(lib().og_pcg(self.h, rhs, x, level, nu1, nu2, omega, coarse_tol, iters, _pd(res)))
        return res

    def coarse_solver(self, mode, nsm=148):
        """0: matrix-free CG with sequential dots (default); 1: the product's
        coarse solve (assembled constrained CSR, the device kernels' reduction
        shapes; nsm = SM count, which only the largest systems depend on)."""
        lib().og_coarse_solver(self.h, mode, nsm)

    def coarse_matrix(self, scratch):
        """the min-level CSR of coarse_solver(1) as COO (rows, cols, vals)"""
        n = C.c_int64()
        _ck(lib().og_coarse_matrix(self.h, scratch, None, None, None, 0, C.byref(n)))
        r = np.empty(n.value, dtype=np.int64)
        c = np.empty(n.value, dtype=np.int64)
        v = np.empty(n.value)
        _ck(lib().og_coarse_matrix(self.h, scratch, r.ctypes.data_as(C.POINTER(C.c_int64)),
                                   c.ctypes.data_as(C.POINTER(C.c_int64)), _pd(v), n.value, C.byref(n)))
        return r, c, v

    def restrict(self, fine, coarse, lc, mask=7):
        _ck(lib().og_restrict(self.h, fine, coarse, lc, mask))

    def prolongate(self, coarse, fine, lc, mask=7):
        _ck(lib().og_prolongate(self.h, coarse, fine, lc, mask))

    def assign(self, alpha, x1, beta, x2, dst, level, mask=7):
        _ck(lib().og_assign(self.h, alpha, x1, beta, x2, dst, level, mask))

    def add_scaled(self, dst, gamma, y, level, mask=7):
        _ck(lib().og_add_scaled(self.h, dst, gamma, y, level, mask))

    def dot(self, a, b, level):
        out = C.c_double()
        _ck(lib().og_dot(self.h, a, b, level, C.byref(out)))
        return out.value

    def vcycle_jacobi(self, rhs, x, level, nu1, nu2, omega, coarse_tol, ncycles):
        res = np.zeros(ncycles + 1)
        _ck(lib().og_vcycle_jacobi(self.h, rhs, x, level, nu1, nu2, omega, coarse_tol, ncycles, _pd(res)))
        return res


def keyed_uniform(mesh: str, level: int, seed: int, stream: int = 0, lo: float = -1.0, hi: float = 1.0):
    return Session(mesh, level, level, 1).keyed_uniform(level, seed, stream, lo, hi)
