"""TEST INFRASTRUCTURE ONLY: ctypes wrapper of oracle/_ref/libhyteg_ref.so.

That library is the unmodified reference (arXiv 1805.10167 "hytegrid",
/root/reference/proj/src/*.cpp) compiled by oracle/Makefile plus the plain-C
adapter oracle/ref_adapter.cpp. Only tests/, __graft_entry__.smoke() and
bench.py's CPU-baseline / --impl reference legs may use it -- as the checker
or the timed CPU reference, never as the product.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_LIB = os.path.join(HERE, "_ref", "libhyteg_ref.so")

_lib = None


def available() -> bool:
    return os.path.exists(REF_LIB)


def lib():
    global _lib
    if _lib is None:
        if not available():
            raise FileNotFoundError(f"{REF_LIB} not built (make -C oracle ref, needs /root/reference)")
        L = C.CDLL(REF_LIB)
        p, i, d, u8, u64, i64 = C.c_void_p, C.c_int, C.c_double, C.c_uint8, C.c_uint64, C.c_int64
        pd = C.POINTER(C.c_double)
        sig = {
            "ref_last_error": (C.c_char_p, []),
            "ref_meshgen": (i, [C.c_char_p, pd, C.c_char_p, i64, C.POINTER(i64)]),
            "ref_partition": (i, [C.c_char_p, i, i, i, C.POINTER(C.c_int)]),
            "ref_create": (i, [C.c_char_p, i, i, i, i, i, C.POINTER(C.c_int), C.POINTER(C.c_uint8), i, i,
                               C.POINTER(p)]),
            "ref_destroy": (None, [p]),
            "ref_create_kind": (i, [C.c_char_p, i, i, i, i, i, C.POINTER(C.c_int), C.POINTER(C.c_uint8), i, i, i,
                                    C.POINTER(p)]),
            "ref_owned": (i64, [p, i]),
            "ref_set": (i, [p, i, i, pd]),
            "ref_get": (i, [p, i, i, pd]),
            "ref_flags": (i, [p, i, i, C.POINTER(C.c_uint8)]),
            "ref_coords": (i, [p, i, pd]),
            "ref_sync": (i, [p, i, i]),
            "ref_serialize": (i, [p, i, C.c_uint64, C.POINTER(C.c_uint8), C.c_int64, C.POINTER(C.c_int64)]),
            "ref_apply": (i, [p, i, i, i, u8]),
            "ref_residual": (i, [p, i, i, i, i]),
            "ref_jacobi": (i, [p, i, i, d, i]),
            "ref_gs": (i, [p, i, i, i]),
            "ref_restrict": (i, [p, i, i, i, u8]),
            "ref_prolongate": (i, [p, i, i, i, u8]),
            "ref_assign": (i, [p, d, i, d, i, i, i, u8]),
            "ref_add_scaled": (i, [p, i, d, i, i, u8]),
            "ref_dot": (i, [p, i, i, i, pd]),
            "ref_stencil": (i, [p, u64, i, pd, C.POINTER(C.c_int)]),
            "ref_vcycle_jacobi": (i, [p, i, i, i, i, i, d, d, i, pd]),
            "ref_diagonal": (i, [p, i, i, i]),
            "ref_set_form": (i, [p, i]),
            "ref_sync_dirs": (i, [p, i, i, C.POINTER(C.c_int), i]),
            "ref_values": (i, [p, i, u64, i, pd, i64, C.POINTER(i64)]),
            "ref_set_values": (i, [p, i, u64, i, pd, i64]),
            "ref_fill_keyed": (i, [p, i, i, u64, u64, d, d]),
            "ref_coarse_matrix": (i, [p, i, C.POINTER(i64), C.POINTER(i64), pd, i64, C.POINTER(i64)]),
            "ref_gridhierarchy_solve": (i, [p, i, i, i, d, i, i, i, pd, C.POINTER(C.c_int)]),
            "ref_stokes_create": (i, [C.c_char_p, i, i, i, i, i, C.POINTER(C.c_int), C.POINTER(C.c_uint8), i,
                                      C.POINTER(C.c_int), C.POINTER(C.c_uint8), i, i, d, C.POINTER(p)]),
            "ref_stokes_destroy": (None, [p]),
            "ref_controller_trace": (i, [C.c_char_p, i, i, i, i, C.POINTER(C.c_int), i, C.POINTER(i64), i64,
                                         C.POINTER(i64)]),
            "ref_stokes_set": (i, [p, i, i, i, pd]),
            "ref_stokes_get": (i, [p, i, i, i, pd]),
            "ref_stokes_uzawa": (i, [p, i, d]),
            "ref_stokes_residual": (i, [p, i]),
            "ref_stokes_vcycle": (i, [p, i, i, i]),
            "ref_stokes_solve": (i, [p, i, d, i, i, i, pd, C.POINTER(C.c_int), C.POINTER(C.c_int)]),
            "ref_stokes_residual_norm": (i, [p, i, pd]),
            "ref_stokes_pressure_mean": (i, [p, i, pd]),
            "ref_stokes_matrix": (i, [p, i, C.POINTER(i64), C.POINTER(i64), pd, i64, C.POINTER(i64)]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


class RefError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


def _ck(code: int) -> None:
    if code != 0:
        raise RefError(code, lib().ref_last_error().decode(errors="replace"))


def meshgen(kind: str, *params: float) -> str:
    arr = (C.c_double * 4)(*params, *([0.0] * (4 - len(params))))
    n = C.c_int64()
    _ck(lib().ref_meshgen(kind.encode(), arr, None, 0, C.byref(n)))
    buf = C.create_string_buffer(n.value + 1)
    _ck(lib().ref_meshgen(kind.encode(), arr, buf, n.value + 1, C.byref(n)))
    return buf.value.decode()


def partition(mesh: str, ranks: int, partitioner: int, weight_level: int = 1) -> np.ndarray:
    out = np.zeros(_count(mesh), dtype=np.int32)
    _ck(lib().ref_partition(mesh.encode(), ranks, partitioner, weight_level, out.ctypes.data_as(C.POINTER(C.c_int))))
    return out


def _count(mesh: str) -> int:
    lines = [ln.split("#")[0].split() for ln in mesh.splitlines()]
    lines = [ln for ln in lines if ln]
    nv, nt = int(lines[0][0]), int(lines[0][1])
    edges = set()
    for t in lines[1 + nv: 1 + nv + nt]:
        a, b, c = int(t[0]), int(t[1]), int(t[2])
        edges |= {(min(a, b), max(a, b)), (min(a, c), max(a, c)), (min(b, c), max(b, c))}
    return nv + len(edges) + nt


class RefSession:
    """Reference domain + controller + nfuncs functions + LAPLACE operator."""

    def __init__(self, mesh: str, ranks: int, min_level: int, max_level: int, nfuncs: int = 4,
                 bc: dict | None = None, partitioner: int = 0, weight_level: int = 1, kind: int = 0):
        bc = bc or {}
        m = (C.c_int * max(len(bc), 1))(*bc.keys())
        f = (C.c_uint8 * max(len(bc), 1))(*bc.values())
        h = C.c_void_p()
        _ck(lib().ref_create_kind(mesh.encode(), ranks, partitioner, weight_level, min_level, max_level, m, f,
                                  len(bc), nfuncs, kind, C.byref(h)))
        self.h = h
        self.min_level, self.max_level = min_level, max_level

    def __del__(self):
        if getattr(self, "h", None):
            lib().ref_destroy(self.h)
            self.h = None

    def owned(self, level: int) -> int:
        return int(lib().ref_owned(self.h, level))

    def set(self, fi: int, level: int, values) -> None:
        v = np.ascontiguousarray(values, dtype=np.float64)
        assert v.size == self.owned(level)
        _ck(lib().ref_set(self.h, fi, level, v.ctypes.data_as(C.POINTER(C.c_double))))

    def get(self, fi: int, level: int) -> np.ndarray:
        out = np.empty(self.owned(level))
        _ck(lib().ref_get(self.h, fi, level, out.ctypes.data_as(C.POINTER(C.c_double))))
        return out

    def flags(self, fi: int, level: int) -> np.ndarray:
        out = np.zeros(self.owned(level), dtype=np.uint8)
        _ck(lib().ref_flags(self.h, fi, level, out.ctypes.data_as(C.POINTER(C.c_uint8))))
        return out

    def coords(self, level: int) -> np.ndarray:
        out = np.zeros((self.owned(level), 2))
        _ck(lib().ref_coords(self.h, level, out.ctypes.data_as(C.POINTER(C.c_double))))
        return out

    def sync(self, fi, level):
        _ck(lib().ref_sync(self.h, fi, level))

    def serialize(self, fi, prim) -> bytes:
        """The reference's DataCallbacks::serialize of primitive `prim`'s data of function fi."""
        n = C.c_int64()
        _ck(lib().ref_serialize(self.h, fi, prim, None, 0, C.byref(n)))
        buf = (C.c_uint8 * max(n.value, 1))()
        _ck(lib().ref_serialize(self.h, fi, prim, buf, n.value, C.byref(n)))
        return bytes(buf[: n.value])

    def apply(self, src, dst, level, mask=7):
        _ck(lib().ref_apply(self.h, src, dst, level, mask))

    def residual(self, rhs, x, r, level):
        _ck(lib().ref_residual(self.h, rhs, x, r, level))

    def jacobi(self, rhs, x, omega, level):
        _ck(lib().ref_jacobi(self.h, rhs, x, omega, level))

    def gs(self, rhs, x, level):
        _ck(lib().ref_gs(self.h, rhs, x, level))

    def restrict(self, fine, coarse, lc, mask=7):
        _ck(lib().ref_restrict(self.h, fine, coarse, lc, mask))

    def prolongate(self, coarse, fine, lc, mask=7):
        _ck(lib().ref_prolongate(self.h, coarse, fine, lc, mask))

    def assign(self, alpha, x1, beta, x2, dst, level, mask=7):
        _ck(lib().ref_assign(self.h, alpha, x1, beta, x2, dst, level, mask))

    def add_scaled(self, dst, gamma, y, level, mask=7):
        _ck(lib().ref_add_scaled(self.h, dst, gamma, y, level, mask))

    def dot(self, a, b, level) -> float:
        out = C.c_double()
        _ck(lib().ref_dot(self.h, a, b, level, C.byref(out)))
        return out.value

    def stencil(self, pid: int, level: int) -> np.ndarray:
        out = np.zeros(64)
        n = C.c_int()
        _ck(lib().ref_stencil(self.h, pid, level, out.ctypes.data_as(C.POINTER(C.c_double)), C.byref(n)))
        return out[: n.value].copy()

    def vcycle_jacobi(self, rhs, x, level, nu1, nu2, omega, coarse_tol, ncycles) -> np.ndarray:
        res = np.zeros(ncycles + 1)
        _ck(lib().ref_vcycle_jacobi(self.h, rhs, x, level, nu1, nu2, omega, coarse_tol, ncycles,
                                    res.ctypes.data_as(C.POINTER(C.c_double))))
        return res

    def sync_dirs(self, fi, level, dirs):
        d = (C.c_int * max(len(dirs), 1))(*dirs)
        _ck(lib().ref_sync_dirs(self.h, fi, level, d, len(dirs)))

    def values(self, fi, prim, level):
        n = C.c_int64()
        _ck(lib().ref_values(self.h, fi, prim, level, None, 0, C.byref(n)))
        out = np.zeros(n.value)
        _ck(lib().ref_values(self.h, fi, prim, level, out.ctypes.data_as(C.POINTER(C.c_double)), n.value,
                             C.byref(n)))
        return out

    def set_values(self, fi, prim, level, v):
        v = np.ascontiguousarray(v, dtype=np.float64)
        _ck(lib().ref_set_values(self.h, fi, prim, level, v.ctypes.data_as(C.POINTER(C.c_double)), v.size))

    def set_form(self, form):
        """operator of `form` (0 LAPLACE .. 6 PSPG) for apply / residual / stencil"""
        _ck(lib().ref_set_form(self.h, form))

    def fill_keyed(self, fi, level, seed, stream=0, lo=-1.0, hi=1.0):
        """keyed U[lo, hi] of the device generator, written in place"""
        _ck(lib().ref_fill_keyed(self.h, fi, level, seed, stream, lo, hi))

    def diagonal(self, form, d, level):
        _ck(lib().ref_diagonal(self.h, form, d, level))

    def coarse_matrix(self, level):
        """GridHierarchy's constrained min-level matrix as COO (rows, cols, vals)."""
        n = C.c_int64()
        _ck(lib().ref_coarse_matrix(self.h, level, None, None, None, 0, C.byref(n)))
        r = np.empty(n.value, dtype=np.int64)
        c = np.empty(n.value, dtype=np.int64)
        v = np.empty(n.value)
        _ck(lib().ref_coarse_matrix(self.h, level, r.ctypes.data_as(C.POINTER(C.c_int64)),
                                    c.ctypes.data_as(C.POINTER(C.c_int64)), v.ctypes.data_as(C.POINTER(C.c_double)), n.value,
                                    C.byref(n)))
        return r, c, v

    def gridhierarchy_solve(self, rhs, x, level, tol, max_cycles, nu1=2, nu2=2) -> np.ndarray:
        res = np.zeros(max_cycles + 1)
        n = C.c_int()
        _ck(lib().ref_gridhierarchy_solve(self.h, rhs, x, level, tol, max_cycles, nu1, nu2,
                                          res.ctypes.data_as(C.POINTER(C.c_double)), C.byref(n)))
        return res[: n.value]


def _bc_arrays(bc: dict):
    m = (C.c_int * max(len(bc), 1))(*bc.keys())
    f = (C.c_uint8 * max(len(bc), 1))(*bc.values())
    return m, f, len(bc)


class RefStokes:
    """The reference's StokesMultigrid (src/solvers.cpp:640-753) with states
    rhs (0), x (1), r (2); components 0 u1, 1 u2, 2 p."""

    def __init__(self, mesh: str, ranks: int, min_level: int, max_level: int, bc_velocity: dict,
                 bc_pressure: dict, project: bool = False, omega: float = 0.3, partitioner: int = 0,
                 weight_level: int = 1):
        mu, fu, nu = _bc_arrays(bc_velocity)
        mp, fp, npr = _bc_arrays(bc_pressure)
        h = C.c_void_p()
        _ck(lib().ref_stokes_create(mesh.encode(), ranks, partitioner, weight_level, min_level, max_level, mu, fu, nu,
                                    mp, fp, npr, int(project), omega, C.byref(h)))
        self.h = h
        self.mesh, self.ranks = mesh, ranks
        self._owned = RefSession(mesh, 1, min_level, max_level, nfuncs=1)

    def __del__(self):
        if getattr(self, "h", None):
            lib().ref_stokes_destroy(self.h)
            self.h = None

    def owned(self, level):
        return self._owned.owned(level)

    def set(self, state, comp, level, values):
        v = np.ascontiguousarray(values, dtype=np.float64)
        assert v.size == self.owned(level)
        _ck(lib().ref_stokes_set(self.h, state, comp, level, v.ctypes.data_as(C.POINTER(C.c_double))))

    def get(self, state, comp, level) -> np.ndarray:
        out = np.empty(self.owned(level))
        _ck(lib().ref_stokes_get(self.h, state, comp, level, out.ctypes.data_as(C.POINTER(C.c_double))))
        return out

    def uzawa(self, level, omega=0.3):
        _ck(lib().ref_stokes_uzawa(self.h, level, omega))

    def residual(self, level):
        _ck(lib().ref_stokes_residual(self.h, level))

    def vcycle(self, level, nu1=2, nu2=2):
        _ck(lib().ref_stokes_vcycle(self.h, level, nu1, nu2))

    def solve(self, level, tol, max_cycles, nu1=2, nu2=2):
        """(residual history, converged); raises RefError(3) when a coarse MINRES fails"""
        res = np.zeros(max_cycles + 1)
        n, conv = C.c_int(), C.c_int()
        _ck(lib().ref_stokes_solve(self.h, level, tol, max_cycles, nu1, nu2,
                                   res.ctypes.data_as(C.POINTER(C.c_double)), C.byref(n), C.byref(conv)))
        return res[: n.value], bool(conv.value)

    def residual_norm(self, level) -> float:
        out = C.c_double()
        _ck(lib().ref_stokes_residual_norm(self.h, level, C.byref(out)))
        return out.value

    def pressure_mean(self, level) -> float:
        out = C.c_double()
        _ck(lib().ref_stokes_pressure_mean(self.h, level, C.byref(out)))
        return out.value

    def matrix(self, level):
        n = C.c_int64()
        _ck(lib().ref_stokes_matrix(self.h, level, None, None, None, 0, C.byref(n)))
        r = np.empty(n.value, dtype=np.int64)
        c = np.empty(n.value, dtype=np.int64)
        v = np.empty(n.value)
        _ck(lib().ref_stokes_matrix(self.h, level, r.ctypes.data_as(C.POINTER(C.c_int64)),
                                    c.ctypes.data_as(C.POINTER(C.c_int64)), v.ctypes.data_as(C.POINTER(C.c_double)),
                                    n.value, C.byref(n)))
        return r, c, v


def controller_trace(mesh: str, ranks: int, level: int, dirs, partitioner: int = 0) -> np.ndarray:
    """The reference Controller's unpack sequence for a tracing PackInfo: rows
    (receiver, sender, direction, level, message sender, receiver, direction, level)."""
    d = (C.c_int * max(len(dirs), 1))(*dirs)
    n = C.c_int64()
    _ck(lib().ref_controller_trace(mesh.encode(), ranks, partitioner, 1, level, d, len(dirs), None, 0, C.byref(n)))
    out = np.zeros(n.value, dtype=np.int64)
    _ck(lib().ref_controller_trace(mesh.encode(), ranks, partitioner, 1, level, d, len(dirs),
                                   out.ctypes.data_as(C.POINTER(C.c_int64)), n.value, C.byref(n)))
    return out.reshape(-1, 8)
