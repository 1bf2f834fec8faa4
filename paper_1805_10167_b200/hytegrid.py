"""Reference-shaped host API over the B200 C ABI.

Mirrors the reference's public C++ API for the multigrid hot path
(/root/reference/proj/include/hytegrid/{primitives,function,operators,
solvers}.hpp): same names, argument meaning and error classes, so code written
against ``hytegrid`` ports line by line. Differences, all forced by device
residency:

* values live in HBM; ``ScalarFunction.values(id, level)`` is replaced by
  ``upload`` / ``download`` of owned DoFs in GlobalDoFMap order
  (numbering.hpp:41-43);
* ``interpolate`` with a Python callable evaluates it on the host at the
  owned DoF coordinates (bitwise the reference's for_each_owned_coord) and
  uploads the masked values; ``interpolate_random`` and constants run on the
  device;
* ``Controller`` carries no state: ghost-exchange plans belong to the domain,
  and ``register_function`` is accepted for source compatibility.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from ._lib import (CudaError, HybError, HybRuntimeError, InvalidArgument, LogicError, NcclError,  # noqa: F401
                   OutOfRange, alive, check, lib)

INNER = 1
DIRICHLET = 2
NEUMANN = 4
ALL_DOF_FLAGS = 7
SMOOTH_MASK = INNER | NEUMANN
P1, P2 = 0, 1  # FunctionKind (reference include/hytegrid/indexing.hpp:28)

LAPLACE = 0
MASS = 1
DIV_X = 2
DIV_Y = 3
GRAD_X = 4
GRAD_Y = 5
PSPG = 6
FORMS = {"LAPLACE": LAPLACE, "MASS": MASS, "DIV_X": DIV_X, "DIV_Y": DIV_Y, "GRAD_X": GRAD_X, "GRAD_Y": GRAD_Y,
         "PSPG": PSPG}

SMOOTHERS = {"jacobi": 0, "gs": 1, "colored_gs": 2}

# analytic expressions for interpolate_expr (evaluated on the device)
EXPR_POLY2 = 0   # p0 + p1 x + p2 y + p3 x^2 + p4 x y + p5 y^2
EXPR_SINSIN = 1  # p0 sin(p1 x + p2) sin(p3 y + p4) + p5


def _pd(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _text_call(fn, *args) -> str:
    n = C.c_int64(0)
    check(fn(*args, None, 0, C.byref(n)))
    buf = C.create_string_buffer(n.value + 1)
    check(fn(*args, buf, n.value + 1, C.byref(n)))
    return buf.value.decode()


class meshgen:
    """Fixture meshes in the reference mesh-file format (src/meshgen.cpp)."""

    @staticmethod
    def _gen(kind: str, *params: float) -> str:
        arr = (C.c_double * max(len(params), 1))(*params)
        return _text_call(lib.hyb_meshgen, kind.encode(), arr, len(params))

    @staticmethod
    def unit_triangle() -> str:
        return meshgen._gen("unit_triangle")

    @staticmethod
    def unit_square() -> str:
        return meshgen._gen("unit_square")

    @staticmethod
    def unit_square_reversed() -> str:
        return meshgen._gen("unit_square_reversed")

    @staticmethod
    def square_ring8() -> str:
        return meshgen._gen("square_ring8")

    @staticmethod
    def channel(nx: int, ny: int, width: float = 1.0, height: float = 1.0) -> str:
        return meshgen._gen("channel", nx, ny, width, height)

    @staticmethod
    def annulus(segments: int, layers: int, r_inner: float, r_outer: float) -> str:
        return meshgen._gen("annulus", segments, layers, r_inner, r_outer)

    @staticmethod
    def perturb(mesh_text: str, frac: float, seed: int) -> str:
        return _text_call(lib.hyb_mesh_perturb, mesh_text.encode(), frac, seed)


def mesh_counts(mesh_text: str) -> tuple[int, int, int]:
    nv, ne, nf = C.c_int64(), C.c_int64(), C.c_int64()
    check(lib.hyb_mesh_counts(mesh_text.encode(), C.byref(nv), C.byref(ne), C.byref(nf)))
    return nv.value, ne.value, nf.value


def _partition(mesh_text: str, ranks: int, kind: int, level: int) -> np.ndarray:
    out = np.zeros(sum(mesh_counts(mesh_text)), dtype=np.int32)
    check(lib.hyb_partition(mesh_text.encode(), ranks, kind, level, out.ctypes.data_as(C.POINTER(C.c_int32))))
    return out


def partition_round_robin(mesh_text: str, ranks: int) -> np.ndarray:
    return _partition(mesh_text, ranks, 0, 0)


def partition_greedy_edgecut(mesh_text: str, ranks: int, weight_level: int) -> np.ndarray:
    return _partition(mesh_text, ranks, 1, weight_level)


def stencil_host(mesh_text: str, level: int, primitive_id: int, form: int = 0) -> np.ndarray:
    """Stencil of one primitive assembled on the host (no device needed)."""
    out = np.zeros(64)
    n = C.c_int()
    check(lib.hyb_stencil_host(mesh_text.encode(), form, level, primitive_id, _pd(out), 64, C.byref(n)))
    return out[: n.value].copy()


def coarse_matrix_host(mesh_text: str, level: int, form: int = 0, bc: dict | None = None):
    """GridHierarchy's constrained min-level matrix exactly as the device coarse
    CG holds it, as COO (rows, cols, vals); host only."""
    m, f, nb = _bc_arrays(bc)
    n = C.c_int64()
    check(lib.hyb_coarse_matrix_host(mesh_text.encode(), form, level, m, f, nb, None, None, None, 0, C.byref(n)))
    r = np.empty(n.value, dtype=np.int64)
    c = np.empty(n.value, dtype=np.int64)
    v = np.empty(n.value)
    i64p = C.POINTER(C.c_int64)
    check(lib.hyb_coarse_matrix_host(mesh_text.encode(), form, level, m, f, nb, r.ctypes.data_as(i64p),
                                     c.ctypes.data_as(i64p), _pd(v), n.value, C.byref(n)))
    return r, c, v


class ExchangePlan:
    """Host-only view of the layout and one-round ghost-exchange plan that a
    process driving ``local_ranks`` builds for ``level`` (no device needed)."""

    ARRAYS = {"owned_slots": 0, "owned_global": 1, "gather_dst": 2, "gather_src": 3, "pack_src": 4,
              "owner_global": 5, "inproc": 6, "sends": 7, "recvs": 8}

    def __init__(self, mesh_text: str, ranks: int, assignment, local_ranks, level: int, kind: int = 0):
        a = np.ascontiguousarray(assignment, dtype=np.int32)
        lr = (C.c_int32 * len(local_ranks))(*local_ranks)
        h = C.c_void_p()
        check(lib.hyb_plan_create_kind(mesh_text.encode(), ranks, a.ctypes.data_as(C.POINTER(C.c_int32)), lr,
                                       len(local_ranks), level, kind, C.byref(h)))
        self._h = h
        s = (C.c_int64 * 8)()
        check(lib.hyb_plan_sizes(h, s))
        (self.arena_size, self.owned_local, self.nlocal, self.ntotal, self.npack, self.n_inproc, self.n_sends,
         self.n_recvs) = list(s)

    def __del__(self):
        if getattr(self, "_h", None) and alive():
            lib.hyb_plan_destroy(self._h)
            self._h = None

    def array(self, name: str) -> np.ndarray:
        which = self.ARRAYS[name]
        n = C.c_int64()
        check(lib.hyb_plan_array(self._h, which, None, 0, C.byref(n)))
        out = np.zeros(n.value, dtype=np.int64)
        check(lib.hyb_plan_array(self._h, which, out.ctypes.data_as(C.POINTER(C.c_int64)), n.value, C.byref(n)))
        if which >= 6:
            out = out.reshape(-1, 5)
        return out


def _bc_arrays(bc: dict | None):
    bc = bc or {}
    markers = (C.c_int32 * max(len(bc), 1))(*[int(k) for k in bc])
    flags = (C.c_uint8 * max(len(bc), 1))(*[int(v) for v in bc.values()])
    return markers, flags, len(bc)


class DistributedDomain:
    """Macro-primitive graph distributed over ``ranks`` logical ranks.

    ``local_ranks`` (default: all) are driven by this process on ``device``;
    co-resident ranks exchange ghosts through device copies, remote ranks
    (one per process) through NCCL after ``connect_nccl``.
    """

    def __init__(self, mesh_text: str, ranks: int = 1, assignment=None, local_ranks=None, device: int = 0):
        self.mesh_text = mesh_text
        self.ranks = ranks
        self.counts = mesh_counts(mesh_text)
        if assignment is None:
            assignment = partition_round_robin(mesh_text, ranks)
        self.assignment = np.ascontiguousarray(assignment, dtype=np.int32)
        lr = list(range(ranks)) if local_ranks is None else list(local_ranks)
        lr_arr = (C.c_int32 * len(lr))(*lr)
        h = C.c_void_p()
        check(lib.hyb_domain_create(mesh_text.encode(), ranks, self.assignment.ctypes.data_as(C.POINTER(C.c_int32)),
                                    lr_arr, len(lr), device, C.byref(h)))
        self._h = h
        self.local_ranks = lr

    def __del__(self):
        if getattr(self, "_h", None) and alive():
            lib.hyb_domain_destroy(self._h)
            self._h = None

    @staticmethod
    def nccl_unique_id() -> bytes:
        buf = C.create_string_buffer(128)
        check(lib.hyb_nccl_unique_id(buf))
        return buf.raw

    def connect_nccl(self, uid: bytes, rank: int) -> None:
        check(lib.hyb_domain_connect_nccl(self._h, uid, rank))

    def owned_count(self, level: int) -> tuple[int, int]:
        t, l_ = C.c_int64(), C.c_int64()
        check(lib.hyb_domain_owned_count(self._h, level, C.byref(t), C.byref(l_)))
        return t.value, l_.value

    def arena_bytes(self, level: int) -> int:
        b = C.c_int64()
        check(lib.hyb_domain_arena_bytes(self._h, level, C.byref(b)))
        return b.value

    def coords(self, level: int, global_order: bool = True, kind: int = 0) -> np.ndarray:
        """owned DoF coordinates (for_each_owned_coord, src/layout.cpp:239-282) of a P1 or P2 function"""
        n = self.owned_count(level + (1 if kind == 1 else 0))[0 if global_order else 1]
        xy = np.zeros((n, 2))
        check(lib.hyb_owned_coords_kind(self._h, kind, level, int(global_order), _pd(xy), n))
        return xy

    def overlap(self, enable: bool | None = None) -> int:
        """Toggle communication/computation overlap (default on); returns the
        number of split (interior / boundary) launches so far."""
        n = C.c_int64()
        check(lib.hyb_domain_overlap(self._h, -1 if enable is None else int(enable), C.byref(n)))
        return n.value

    def synchronize(self) -> None:
        check(lib.hyb_domain_synchronize(self._h))

    def profile(self, enable: bool = True) -> None:
        check(lib.hyb_domain_profile(self._h, int(enable)))

    def timer(self, name: str) -> tuple[float, int]:
        ms, cnt = C.c_double(), C.c_int64()
        check(lib.hyb_domain_timer(self._h, name.encode(), C.byref(ms), C.byref(cnt)))
        return ms.value, cnt.value

    def timer_reset(self) -> None:
        check(lib.hyb_domain_timer_reset(self._h))

    def event_record(self, slot: int) -> None:
        check(lib.hyb_domain_event_record(self._h, slot))

    def event_elapsed(self, a: int, b: int) -> float:
        ms = C.c_double()
        check(lib.hyb_domain_event_elapsed(self._h, a, b, C.byref(ms)))
        return ms.value


def kernel_launches() -> int:
    n = C.c_int64()
    check(lib.hyb_kernel_launches(C.byref(n)))
    return n.value


_PACK_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_uint64, C.c_uint64, C.c_int, C.c_int, C.POINTER(C.c_uint8),
                       C.c_int64, C.POINTER(C.c_int64))
_UNPACK_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_uint64, C.c_uint64, C.c_int, C.c_int, C.POINTER(C.c_uint8),
                         C.c_int64, C.POINTER(C.c_int64))


class PackInfo:
    """The reference's extension point (communication.hpp:24-34) for data kept
    on the host: pack(sender, receiver, direction, level) -> bytes and
    unpack(receiver, sender, direction, level, data) -> bytes consumed."""

    def pack(self, sender: int, receiver: int, direction: int, level: int) -> bytes:
        raise NotImplementedError

    def unpack(self, receiver: int, sender: int, direction: int, level: int, data: bytes) -> int:
        raise NotImplementedError


class Controller:
    """hytegrid::Controller: the device fields' exchange plans live in the
    domain; user PackInfo plugins are driven with the reference's schedule."""

    def __init__(self, domain: DistributedDomain):
        self.domain = domain
        self._infos = {}  # channel -> (PackInfo, C callbacks kept alive)

    def register_pack_info(self, channel: int, info: PackInfo) -> None:
        def pack(_user, sender, receiver, direction, level, out, cap, length):
            try:
                data = info.pack(sender, receiver, direction, level)
                length[0] = len(data)
                if out and cap >= len(data):
                    C.memmove(out, data, len(data))
                return 0
            except Exception:  # noqa: BLE001 - reported as the reference's runtime_error
                return 1

        def unpack(_user, receiver, sender, direction, level, data, length, used):
            try:
                used[0] = int(info.unpack(receiver, sender, direction, level, C.string_at(data, length)))
                return 0
            except Exception:  # noqa: BLE001
                return 1

        cbs = (_PACK_FN(pack), _UNPACK_FN(unpack))
        check(lib.hyb_register_pack_info(self.domain._h, channel, C.cast(cbs[0], C.c_void_p),
                                         C.cast(cbs[1], C.c_void_p), None))
        self._infos[channel] = (info, cbs)

    def sync(self, channel: int, level: int, directions) -> None:
        """Controller::sync(channel, level, directions) (src/communication.cpp:126-173)."""
        d = (C.c_int * max(len(directions), 1))(*[int(x) for x in directions])
        check(lib.hyb_controller_sync(self.domain._h, channel, level, d, len(directions)))


def register_function(ctl: Controller, f: "ScalarFunction") -> None:  # noqa: ARG001 - API parity
    return None


class ScalarFunction:
    """P1 or P2 grid function: one HBM arena per level (zero-initialised).
    kind: P1 (default) or P2 (reference FunctionKind, indexing.hpp:28)."""

    def __init__(self, name: str, domain: DistributedDomain, min_level: int, max_level: int, bc: dict | None = None,
                 kind: int = 0):
        self.name = name
        self.domain = domain
        self.min_level = min_level
        self.max_level = max_level
        self.kind = kind
        self.bc = dict(bc or {})
        m, f, n = _bc_arrays(self.bc)
        h = C.c_void_p()
        check(lib.hyb_function_create_kind(domain._h, name.encode(), kind, min_level, max_level, m, f, n, C.byref(h)))
        self._h = h

    def __del__(self):
        if getattr(self, "_h", None) and alive():
            lib.hyb_function_destroy(self._h)
            self._h = None

    def _n(self, level: int, global_order: bool) -> int:
        # a P2 function at level L holds the DoF count of P1 at level L + 1
        return self.domain.owned_count(level + (1 if self.kind == P2 else 0))[0 if global_order else 1]

    def upload(self, level: int, values, global_order: bool = True, mask: int = ALL_DOF_FLAGS) -> None:
        v = np.ascontiguousarray(values, dtype=np.float64)
        check(lib.hyb_function_upload(self._h, level, _pd(v), v.size, int(global_order), mask))

    def download(self, level: int, global_order: bool = True, out: np.ndarray | None = None) -> np.ndarray:
        n = self._n(level, global_order)
        if out is None:
            out = np.empty(n)
        check(lib.hyb_function_download(self._h, level, _pd(out), n, int(global_order)))
        return out

    def upload_async(self, level: int, values: np.ndarray, mask: int = ALL_DOF_FLAGS) -> None:
        """Stream-ordered upload of this process's owned DoFs (local order);
        `values` (float64, contiguous; page-locked for overlap, see
        PinnedBuffer) must stay alive until the domain synchronises."""
        if values.dtype != np.float64 or not values.flags["C_CONTIGUOUS"]:
            raise ValueError("upload_async needs a contiguous float64 array (no temporary copy)")
        check(lib.hyb_function_upload_async(self._h, level, _pd(values), values.size, mask))

    def download_async(self, level: int, out: np.ndarray) -> None:
        """Stream-ordered download into `out` (local order), complete after
        domain.synchronize()."""
        if out.dtype != np.float64 or not out.flags["C_CONTIGUOUS"]:
            raise ValueError("download_async needs a contiguous float64 array")
        check(lib.hyb_function_download_async(self._h, level, _pd(out), out.size))

    def serialize(self, prim: int) -> bytes:
        """The primitive's record in the reference's DataCallbacks::serialize
        format (src/field.cpp:157-175), after a ghost refresh of every level."""
        n = C.c_int64(0)
        check(lib.hyb_function_serialize(self._h, prim, None, 0, C.byref(n)))
        out = np.zeros(n.value, dtype=np.uint8)
        check(lib.hyb_function_serialize(self._h, prim, out.ctypes.data_as(C.POINTER(C.c_uint8)), out.size,
                                         C.byref(n)))
        return out.tobytes()

    def deserialize(self, prim: int, record: bytes) -> None:
        """Inverse of serialize (DataCallbacks::deserialize); the record's
        levels, sizes and flags must match this function."""
        buf = np.frombuffer(bytes(record), dtype=np.uint8).copy()
        check(lib.hyb_function_deserialize(self._h, prim, buf.ctypes.data_as(C.POINTER(C.c_uint8)), buf.size))

    def values(self, prim: int, level: int) -> np.ndarray:
        """values(id, level) (function.hpp:37-39) without a refresh: the
        primitive's slots in the reference layout (an edge's halo row 0, not
        stored on the device, reads as the edge's line)."""
        n = C.c_int64(0)
        check(lib.hyb_function_values(self._h, prim, level, None, 0, C.byref(n)))
        out = np.zeros(n.value)
        check(lib.hyb_function_values(self._h, prim, level, _pd(out), out.size, C.byref(n)))
        return out

    def set_values(self, prim: int, level: int, v) -> None:
        v = np.ascontiguousarray(v, dtype=np.float64)
        check(lib.hyb_function_set_values(self._h, prim, level, _pd(v), v.size))

    def flags(self, level: int, global_order: bool = True) -> np.ndarray:
        n = self._n(level, global_order)
        out = np.zeros(n, dtype=np.uint8)
        check(lib.hyb_function_flags(self._h, level, out.ctypes.data_as(C.POINTER(C.c_uint8)), n,
                                     int(global_order)))
        return out


class StencilOperator:
    """Constant-coefficient P1 operator (LAPLACE or MASS), stencils per level."""

    def __init__(self, domain: DistributedDomain, form: int = LAPLACE, min_level: int = 0, max_level: int = 0,
                 bc: dict | None = None, kind: int = 0):
        self.domain = domain
        self.form = form
        self.kind = kind
        self.min_level = min_level
        self.max_level = max_level
        self.bc = dict(bc or {})
        m, f, n = _bc_arrays(self.bc)
        h = C.c_void_p()
        check(lib.hyb_operator_create_kind(domain._h, form, kind, min_level, max_level, m, f, n, C.byref(h)))
        self._h = h

    def __del__(self):
        if getattr(self, "_h", None) and alive():
            lib.hyb_operator_destroy(self._h)
            self._h = None

    def stencil(self, level: int, primitive_id: int) -> np.ndarray:
        out = np.zeros(64)
        n = C.c_int()
        check(lib.hyb_operator_stencil(self._h, level, primitive_id, _pd(out), 64, C.byref(n)))
        return out[: n.value].copy()


# ---------------------------------------------------------------- operations
def interpolate(f: ScalarFunction, expr, level: int, flag_mask: int = ALL_DOF_FLAGS) -> None:
    """Owned DoFs with flag in mask := expr(x, y) (or a constant)."""
    if callable(expr):
        xy = f.domain.coords(level, global_order=False, kind=f.kind)
        vals = np.asarray(expr(xy[:, 0], xy[:, 1]), dtype=np.float64)
        if vals.shape != (xy.shape[0],):
            vals = np.array([expr(x, y) for x, y in xy], dtype=np.float64)
        f.upload(level, vals, global_order=False, mask=flag_mask)
    else:
        check(lib.hyb_interpolate_const(f._h, float(expr), level, flag_mask))


def interpolate_expr(f: ScalarFunction, level: int, kind: int, params, flag_mask: int = ALL_DOF_FLAGS) -> None:
    """Owned DoFs with flag in mask := an analytic expression (EXPR_POLY2 / EXPR_SINSIN) of the
    reference's DoF coordinates, evaluated on the device: no host coordinates, no upload, so it
    works at sizes the host cannot hold (configuration 4's rhs at level 11 is 137 GB)."""
    p = np.ascontiguousarray(np.asarray(params, dtype=np.float64).ravel())
    check(lib.hyb_interpolate_expr(f._h, level, int(kind), p.ctypes.data if p.size else None, int(p.size),
                                   flag_mask))


def interpolate_random(f: ScalarFunction, level: int, seed: int, stream: int = 0, lo: float = -1.0, hi: float = 1.0,
                       flag_mask: int = ALL_DOF_FLAGS) -> None:
    check(lib.hyb_interpolate_random(f._h, level, seed, stream, lo, hi, flag_mask))


def sync_all(ctl: Controller, f: ScalarFunction, level: int) -> None:  # noqa: ARG001
    check(lib.hyb_sync(f._h, level))


# reference Direction (transport.hpp:19-26)
VERTEX_TO_EDGE, EDGE_TO_FACE, FACE_TO_EDGE, EDGE_TO_VERTEX = 0, 1, 2, 3
FULL_SYNC_SCHEDULE = (VERTEX_TO_EDGE, EDGE_TO_FACE, FACE_TO_EDGE, EDGE_TO_VERTEX)


def sync(ctl: Controller, f: ScalarFunction, level: int, directions) -> None:  # noqa: ARG001
    """sync(c, f, level, span<Direction>) (src/function.cpp:234-237): the given
    relay directions in order, each exactly as the reference's pack/unpack."""
    d = (C.c_int * max(len(directions), 1))(*[int(x) for x in directions])
    check(lib.hyb_sync_directions(f._h, level, d, len(directions)))


def apply(A: StencilOperator, ctl: Controller, src: ScalarFunction, dst: ScalarFunction, level: int,  # noqa: ARG001
          flag_mask: int = ALL_DOF_FLAGS) -> None:
    check(lib.hyb_apply(A._h, src._h, dst._h, level, flag_mask))


def residual(A: StencilOperator, ctl: Controller, rhs: ScalarFunction, x: ScalarFunction,  # noqa: ARG001
             r: ScalarFunction, level: int) -> None:
    check(lib.hyb_residual(A._h, rhs._h, x._h, r._h, level))


def smooth_gs(A: StencilOperator, ctl: Controller, rhs: ScalarFunction, x: ScalarFunction,  # noqa: ARG001
              level: int) -> None:
    """Hybrid Gauss-Seidel (reference smooth_gs), bitwise the reference's."""
    check(lib.hyb_smooth_gs(A._h, rhs._h, x._h, level))


def smooth_colored_gs(A: StencilOperator, ctl: Controller, rhs: ScalarFunction,  # noqa: ARG001
                      x: ScalarFunction, level: int, count: int = 1) -> None:
    """Coloured hybrid Gauss-Seidel: faces by (c + 2r) mod 3, edges odd/even k. With count > 1,
    `count` sweeps (consecutive pairs in one face pass where possible; bitwise the same)."""
    if count == 1:
        check(lib.hyb_smooth_cgs(A._h, rhs._h, x._h, level))
    else:
        check(lib.hyb_smooth_cgs_n(A._h, rhs._h, x._h, level, count))


def smooth_jacobi(A: StencilOperator, ctl: Controller, rhs: ScalarFunction, x: ScalarFunction,  # noqa: ARG001
                  omega: float, level: int) -> None:
    check(lib.hyb_smooth_jacobi(A._h, rhs._h, x._h, omega, level))


def smooth_jacobi2(A: StencilOperator, ctl: Controller, rhs: ScalarFunction, x: ScalarFunction,  # noqa: ARG001
                   omega: float, level: int) -> None:
    """Two smooth_jacobi sweeps, bitwise, in one pass over the faces (temporal blocking)."""
    check(lib.hyb_smooth_jacobi2(A._h, rhs._h, x._h, omega, level))


def tuning(name: str, value: int = -1) -> int:
    """Set a measurement knob (value >= 0) and return its previous value."""
    prev = C.c_int64()
    check(lib.hyb_tuning(name.encode(), value, C.byref(prev)))
    return prev.value


def diagonal(A: StencilOperator, d: ScalarFunction, level: int) -> None:
    check(lib.hyb_diagonal(A._h, d._h, level))


def prolongate(ctl: Controller, coarse: ScalarFunction, fine: ScalarFunction, coarse_level: int,  # noqa: ARG001
               flag_mask: int = ALL_DOF_FLAGS) -> None:
    check(lib.hyb_prolongate(coarse._h, fine._h, coarse_level, flag_mask))


def prolongate_add(ctl: Controller, coarse: ScalarFunction, fine: ScalarFunction, coarse_level: int,  # noqa: ARG001
                   flag_mask: int = ALL_DOF_FLAGS) -> None:
    check(lib.hyb_prolongate_add(coarse._h, fine._h, coarse_level, flag_mask))


def restrict_to_coarse(ctl: Controller, fine: ScalarFunction, coarse: ScalarFunction, coarse_level: int,  # noqa
                       flag_mask: int = ALL_DOF_FLAGS) -> None:
    check(lib.hyb_restrict(fine._h, coarse._h, coarse_level, flag_mask))


def residual_restrict(A: StencilOperator, ctl: Controller, rhs: ScalarFunction, x: ScalarFunction,  # noqa: ARG001
                      r: ScalarFunction, coarse: ScalarFunction, coarse_level: int) -> None:
    """coarse := P^T (rhs - A x) at coarse_level, fused on face interiors (the
    V-cycle's residual + restrict_to_coarse); r is scratch."""
    check(lib.hyb_residual_restrict(A._h, rhs._h, x._h, r._h, coarse._h, coarse_level))


def prolongate_add_jacobi(A: StencilOperator, ctl: Controller, e: ScalarFunction, rhs: ScalarFunction,  # noqa: ARG001
                          x: ScalarFunction, omega: float, coarse_level: int) -> None:
    """prolongate_add(e -> x, smooth mask) then smooth_jacobi(rhs, x, omega),
    fused (the V-cycle's correction and first post-smoothing sweep)."""
    check(lib.hyb_prolongate_add_jacobi(A._h, e._h, rhs._h, x._h, omega, coarse_level))


def prolongate_add_colored_gs(A: StencilOperator, ctl: Controller, e: ScalarFunction,  # noqa: ARG001
                              rhs: ScalarFunction, x: ScalarFunction, coarse_level: int) -> None:
    """prolongate_add(e -> x, smooth mask) then smooth_colored_gs(rhs, x), fused on faces of
    n >= 256 (the V-cycle's correction and first coloured post-sweep); bitwise the two calls."""
    check(lib.hyb_prolongate_add_cgs(A._h, e._h, rhs._h, x._h, coarse_level))


def assign(alpha: float, x1: ScalarFunction, beta: float, x2: ScalarFunction, dst: ScalarFunction, level: int,
           flag_mask: int = ALL_DOF_FLAGS) -> None:
    check(lib.hyb_assign(alpha, x1._h, beta, x2._h, dst._h, level, flag_mask))


def add_scaled(dst: ScalarFunction, gamma: float, y: ScalarFunction, level: int,
               flag_mask: int = ALL_DOF_FLAGS) -> None:
    check(lib.hyb_add_scaled(dst._h, gamma, y._h, level, flag_mask))


def dot(a: ScalarFunction, b: ScalarFunction, level: int) -> float:
    out = C.c_double()
    check(lib.hyb_dot(a._h, b._h, level, C.byref(out)))
    return out.value


def norm2(a: ScalarFunction, level: int) -> float:
    out = C.c_double()
    check(lib.hyb_norm2(a._h, level, C.byref(out)))
    return out.value


def max_abs(a: ScalarFunction, level: int) -> float:
    out = C.c_double()
    check(lib.hyb_max_abs(a._h, level, C.byref(out)))
    return out.value


@dataclass
class SolveReport:
    """reference include/hytegrid/solvers.hpp:42-50"""
    converged: bool = False
    iterations: int = 0
    residuals: list = field(default_factory=list)

    def history(self) -> str:
        lines = []
        for k, r in enumerate(self.residuals):
            if k == 0:
                lines.append(f"cycle {k} residual {r:.6e}")
            else:
                prev = self.residuals[k - 1]
                f = r / prev if prev > 0 else 0.0
                lines.append(f"cycle {k} residual {r:.6e} factor {f:.4f}")
        return "\n".join(lines) + "\n"


class GridHierarchy:
    """V-cycle multigrid (reference GridHierarchy, solvers.hpp:81-102).

    smoother 'gs' (default: the reference's hybrid Gauss-Seidel, hardcoded at
    src/solvers.cpp:417, 427), 'jacobi' with weight omega, or 'colored_gs';
    coarse level solved on the device by CG to coarse_tol (reference default
    1e-12, max_iter #DoFs + 100).
    """

    def __init__(self, domain: DistributedDomain, ctl: Controller, form: int, min_level: int, max_level: int,  # noqa
                 bc: dict | None = None, smoother: str = "gs", omega: float = 2.0 / 3.0,
                 coarse_tol: float = 1e-12, coarse_max_iter: int = -1):
        self.domain = domain
        self.min_level = min_level
        self.max_level = max_level
        m, f, n = _bc_arrays(bc)
        h = C.c_void_p()
        check(lib.hyb_hierarchy_create(domain._h, form, min_level, max_level, m, f, n, SMOOTHERS[smoother], omega,
                                       coarse_tol, coarse_max_iter, C.byref(h)))
        self._h = h

    def __del__(self):
        if getattr(self, "_h", None) and alive():
            lib.hyb_hierarchy_destroy(self._h)
            self._h = None

    def vcycle(self, rhs: ScalarFunction, x: ScalarFunction, level: int, nu_pre: int = 2, nu_post: int = 2) -> None:
        check(lib.hyb_hierarchy_vcycle(self._h, rhs._h, x._h, level, nu_pre, nu_post))

    def use_graphs(self, enable: bool | None = None) -> int:
        """Toggle CUDA-graph replay of V-cycles; returns graph launches so far."""
        n = C.c_int64()
        check(lib.hyb_hierarchy_graphs(self._h, -1 if enable is None else int(enable), C.byref(n)))
        return n.value

    def residual_norm(self, rhs: ScalarFunction, x: ScalarFunction, level: int) -> float:
        out = C.c_double()
        check(lib.hyb_hierarchy_residual_norm(self._h, rhs._h, x._h, level, C.byref(out)))
        return out.value

    def use_mega(self, enable: bool | str | None = None, max_n: int = 0) -> int:
        """The one-kernel coarse end of Jacobi cycles (levels with 2^level <= max_n): True
        always, False never, "auto" (default) on small domains; returns such launches so far."""
        n = C.c_int64()
        mode = -1 if enable is None else (2 if enable == "auto" else int(bool(enable)))
        check(lib.hyb_hierarchy_mega(self._h, mode, max_n, C.byref(n)))
        return n.value

    def use_temporal(self, enable: bool | None = None) -> bool:
        """Toggle the two-sweep pre-smoothing pass of Jacobi V(2, >=2) cycles (default on)."""
        st = C.c_int()
        check(lib.hyb_hierarchy_temporal(self._h, -1 if enable is None else int(enable), C.byref(st)))
        return bool(st.value)

    def solve(self, rhs: ScalarFunction, x: ScalarFunction, level: int, tol: float, max_cycles: int,
              nu_pre: int = 2, nu_post: int = 2) -> SolveReport:
        res = np.zeros(max_cycles + 1)
        n = C.c_int()
        conv = C.c_int()
        check(lib.hyb_hierarchy_solve(self._h, rhs._h, x._h, level, tol, max_cycles, nu_pre, nu_post, _pd(res),
                                      C.byref(n), C.byref(conv)))
        return SolveReport(bool(conv.value), n.value - 1, list(res[: n.value]))

    def fmg(self, rhs: ScalarFunction, x: ScalarFunction, level: int, tol: float, max_cycles: int,
            nu_pre: int = 2, nu_post: int = 2, cycles_per_level: int = 1) -> SolveReport:
        """Full multigrid then V-cycles to tol * ||r(x = 0)|| (no reference
        counterpart; configuration 4). rhs is given at `level`; its coarser
        levels are overwritten by restriction. residuals[0] = ||r(x = 0)||,
        [1] after the FMG sweep, then one per cycle; iterations counts the
        cycles after the sweep."""
        res = np.zeros(max_cycles + 2)
        n = C.c_int()
        conv = C.c_int()
        check(lib.hyb_hierarchy_fmg(self._h, rhs._h, x._h, level, cycles_per_level, nu_pre, nu_post, tol, max_cycles,
                                    _pd(res), C.byref(n), C.byref(conv)))
        return SolveReport(bool(conv.value), n.value - 2, list(res[: n.value]))

    def pcg(self, rhs: ScalarFunction, x: ScalarFunction, level: int, max_iter: int, tol: float = 0.0,
            nu_pre: int = 1, nu_post: int = 1) -> SolveReport:
        """CG preconditioned by one V(nu_pre, nu_post) cycle (configuration 5);
        x starts at zero. residuals[k] = ||r_k||."""
        res = np.zeros(max_iter + 1)
        n = C.c_int()
        conv = C.c_int()
        check(lib.hyb_hierarchy_pcg(self._h, rhs._h, x._h, level, max_iter, nu_pre, nu_post, tol, _pd(res),
                                    C.byref(n), C.byref(conv)))
        return SolveReport(bool(conv.value), n.value - 1, list(res[: n.value]))



# ---- P1-P1-PSPG Stokes (include/hytegrid/solvers.hpp:117-236) ----

class StokesState:
    """u1, u2 (velocity BCs) and p (pressure BCs) (reference StokesState)."""

    def __init__(self, name: str, domain: DistributedDomain, min_level: int, max_level: int,
                 bc_velocity: dict | None = None, bc_pressure: dict | None = None):
        self.u1 = ScalarFunction(name + ".u1", domain, min_level, max_level, bc_velocity)
        self.u2 = ScalarFunction(name + ".u2", domain, min_level, max_level, bc_velocity)
        self.p = ScalarFunction(name + ".p", domain, min_level, max_level, bc_pressure)

    def _arr(self):
        return (C.c_void_p * 3)(self.u1._h, self.u2._h, self.p._h)

    def components(self):
        return (self.u1, self.u2, self.p)


def register_state(ctl: Controller, s: StokesState) -> None:  # noqa: ARG001 - API parity
    """register_state: every function of the domain shares the exchange plan."""


def stokes_dot(a: StokesState, b: StokesState, level: int) -> float:
    out = C.c_double()
    check(lib.hyb_stokes_dot(a._arr(), b._arr(), level, C.byref(out)))
    return out.value


class _StokesHandle:
    def __init__(self, domain, min_level, max_level, bc_velocity, bc_pressure, multigrid, project, omega):
        mu, fu, nu = _bc_arrays(bc_velocity)
        mp, fp, npr = _bc_arrays(bc_pressure)
        h = C.c_void_p()
        check(lib.hyb_stokes_create(domain._h, min_level, max_level, mu, fu, nu, mp, fp, npr, int(multigrid),
                                    int(project), omega, C.byref(h)))
        self._h = h
        self.domain = domain
        self.min_level, self.max_level = min_level, max_level

    def __del__(self):
        if getattr(self, "_h", None) and alive():
            lib.hyb_stokes_destroy(self._h)
            self._h = None


class StokesSystem(_StokesHandle):
    """Operator blocks A (per velocity component), G = (GRAD_X, GRAD_Y),
    B = (DIV_X, DIV_Y) and the PSPG block C (reference StokesSystem)."""

    def __init__(self, domain: DistributedDomain, min_level: int, max_level: int, bc_velocity: dict | None = None,
                 bc_pressure: dict | None = None):
        super().__init__(domain, min_level, max_level, bc_velocity, bc_pressure, False, False, 0.3)


def uzawa_smooth(S, ctl: Controller, rhs: StokesState, x: StokesState, level: int,  # noqa: ARG001
                 omega: float = 0.3) -> None:
    """One inexact-Uzawa sweep (src/solvers.cpp:506-546); S is a StokesSystem
    or a StokesMultigrid's system()."""
    check(lib.hyb_uzawa_smooth(S._h, rhs._arr(), x._arr(), level, omega))


def stokes_residual(S, ctl: Controller, rhs: StokesState, x: StokesState, r: StokesState,  # noqa: ARG001
                    level: int) -> None:
    check(lib.hyb_stokes_residual(S._h, rhs._arr(), x._arr(), r._arr(), level))


class StokesMultigrid(_StokesHandle):
    """Monolithic Uzawa-smoothed multigrid with a device MINRES on the
    assembled min-level system (reference StokesMultigrid)."""

    def __init__(self, domain: DistributedDomain, ctl: Controller, min_level: int, max_level: int,  # noqa: ARG002
                 bc_velocity: dict | None = None, bc_pressure: dict | None = None,
                 project_pressure_mean: bool = False, omega: float = 0.3):
        super().__init__(domain, min_level, max_level, bc_velocity, bc_pressure, True, project_pressure_mean, omega)

    def system(self) -> "StokesMultigrid":
        return self

    def vcycle(self, rhs: StokesState, x: StokesState, level: int, nu_pre: int = 2, nu_post: int = 2) -> None:
        check(lib.hyb_stokes_vcycle(self._h, rhs._arr(), x._arr(), level, nu_pre, nu_post))

    def solve(self, rhs: StokesState, x: StokesState, level: int, tol: float, max_cycles: int, nu_pre: int = 2,
              nu_post: int = 2) -> SolveReport:
        res = np.zeros(max_cycles + 1)
        n = C.c_int()
        conv = C.c_int()
        check(lib.hyb_stokes_solve(self._h, rhs._arr(), x._arr(), level, tol, max_cycles, nu_pre, nu_post, _pd(res),
                                   C.byref(n), C.byref(conv)))
        return SolveReport(bool(conv.value), n.value - 1, list(res[: n.value]))

    def residual_norm(self, rhs: StokesState, x: StokesState, level: int) -> float:
        out = C.c_double()
        check(lib.hyb_stokes_residual_norm(self._h, rhs._arr(), x._arr(), level, C.byref(out)))
        return out.value

    def pressure_mean(self, p: ScalarFunction, level: int) -> float:
        out = C.c_double()
        check(lib.hyb_stokes_pressure_mean(self._h, p._h, level, C.byref(out)))
        return out.value

    def coarse_iterations(self) -> int:
        out = C.c_int()
        check(lib.hyb_stokes_coarse_iterations(self._h, C.byref(out)))
        return out.value


def stokes_matrix_host(mesh_text: str, level: int, bc_velocity: dict | None = None, bc_pressure: dict | None = None):
    """StokesMultigrid's constrained monolithic min-level matrix (COO), host only."""
    mu, fu, nu = _bc_arrays(bc_velocity)
    mp, fp, npr = _bc_arrays(bc_pressure)
    n = C.c_int64()
    check(lib.hyb_stokes_matrix_host(mesh_text.encode(), level, mu, fu, nu, mp, fp, npr, None, None, None, 0,
                                     C.byref(n)))
    r = np.empty(n.value, dtype=np.int64)
    c = np.empty(n.value, dtype=np.int64)
    v = np.empty(n.value)
    check(lib.hyb_stokes_matrix_host(mesh_text.encode(), level, mu, fu, nu, mp, fp, npr,
                                     r.ctypes.data_as(C.POINTER(C.c_int64)), c.ctypes.data_as(C.POINTER(C.c_int64)),
                                     _pd(v), n.value, C.byref(n)))
    return r, c, v

class PinnedBuffer:
    """Page-locked host memory (for end-to-end H2D/D2H timing)."""

    def __init__(self, n_doubles: int):
        p = C.c_void_p()
        check(lib.hyb_host_alloc(n_doubles * 8, C.byref(p)))
        self._p = p
        self.array = np.ctypeslib.as_array(C.cast(p, C.POINTER(C.c_double)), shape=(n_doubles,))

    def __del__(self):
        if getattr(self, "_p", None) and alive():
            lib.hyb_host_free(self._p)
            self._p = None
