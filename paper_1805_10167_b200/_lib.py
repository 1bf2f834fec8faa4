"""ctypes binding of the C ABI in include/hyteg_b200.h.

The shared library is built in-tree (``make lib`` / ``__graft_entry__.build()``)
and is the only compute path: importing this module without the library
raises, there is no fallback.
"""
from __future__ import annotations

import atexit
import ctypes as C
import os
import re

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libhyteg_b200.so")
HEADER_PATH = os.path.join(os.path.dirname(_HERE), "include", "hyteg_b200.h")


class HybError(Exception):
    """Base of all errors raised through the C ABI."""


class InvalidArgument(HybError, ValueError):
    """std::invalid_argument in the reference."""


class OutOfRange(HybError, IndexError):
    """std::out_of_range in the reference."""


class HybRuntimeError(HybError, RuntimeError):
    """std::runtime_error in the reference."""


class LogicError(HybError):
    """std::logic_error in the reference."""


class CudaError(HybError):
    pass


class NcclError(HybError):
    pass


_STATUS = {1: InvalidArgument, 2: OutOfRange, 3: HybRuntimeError, 4: LogicError, 5: CudaError, 6: NcclError,
           7: HybError}

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: build it with `make lib` (or __graft_entry__.build()); "
                      "there is no CPU fallback for the hot path")

lib = C.CDLL(LIB_PATH)

_p = C.c_void_p
_i = C.c_int
_i64 = C.c_int64
_u64 = C.c_uint64
_u8 = C.c_uint8
_d = C.c_double
_pd = C.POINTER(C.c_double)
_pi32 = C.POINTER(C.c_int32)
_pu8 = C.POINTER(C.c_uint8)
_pi64 = C.POINTER(C.c_int64)
_cs = C.c_char_p

_SIGS = {
    "hyb_last_error": (C.c_char_p, []),
    "hyb_abi_version": (_i, []),
    "hyb_meshgen": (_i, [_cs, _pd, _i, C.c_char_p, _i64, _pi64]),
    "hyb_mesh_perturb": (_i, [_cs, _d, _u64, C.c_char_p, _i64, _pi64]),
    "hyb_mesh_counts": (_i, [_cs, _pi64, _pi64, _pi64]),
    "hyb_partition": (_i, [_cs, _i, _i, _i, _pi32]),
    "hyb_stencil_host": (_i, [_cs, _i, _i, _u64, _pd, _i, C.POINTER(_i)]),
    "hyb_coarse_matrix_host": (_i, [_cs, _i, _i, _pi32, C.POINTER(C.c_uint8), _i, _pi64, _pi64, _pd, _i64, _pi64]),
    "hyb_plan_create": (_i, [_cs, _i, _pi32, _pi32, _i, _i, C.POINTER(_p)]),
    "hyb_plan_destroy": (_i, [_p]),
    "hyb_plan_sizes": (_i, [_p, _pi64]),
    "hyb_plan_array": (_i, [_p, _i, _pi64, _i64, _pi64]),
    "hyb_domain_create": (_i, [_cs, _i, _pi32, _pi32, _i, _i, C.POINTER(_p)]),
    "hyb_domain_destroy": (_i, [_p]),
    "hyb_nccl_unique_id": (_i, [C.c_char_p]),
    "hyb_domain_connect_nccl": (_i, [_p, C.c_char_p, _i]),
    "hyb_domain_owned_count": (_i, [_p, _i, _pi64, _pi64]),
    "hyb_domain_arena_bytes": (_i, [_p, _i, _pi64]),
    "hyb_domain_synchronize": (_i, [_p]),
    "hyb_domain_profile": (_i, [_p, _i]),
    "hyb_domain_timer": (_i, [_p, _cs, _pd, _pi64]),
    "hyb_domain_timer_reset": (_i, [_p]),
    "hyb_domain_event_record": (_i, [_p, _i]),
    "hyb_domain_event_elapsed": (_i, [_p, _i, _i, _pd]),
    "hyb_kernel_launches": (_i, [_pi64]),
    "hyb_owned_coords": (_i, [_p, _i, _i, _pd, _i64]),
    "hyb_function_create": (_i, [_p, _cs, _i, _i, _pi32, _pu8, _i, C.POINTER(_p)]),
    "hyb_function_destroy": (_i, [_p]),
    "hyb_function_upload": (_i, [_p, _i, _pd, _i64, _i, _u8]),
    "hyb_function_download": (_i, [_p, _i, _pd, _i64, _i]),
    "hyb_function_upload_async": (_i, [_p, _i, _pd, _i64, _u8]),
    "hyb_function_download_async": (_i, [_p, _i, _pd, _i64]),
    "hyb_function_flags": (_i, [_p, _i, _pu8, _i64, _i]),
    "hyb_function_serialize": (_i, [_p, _u64, _pu8, _i64, C.POINTER(_i64)]),
    "hyb_function_deserialize": (_i, [_p, _u64, _pu8, _i64]),
    "hyb_interpolate_const": (_i, [_p, _d, _i, _u8]),
    "hyb_interpolate_random": (_i, [_p, _i, _u64, _u64, _d, _d, _u8]),
    "hyb_interpolate_expr": (_i, [_p, _i, _i, _p, _i, _u8]),
    "hyb_sync": (_i, [_p, _i]),
    "hyb_sync_directions": (_i, [_p, _i, C.POINTER(_i), _i]),
    "hyb_function_values": (_i, [_p, _u64, _i, _pd, _i64, _pi64]),
    "hyb_function_set_values": (_i, [_p, _u64, _i, _pd, _i64]),
    "hyb_operator_create": (_i, [_p, _i, _i, _i, _pi32, _pu8, _i, C.POINTER(_p)]),
    "hyb_operator_destroy": (_i, [_p]),
    "hyb_operator_stencil": (_i, [_p, _i, _u64, _pd, _i, C.POINTER(_i)]),
    "hyb_apply": (_i, [_p, _p, _p, _i, _u8]),
    "hyb_residual": (_i, [_p, _p, _p, _p, _i]),
    "hyb_smooth_jacobi": (_i, [_p, _p, _p, _d, _i]),
    "hyb_smooth_gs": (_i, [_p, _p, _p, _i]),
    "hyb_smooth_cgs": (_i, [_p, _p, _p, _i]),
    "hyb_diagonal": (_i, [_p, _p, _i]),
    "hyb_prolongate": (_i, [_p, _p, _i, _u8]),
    "hyb_prolongate_add": (_i, [_p, _p, _i, _u8]),
    "hyb_restrict": (_i, [_p, _p, _i, _u8]),
    "hyb_residual_restrict": (_i, [_p, _p, _p, _p, _p, _i]),
    "hyb_prolongate_add_jacobi": (_i, [_p, _p, _p, _p, _d, _i]),
    "hyb_prolongate_add_cgs": (_i, [_p, _p, _p, _p, _i]),
    "hyb_assign": (_i, [_d, _p, _d, _p, _p, _i, _u8]),
    "hyb_add_scaled": (_i, [_p, _d, _p, _i, _u8]),
    "hyb_dot": (_i, [_p, _p, _i, _pd]),
    "hyb_norm2": (_i, [_p, _i, _pd]),
    "hyb_max_abs": (_i, [_p, _i, _pd]),
    "hyb_hierarchy_create": (_i, [_p, _i, _i, _i, _pi32, _pu8, _i, _i, _d, _d, _i, C.POINTER(_p)]),
    "hyb_hierarchy_destroy": (_i, [_p]),
    "hyb_hierarchy_vcycle": (_i, [_p, _p, _p, _i, _i, _i]),
    "hyb_hierarchy_graphs": (_i, [_p, _i, _pi64]),
    "hyb_hierarchy_residual_norm": (_i, [_p, _p, _p, _i, _pd]),
    "hyb_hierarchy_solve": (_i, [_p, _p, _p, _i, _d, _i, _i, _i, _pd, C.POINTER(_i), C.POINTER(_i)]),
    "hyb_hierarchy_fmg": (_i, [_p, _p, _p, _i, _i, _i, _i, _d, _i, _pd, C.POINTER(_i), C.POINTER(_i)]),
    "hyb_hierarchy_pcg": (_i, [_p, _p, _p, _i, _i, _i, _i, _d, _pd, C.POINTER(_i), C.POINTER(_i)]),
    "hyb_function_create_kind": (_i, [_p, _cs, _i, _i, _i, _pi32, _pu8, _i, C.POINTER(_p)]),
    "hyb_function_kind": (_i, [_p, C.POINTER(_i)]),
    "hyb_domain_overlap": (_i, [_p, _i, _pi64]),
    "hyb_smooth_jacobi2": (_i, [_p, _p, _p, _d, _i]),
    "hyb_tuning": (_i, [_cs, _i64, _pi64]),
    "hyb_plan_create_kind": (_i, [_cs, _i, _pi32, _pi32, _i, _i, _i, C.POINTER(_p)]),
    "hyb_hierarchy_temporal": (_i, [_p, _i, C.POINTER(_i)]),
    "hyb_hierarchy_mega": (_i, [_p, _i, _i, _pi64]),
    "hyb_register_pack_info": (_i, [_p, C.c_uint32, _p, _p, _p]),
    "hyb_controller_sync": (_i, [_p, C.c_uint32, _i, C.POINTER(_i), _i]),
    "hyb_owned_coords_kind": (_i, [_p, _i, _i, _i, _pd, _i64]),
    "hyb_operator_create_kind": (_i, [_p, _i, _i, _i, _i, _pi32, _pu8, _i, C.POINTER(_p)]),
    "hyb_stokes_create": (_i, [_p, _i, _i, _pi32, _pu8, _i, _pi32, _pu8, _i, _i, _i, _d, C.POINTER(_p)]),
    "hyb_stokes_destroy": (_i, [_p]),
    "hyb_uzawa_smooth": (_i, [_p, C.POINTER(_p), C.POINTER(_p), _i, _d]),
    "hyb_stokes_residual": (_i, [_p, C.POINTER(_p), C.POINTER(_p), C.POINTER(_p), _i]),
    "hyb_stokes_dot": (_i, [C.POINTER(_p), C.POINTER(_p), _i, _pd]),
    "hyb_stokes_vcycle": (_i, [_p, C.POINTER(_p), C.POINTER(_p), _i, _i, _i]),
    "hyb_stokes_solve": (_i, [_p, C.POINTER(_p), C.POINTER(_p), _i, _d, _i, _i, _i, _pd, C.POINTER(_i),
                              C.POINTER(_i)]),
    "hyb_stokes_residual_norm": (_i, [_p, C.POINTER(_p), C.POINTER(_p), _i, _pd]),
    "hyb_stokes_pressure_mean": (_i, [_p, _p, _i, _pd]),
    "hyb_stokes_coarse_iterations": (_i, [_p, C.POINTER(_i)]),
    "hyb_stokes_matrix_host": (_i, [_cs, _i, _pi32, _pu8, _i, _pi32, _pu8, _i, _pi64, _pi64, _pd, _i64, _pi64]),
    "hyb_coarse_hypot": (_d, [_d, _d]),
    "hyb_host_alloc": (_i, [_i64, C.POINTER(_p)]),
    "hyb_host_free": (_i, [_p]),
}

for _name, (_res, _args) in _SIGS.items():
    _fn = getattr(lib, _name)
    _fn.restype = _res
    _fn.argtypes = _args


_state = {"alive": True}


@atexit.register
def _mark_shutdown() -> None:
    # handles still alive at interpreter exit are left to process teardown:
    # destroying them while the CUDA runtime shuts down is unsafe
    _state["alive"] = False


def alive() -> bool:
    return _state["alive"]


def check(status: int) -> None:
    if status != 0:
        msg = lib.hyb_last_error().decode(errors="replace")
        raise _STATUS.get(status, HybError)(msg)


def header_symbols() -> list[str]:
    """Every function the public header declares."""
    with open(HEADER_PATH) as fh:
        text = fh.read()
    return sorted(set(re.findall(r"\b(hyb_[a-z0-9_]+)\s*\(", text)))
