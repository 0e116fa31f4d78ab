"""ctypes binding of libmagiplan.so — the C ABI in include/magiplan.h.

This is exactly the binding a reference consumer would write against the
reference's magiplan.h. Loading fails loudly: there is
no Python or CPU fallback for any entry point.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

_LIB_PATH = Path(__file__).resolve().parent / "libmagiplan.so"

OK, ERR_USAGE, ERR_CONSTRAINT, ERR_INTERNAL = 0, 2, 3, 4
COUNT_MULTIPLICITY, COUNT_UNION = 0, 1
F32, BF16 = 0, 1

_vp, _i64, _i32, _f32, _cp = C.c_void_p, C.c_int64, C.c_int32, C.c_float, C.c_char_p
_pi64, _pi32, _pf32 = C.POINTER(C.c_int64), C.POINTER(C.c_int32), C.POINTER(C.c_float)

# name -> (restype, argtypes); mirrors include/magiplan.h one to one.
SIGNATURES: dict[str, tuple] = {
    "magiplan_version": (_cp, []),
    "magiplan_last_error": (_cp, []),
    "magiplan_string_free": (None, [_vp]),
    "magiplan_mask_parse": (C.c_int, [_cp, C.POINTER(_vp)]),
    "magiplan_mask_free": (None, [_vp]),
    "magiplan_mask_area": (C.c_int, [_vp, C.c_int, _pi64]),
    "magiplan_mask_is_allowed": (C.c_int, [_vp, _i64, _i64, C.POINTER(C.c_int)]),
    "magiplan_mask_render": (C.c_int, [_vp, C.POINTER(_vp)]),
    "magiplan_mask_describe": (C.c_int, [_vp, C.POINTER(_vp)]),
    "magiplan_scenario_parse": (C.c_int, [_cp, _cp, C.POINTER(_vp)]),
    "magiplan_scenario_free": (None, [_vp]),
    "magiplan_scenario_set_seed": (C.c_int, [_vp, C.c_uint64]),
    "magiplan_scenario_plan": (C.c_int, [_vp, C.POINTER(_vp)]),
    "magiplan_scenario_simulate": (C.c_int, [_vp, C.c_int, C.POINTER(_vp)]),
    "magiplan_pack_run": (C.c_int, [_cp, _cp, C.POINTER(_vp)]),
    "magiplan_scenario_exec_plan": (C.c_int, [_vp, C.POINTER(_vp)]),
    "magiplan_ffa_plan_create": (C.c_int, [_pi64, _pi64, _pi32, _i64, _i64, _i64, _i32, C.POINTER(_vp)]),
    "magiplan_ffa_plan_from_mask": (C.c_int, [_vp, _i32, C.POINTER(_vp)]),
    "magiplan_ffa_plan_free": (None, [_vp]),
    "magiplan_ffa_plan_describe": (C.c_int, [_vp, C.POINTER(_vp)]),
    "magiplan_ffa_plan_prepare": (C.c_int, [_vp]),
    "magiplan_ffa_fwd": (C.c_int, [_vp, _vp, _vp, _vp, _vp, _vp, _i64, _i64, _f32, _i32, _i32, _vp]),
    "magiplan_ffa_bwd_preprocess": (C.c_int, [_vp, _vp, _vp, _i64, _i64, _i32, _i32, _vp]),
    "magiplan_ffa_bwd": (C.c_int, [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _i64, _i64, _f32, _i32, _i32, _vp]),
    "magiplan_ffa_bwd_stage": (C.c_int, [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _i64, _i64, _f32, _vp]),
    "magiplan_ffa_bwd_dkdv": (C.c_int, [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _i64, _i64, _f32, _i32, _i32, _vp]),
    "magiplan_ffa_bwd_dq": (C.c_int, [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _i64, _i64, _f32, _i32, _i32, _vp]),
    "magiplan_cp_unique_id": (C.c_int, [_vp]),
    "magiplan_cp_create": (C.c_int, [_vp, _i32, _vp, _i64, _i64, _i32, _f32, C.POINTER(_vp)]),
    "magiplan_cp_create_ex": (C.c_int, [_vp, _i32, _vp, _i64, _i64, _i32, _f32, _i32, C.POINTER(_vp)]),
    "magiplan_cp_free": (None, [_vp]),
    "magiplan_cp_describe": (C.c_int, [_vp, C.POINTER(_vp)]),
    "magiplan_cp_forward": (C.c_int, [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "magiplan_cp_backward": (C.c_int, [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "magiplan_range_gather": (C.c_int, [_vp, _vp, _vp, _vp, _i64, _i64, _i64, _vp]),
    "magiplan_range_scatter_add_f32": (C.c_int, [_vp, _vp, _vp, _vp, _i64, _i64, _i64, _vp]),
    "magiplan_cast_f32_bf16": (C.c_int, [_vp, _vp, _i64, _vp]),
    "magiplan_p2p_malloc": (C.c_int, [_i64, C.POINTER(C.c_void_p), C.c_char_p]),
    "magiplan_p2p_free": (C.c_int, [_vp]),
    "magiplan_p2p_open": (C.c_int, [C.c_char_p, C.POINTER(C.c_void_p)]),
    "magiplan_p2p_close": (C.c_int, [_vp]),
    "magiplan_range_copy_to": (C.c_int, [_vp, _vp, _vp, _vp, _vp, _i64, _i64, _i64, _vp]),
    "magiplan_range_scatter_add_from": (C.c_int, [_vp, _vp, _vp, _vp, _vp, _i64, _i64, _i64, _vp]),
    "magiplan_flags_signal": (C.c_int, [_vp, _i32, C.c_uint32, _vp]),
    "magiplan_flags_wait": (C.c_int, [_vp, C.c_uint32, C.c_uint32, _vp]),
    "magiplan_debug_umma_tile": (C.c_int, [_vp, _vp, _vp, _i32, _vp]),
    "magiplan_debug_eval": (C.c_int, [_cp, C.POINTER(_vp)]),
    "magiplan_debug_set_trace": (C.c_int, [_vp, _i32]),
}


class MagiplanError(RuntimeError):
    def __init__(self, status: int, message: str):
        super().__init__(f"magiplan status {status}: {message}")
        self.status = status
        self.message = message


class UsageError(MagiplanError):
    pass


class ConstraintError(MagiplanError):
    pass


class InternalError(MagiplanError):
    pass


_ERRORS = {ERR_USAGE: UsageError, ERR_CONSTRAINT: ConstraintError, ERR_INTERNAL: InternalError}
_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not _LIB_PATH.exists():
            raise ImportError(
                f"{_LIB_PATH} is missing: run __graft_entry__.build() (there is no fallback path)")
        handle = C.CDLL(str(_LIB_PATH))
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(handle, name, None)
            if fn is None:
                continue
            fn.restype = res
            fn.argtypes = args
        _lib = handle
    return _lib


def check(status: int) -> None:
    if status != OK:
        msg = lib().magiplan_last_error().decode()
        raise _ERRORS.get(status, MagiplanError)(status, msg)


def call(name: str, *args) -> None:
    check(getattr(lib(), name)(*args))


def take_string(ptr: C.c_void_p) -> str:
    """Copy a library-owned string and release it with magiplan_string_free."""
    try:
        return C.string_at(ptr).decode()
    finally:
        lib().magiplan_string_free(ptr)


def exported_symbols() -> list[str]:
    return [name for name in SIGNATURES if hasattr(lib(), name)]
