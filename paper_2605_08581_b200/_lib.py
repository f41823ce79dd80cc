"""ctypes binding of libprism.so (the C ABI in include/prism.h).

Loading fails loudly when the library is missing or no CUDA device is
present: the product path has no CPU fallback.
"""

from __future__ import annotations

import ctypes as C
import os

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(PKG, "libprism.so")

PRISM_OK, PRISM_CAPACITY, PRISM_RELEASE, PRISM_INVALID, PRISM_CUDA, PRISM_FATAL, PRISM_SIMULATION = range(7)
SEG_NONE = -(2**31)

_i64, _i32, _p = C.c_int64, C.c_int32, C.c_void_p

_SIGS = {
    "prism_last_error": (C.c_char_p, []),
    "prism_device_count": (C.c_int, []),
    "prism_tree_create": (_p, [_i64, _i32, _i64, _i64, _i64, _i32]),
    "prism_tree_destroy": (None, [_p]),
    "prism_match": (C.c_int, [_p, _p, _i64, _p, _p, _p, _p]),
    "prism_insert": (C.c_int, [_p, _p, _i64, _i64, _p, _p, _p, _p, _p, _p]),
    "prism_release": (C.c_int, [_p, _i64, _p, _p]),
    "prism_release_device": (C.c_int, [_p, _i64, _p, _p, _p]),
    "prism_pin_device": (C.c_int, [_p, _i64, _p, _p]),
    "prism_tree_stream": (_p, [_p]),
    "prism_evict": (C.c_int, [_p, _i64, _p]),
    "prism_set_protection": (C.c_int, [_p, _i64, _p, _p, _p, _p]),
    "prism_note_active": (C.c_int, [_p, _i64, _p]),
    "prism_admit_wave": (C.c_int, [_p, _i64] + [_p] * 11),
    "prism_admit_wave_device": (C.c_int, [_p, _i64] + [_p] * 12),
    "prism_stats": (C.c_int, [_p, _p]),
    "prism_victims": (C.c_int, [_p, _i64, _i64, _p, _p, _p, _p, _p, _p]),
    "prism_snapshot": (C.c_int, [_p, _i64] + [_p] * 17),
    "prism_arena_read": (C.c_int, [_p, _i64, _i64, _p]),
    "prism_evict_key": (C.c_int, [_p, _i32, _p]),
    "prism_last_op": (C.c_int, [_p, _p]),
    "prism_compactions": (_i64, [_p]),
    "prism_tune": (C.c_int, [_p, _i32, _i64]),
    "prism_qas_create": (_p, [_i32]),
    "prism_qas_destroy": (None, [_p]),
    "prism_qas_round": (C.c_int, [_p, _i64, _p, _p, _p, _p, _p, _i64, _p, _p, _i32, _p] + [_p] * 16),
    "prism_serve_create": (_p, [_p, _p, _i64, _p, _p, _p, _p, _p, _p, _i32, _i64, _i64, _i64, _p, C.c_double,
                                C.c_double, C.c_double, _i64, _i32]),
    "prism_serve_destroy": (None, [_p]),
    "prism_serve_run": (C.c_int, [_p, _i64, _p, _p]),
    "prism_serve_counts": (C.c_int, [_p, _p]),
    "prism_serve_requests": (C.c_int, [_p] + [_p] * 6),
    "prism_serve_waves": (C.c_int, [_p] + [_p] * 6),
    "prism_trace_load_jsonl": (_p, [C.c_char_p, _i32]),
    "prism_trace_info": (C.c_int, [_p, _p]),
    "prism_trace_copy": (C.c_int, [_p] + [_p] * 7),
    "prism_trace_free": (None, [_p]),
}

_LIB: C.CDLL | None = None


class PrismError(RuntimeError):
    pass


def lib() -> C.CDLL:
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise PrismError(
                f"{LIB_PATH} is missing: build it with `python -m paper_2605_08581_b200.build` "
                "(there is no CPU fallback)"
            )
        dll = C.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            fn = getattr(dll, name, None)
            if fn is None:
                continue
            fn.restype = res
            fn.argtypes = args
        _LIB = dll
    return _LIB


def exported_symbols() -> list[str]:
    return [n for n in _SIGS if hasattr(lib(), n)]


def last_error() -> str:
    msg = lib().prism_last_error()
    return msg.decode() if msg else ""


def check(rc: int) -> None:
    if rc == PRISM_OK:
        return
    if rc == PRISM_INVALID:
        raise ValueError(last_error())
    if rc == PRISM_SIMULATION:
        from .types import SimulationError

        raise SimulationError(last_error())
    raise PrismError(f"prism status {rc}: {last_error()}")


def require_device() -> None:
    if lib().prism_device_count() <= 0:
        raise PrismError("no CUDA device visible: the PRISM B200 path has no CPU fallback")
