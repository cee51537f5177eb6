"""ctypes binding of the in-tree C-ABI library `libholmes_b200.so`.

The library is the product: there is no CPU fallback.  Importing the package
never needs the library (pure data-model code works on any host), but every
compute entry point calls `lib()`, which raises if the library is missing or
cannot load — loudly, never silently degrading.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

from . import errors

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("HB_LIB_PATH") or os.path.join(_HERE, "libholmes_b200.so")  # override: A/B experiments

HB_OK, HB_E_INVALID, HB_E_CONFIG, HB_E_EMPTY, HB_E_CUDA, HB_E_STATE, HB_E_METRIC = range(7)

_EXC = {
    HB_E_INVALID: ValueError,
    HB_E_CONFIG: errors.ConfigurationError,
    HB_E_EMPTY: errors.EmptyEnsembleError,
    HB_E_CUDA: errors.DeviceError,
    HB_E_STATE: RuntimeError,
    HB_E_METRIC: errors.UndefinedMetricError,
}


class HbConfig(C.Structure):
    _fields_ = [("max_patients", C.c_int), ("n_leads", C.c_int), ("fs", C.c_int), ("window_len", C.c_int),
                ("hop", C.c_int), ("ring_len", C.c_int), ("keep_windows", C.c_int)]


_P = C.c_void_p
_F = C.POINTER(C.c_float)
_SIGS = {
    "hb_version": (C.c_int, []),
    "hb_last_error": (C.c_char_p, [_P]),
    "hb_create": (C.c_int, [C.c_int, C.POINTER(HbConfig), C.POINTER(_P)]),
    "hb_destroy": (C.c_int, [_P]),
    "hb_add_member": (C.c_int, [_P, C.c_int, C.c_int, C.c_int, C.c_int, _F, C.c_size_t]),
    "hb_set_selector": (C.c_int, [_P, C.POINTER(C.c_uint8), C.c_int]),
    "hb_selected": (C.c_int, [_P, C.POINTER(C.c_int), C.c_int]),
    "hb_ingest": (C.c_int, [_P, _F, C.c_int, _P]),
    "hb_tick": (C.c_int, [_P, _P, _P, _P, _P, _P]),
    "hb_tick_submit": (C.c_int, [_P, _P, C.c_int, _P]),
    "hb_tick_collect": (C.c_int, [_P, C.c_int, _P, _P, _P]),
    "hb_stage_device": (C.c_int, [_P, _P, _P]),
    "hb_tick_device": (C.c_int, [_P, _P]),
    "hb_device_outputs": (C.c_int, [_P, C.POINTER(_P), C.POINTER(_P), C.POINTER(_P)]),
    "hb_last_tick_ms": (C.c_int, [_P, _F]),
    "hb_time_tick": (C.c_int, [_P, C.c_int, _F]),
    "hb_prepare": (C.c_int, [_P]),
    "hb_chain_profile": (C.c_int, [_P, C.c_void_p, C.c_int]),
    "hb_chain_trace": (C.c_int, [_P, C.c_void_p, C.c_void_p, C.c_int]),
    "hb_device_sums": (C.c_int, [_P, C.POINTER(_P)]),
    "hb_finalize_sums": (C.c_int, [_P, C.c_int, C.c_int, _P, _P, _P]),
    "hb_last_windows": (C.c_int, [_P, _F, _F, _P]),
    "hb_profile_tick": (C.c_int, [_P, _P, C.c_int, C.POINTER(C.c_int), _F, C.POINTER(C.c_double),
                                  C.POINTER(C.c_double)]),
    "hb_tick_work": (C.c_int, [_P, C.POINTER(C.c_double), C.POINTER(C.c_double)]),
    "hb_last_normalized": (C.c_int, [_P, _P, _P]),
    "hb_member_layers": (C.c_int, [C.c_int, C.c_int, C.c_int, C.POINTER(C.c_int), C.c_int]),
    "hb_sweep_auc": (C.c_int, [C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_int8), C.c_int, C.c_int,
                               C.POINTER(C.c_uint32), C.c_int, C.POINTER(C.c_double)]),
    "hb_cohort_create": (C.c_int, [C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_int8), C.c_int, C.c_int,
                                   C.POINTER(_P)]),
    "hb_cohort_destroy": (C.c_int, [_P]),
    "hb_cohort_last_error": (C.c_char_p, [_P]),
    "hb_cohort_auc": (C.c_int, [_P, C.POINTER(C.c_uint8), C.c_int, C.POINTER(C.c_double)]),
    "hb_cohort_auc_range": (C.c_int, [_P, C.c_ulonglong, C.c_longlong, C.POINTER(C.c_double)]),
    "hb_cohort_ensemble": (C.c_int, [_P, C.POINTER(C.c_uint8), C.POINTER(C.c_double), C.POINTER(C.c_double)]),
    "hb_arrival_widths": (C.c_int, [C.POINTER(C.c_double), C.c_int, C.POINTER(C.c_double)]),
    "hb_binned_best": (C.c_int, [C.POINTER(C.c_double), C.c_int, C.POINTER(C.c_double)]),
    "hb_curve_last_error": (C.c_char_p, []),
    "hb_op_conv1d": (C.c_int, [_P, C.c_int, C.c_int, C.c_int, C.c_int, _F, _F, C.c_int, _P, C.c_int, C.c_int,
                               C.c_int, _P, C.c_int, _F, _P, _P]),
    "hb_conv_mt": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int]),
    "hb_bench_conv": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, _F]),
    "hb_op_stem": (C.c_int, [_P, C.c_int, C.c_int, _F, _F, C.c_int, _P, _P]),
    "hb_op_conv1d_q": (C.c_int, [_P, C.c_int, C.c_int, C.c_int, C.c_int, _F, _F, C.c_int, _P, C.c_int, C.c_int,
                                 C.c_int, C.c_int, _P, C.c_int, _F, _P, C.c_int, _P]),
    "hb_conv_kind": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int]),
    "hb_conv_head_mt": (C.c_int, [C.c_int] * 7),
    "hb_bench_conv_k": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, _F]),
    "hb_op_stem_q": (C.c_int, [_P, C.c_int, C.c_int, _F, _F, C.c_int, _P, C.c_int, _P]),
    "hb_bench_stem": (C.c_int, [C.c_int] * 6 + [_F]),
}

_lock = threading.Lock()
_lib = None


def lib() -> C.CDLL:
    """Load (once) and return the C-ABI library; raises if it is absent."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise errors.DeviceError(
                    f"{LIB_PATH} is not built; run `python -c 'import __graft_entry__ as g; g.build()'` "
                    "(there is no CPU fallback)")
            handle = C.CDLL(LIB_PATH)
            for name, (res, args) in _SIGS.items():
                if os.environ.get("HB_LIB_PATH") and not hasattr(handle, name):
                    continue  # an older library under A/B test
                fn = getattr(handle, name)
                fn.restype = res
                fn.argtypes = args
            _lib = handle
    return _lib


def exported_symbols() -> list[str]:
    return sorted(_SIGS)


def check(rc: int, ctx=None, getter: str = "hb_last_error") -> None:
    """Raise the reference's exception class for a non-zero status (errors.py)."""
    if rc == HB_OK:
        return
    fn = getattr(lib(), getter)
    msg = fn() if getter == "hb_curve_last_error" else fn(ctx)
    text = msg.decode() if msg else f"status {rc}"
    raise _EXC.get(rc, RuntimeError)(text)


def dptr(a):
    """float64 numpy array -> POINTER(c_double)."""
    return None if a is None else a.ctypes.data_as(C.POINTER(C.c_double))


def fptr(a):
    """float32 numpy array -> POINTER(c_float) (None passes through)."""
    if a is None:
        return None
    return a.ctypes.data_as(_F)
