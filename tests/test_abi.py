"""The C-ABI library: it loads, exports exactly what include/holmes_b200.h
declares, and fails loudly (no CPU fallback) when there is no device.
CPU only — no compute calls are made here."""
import ctypes as C
import os
import re

import numpy as np
import pytest
import torch

from paper_2008_04063_b200 import _lib, errors

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    names = set()
    for fn in os.listdir(os.path.join(ROOT, "include")):
        if fn.endswith(".h"):
            text = open(os.path.join(ROOT, "include", fn)).read()
            text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
            names |= set(re.findall(r"\b(hb_[a-z0-9_]+)\s*\(", text))
    return names


def test_library_exports_every_declared_symbol():
    lib = _lib.lib()
    decl = declared_symbols()
    assert len(decl) >= 25
    for name in sorted(decl):
        assert hasattr(lib, name), name
    # the ctypes binding covers the whole header
    assert decl == set(_lib.exported_symbols())
    assert lib.hb_version() >= 1


def test_library_is_built_for_sm100a():
    out = os.popen(f"cuobjdump --list-elf {_lib.LIB_PATH} 2>&1").read()
    assert "sm_100a" in out


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-device error path")
def test_no_device_fails_loudly():
    from paper_2008_04063_b200.engine import EnsembleEngine
    from paper_2008_04063_b200.zoo import Selector, holmes_zoo
    with pytest.raises(errors.DeviceError, match="no CUDA device"):
        EnsembleEngine(holmes_zoo(), Selector.from_indices(60, [10]), 2)
    h = C.c_void_p()
    sc = np.zeros((4, 2))
    lab = np.array([0, 1, 0, 1], np.int8)
    rc = _lib.lib().hb_cohort_create(0, _lib.dptr(sc), lab.ctypes.data_as(C.POINTER(C.c_int8)), 4, 2, C.byref(h))
    with pytest.raises(errors.DeviceError):
        _lib.check(rc, None, "hb_cohort_last_error")


def test_cohort_argument_errors_map_to_reference_exceptions():
    """Validation happens before any device work, so it is testable on CPU."""
    L = _lib.lib()
    h = C.c_void_p()
    sc = np.zeros((4, 2))
    one_class = np.ones(4, np.int8)
    rc = L.hb_cohort_create(0, _lib.dptr(sc), one_class.ctypes.data_as(C.POINTER(C.c_int8)), 4, 2, C.byref(h))
    with pytest.raises(errors.UndefinedMetricError):
        _lib.check(rc, None, "hb_cohort_last_error")
    bad = np.array([0, 2, 0, 1], np.int8)
    rc = L.hb_cohort_create(0, _lib.dptr(sc), bad.ctypes.data_as(C.POINTER(C.c_int8)), 4, 2, C.byref(h))
    with pytest.raises(ValueError, match="labels must be 0 or 1"):
        _lib.check(rc, None, "hb_cohort_last_error")
    nan = sc.copy()
    nan[1, 1] = np.nan
    ok = np.array([0, 1, 0, 1], np.int8)
    rc = L.hb_cohort_create(0, _lib.dptr(nan), ok.ctypes.data_as(C.POINTER(C.c_int8)), 4, 2, C.byref(h))
    with pytest.raises(ValueError, match="finite"):
        _lib.check(rc, None, "hb_cohort_last_error")


def test_config_errors_map_to_configuration_error():
    L = _lib.lib()
    cfg = _lib.HbConfig(4, 3, 250, 7500, 0, 0, 0)   # hop 0
    h = C.c_void_p()
    with pytest.raises(errors.ConfigurationError, match="hop"):
        _lib.check(L.hb_create(0, C.byref(cfg), C.byref(h)))


def test_one_shot_sweep_rejects_wide_cohorts_before_device_work():
    from paper_2008_04063_b200 import metrics
    with pytest.raises(ValueError, match="n must be <= 32"):
        metrics.sweep_auc(np.array([0, 1, 0, 1]), np.zeros((4, 33)), [1])
