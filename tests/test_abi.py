"""The C-ABI library loads without a GPU and exports every symbol that
include/prismesh_cuda.h declares; argument errors come back as codes."""
import ctypes
import os
import re

import numpy as np
import pytest

from paper_1604_05937_b200 import _lib, builtin_layout, P2_LAYOUT

HEADER = os.path.join(os.path.dirname(os.path.dirname(
    os.path.abspath(__file__))), "include", "prismesh_cuda.h")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(pm_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = _lib.host_lib()
    names = declared_functions()
    assert len(names) >= 10
    for name in names:
        assert hasattr(lib, name), name
        assert name in _lib.SIGNATURES, f"{name} has no ctypes signature"


def test_num_slots_and_errors():
    assert _lib.num_slots(builtin_layout("CG1", "CG1")) == 6
    assert _lib.num_slots(P2_LAYOUT) == 18
    lib = _lib.host_lib()
    d = np.array([1, 0, 0, 0, 0, 0], dtype=np.int32)
    i32p = ctypes.POINTER(ctypes.c_int32)
    rc = lib.pm_build_cell_map(None, None, 1, 3, 3, d.ctypes.data_as(i32p),
                               0, 6, None, None, None, None)
    assert rc == _lib.PM_EINVAL and "layer" in _lib.last_error()
    bad = np.array([-1, 0, 0, 0, 0, 0], dtype=np.int32)
    k = ctypes.c_int32(0)
    assert lib.pm_num_slots(bad.ctypes.data_as(i32p), ctypes.byref(k)) == \
        _lib.PM_EINVAL
    with pytest.raises(ValueError):
        _lib.check(_lib.PM_EINVAL)
    # slot count that does not match the layout
    rc = lib.pm_column_mass(d.ctypes.data_as(i32p), 7, 10, 3, None, None,
                            None, None, None, None, None, None, None, None,
                            0, 0, 0, None, 0, None)
    assert rc == _lib.PM_EINVAL and "slot count" in _lib.last_error()
    # coloured variant without a cell list
    mref = np.eye(6)
    rc = lib.pm_column_mass(d.ctypes.data_as(i32p), 6, 10, 3, None, None,
                            None, None, None,
                            mref.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                            None, None, None, None, 0, 1,
                            _lib.VARIANT_COLORED, None, 0, None)
    assert rc == _lib.PM_EINVAL


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("has a GPU")
    with pytest.raises(RuntimeError):
        _lib.cuda_device()


def test_experimental_schedules_gated():
    """The default build leaves the slower experimental kernels out (tile,
    store-first patch strips) and says so through pm_build_flags."""
    import os
    from paper_1604_05937_b200 import _lib
    want = os.environ.get("PM_EXPERIMENTAL", "0") != "0"
    assert _lib.experimental() == want
