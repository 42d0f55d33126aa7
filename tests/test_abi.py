"""The C-ABI library loads on a GPU-less host and exports every symbol
include/vpx.h declares; error codes map onto the reference taxonomy."""

import ctypes

import pytest

from paper_2007_12856_b200 import _lib, errors


def test_library_loads_and_exports_all_declared_symbols():
    lib = _lib.load()
    names = _lib.declared_symbols()
    assert len(names) >= 30
    raw = ctypes.CDLL(str(_lib.LIB_PATH))
    for n in names:
        assert hasattr(raw, n), n
    assert b"sm_100a" in lib.vpx_version()
    # measurement probes live in tools/libvpx_probe.so, not in the product library
    assert not any(hasattr(raw, n) for n in ("vpx_probe_umma", "vpx_probe_tma", "vpx_probe_mma_rate2"))


def test_shape_errors_map_to_reference_exceptions():
    lib = _lib.load()
    bad = (ctypes.c_int * 8)(1, 4, 0, 8, 8, 0, 0, 0)  # zero extent
    ok = (ctypes.c_int * 8)(1, 16, 8, 8, 8, 0, 0, 0)
    with pytest.raises(errors.ShapeMismatch):
        _lib.call("vpx_conv3d_fwd", 0, ctypes.addressof(bad), 0, 3, 1, 0, ctypes.addressof(ok), 0, 0, 0)
    even_k = (ctypes.c_int * 8)(1, 4, 8, 8, 8, 0, 0, 0)
    with pytest.raises(errors.ShapeMismatch):
        _lib.call("vpx_conv3d_fwd", 0, ctypes.addressof(even_k), 0, 2, 1, 0, ctypes.addressof(ok), 0, 0, 0)
    odd = (ctypes.c_int * 8)(1, 4, 7, 8, 8, 0, 0, 0)
    out = (ctypes.c_int * 8)(1, 4, 3, 4, 4, 0, 0, 0)
    with pytest.raises(errors.NonDivisible):
        _lib.call("vpx_pool_fwd", 0, ctypes.addressof(odd), 0, ctypes.addressof(out), 0, 0)
    assert lib.vpx_last_error()


def test_product_path_has_no_oracle_or_cpu_fallback():
    """The package never imports the oracle, and ops raise when the library
    is missing instead of computing on the CPU."""
    import pathlib

    pkg = pathlib.Path(_lib.__file__).parent
    for py in pkg.glob("*.py"):
        text = py.read_text()
        assert "import oracle" not in text and "from oracle" not in text, py
