"""ctypes binding of libvpx.so (the C ABI declared in include/vpx.h).

The library is loaded lazily on first use.  There is no fallback: if the
shared object is missing or fails to load, every hot-path call raises
RuntimeError naming the problem (no multi-backend dispatch).
Non-zero statuses are mapped onto the reference's exception taxonomy
(reference pkg/src/voxpar/errors.py:4-77).
"""

from __future__ import annotations

import ctypes
import os
import re
from pathlib import Path

from . import errors

_HERE = Path(__file__).resolve().parent
LIB_PATH = Path(os.environ.get("VPX_LIB", _HERE / "libvpx.so"))
HEADER = _HERE.parent / "include" / "vpx.h"

_lib = None

_STATUS = {
    -1: errors.ShapeMismatch,
    -2: errors.NonDivisible,
    -3: errors.OutOfBounds,
    -4: errors.LengthMismatch,
    -5: errors.Unsupported,
    -6: errors.DeviceError,
}

c_int, c_void_p, c_float, c_double = ctypes.c_int, ctypes.c_void_p, ctypes.c_float, ctypes.c_double
c_i64, c_u64, c_i32, c_u32 = ctypes.c_int64, ctypes.c_uint64, ctypes.c_int32, ctypes.c_uint32
P = ctypes.POINTER

_CTYPES = {
    "int": c_int, "float": c_float, "double": c_double, "long long": c_i64,
    "unsigned long long": c_u64,
}


def _parse_header(header: Path = HEADER):
    """{name: (restype, [argtypes])} from the prototypes in include/vpx.h.

    Pointers of any type become c_void_p (callers pass torch data_ptr() or
    ctypes addresses); scalars map through _CTYPES.
    """
    text = re.sub(r"/\*.*?\*/", "", Path(header).read_text(), flags=re.S)
    protos = {}
    for m in re.finditer(r"^\s*((?:const\s+)?[\w ]+?\s*\**)\s*(vpx_\w+)\s*\(([^)]*)\)\s*;", text, re.M):
        ret, name, args = m.group(1).strip(), m.group(2), m.group(3)
        types = []
        for a in [a.strip() for a in args.split(",") if a.strip() and a.strip() != "void"]:
            if "*" in a:
                types.append(c_void_p)
            else:
                base = re.sub(r"\s+\w+$", "", a).replace("const", "").strip()
                types.append(_CTYPES[base])
        if "*" in ret:
            rt = ctypes.c_char_p
        else:
            rt = _CTYPES[ret.replace("const", "").strip()]
        protos[name] = (rt, types)
    return protos


def declared_symbols():
    """Every function name declared in include/vpx.h (for the ABI export test)."""
    return sorted(_parse_header())


def load():
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise RuntimeError(f"libvpx.so not built at {LIB_PATH}; run `python -m paper_2007_12856_b200.build`")
    lib = ctypes.CDLL(str(LIB_PATH))
    for name, (rt, args) in _parse_header().items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = rt
    _lib = lib
    return lib


def call(name, *args):
    """Invoke an entry point and raise the mapped exception on a bad status."""
    lib = load()
    rc = getattr(lib, name)(*args)
    if rc != 0:
        msg = lib.vpx_last_error().decode(errors="replace")
        raise _STATUS.get(rc, errors.DeviceError)(f"{name}: {msg}")
    return rc
