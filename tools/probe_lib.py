"""Build and load tools/libvpx_probe.so: the tcgen05/TMA measurement probes
(tools/csrc/probe.cu, prototypes in tools/csrc/vpx_probe.h).  Scaffolding for
tools/probe_*.py only -- kept out of the product library libvpx.so, which it
links against for the shared host helpers."""

from __future__ import annotations

import ctypes
import subprocess
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
ROOT = HERE.parent
sys.path.insert(0, str(ROOT))
from paper_2007_12856_b200 import _lib, build as vbuild  # noqa: E402

SRC = HERE / "csrc" / "probe.cu"
HDR = HERE / "csrc" / "vpx_probe.h"
LIB = HERE / "libvpx_probe.so"
_probe = None


def build(force: bool = False) -> Path:
    vlib = vbuild.build()
    if not force and LIB.exists() and LIB.stat().st_mtime > max(SRC.stat().st_mtime, vlib.stat().st_mtime):
        return LIB
    csrc = ROOT / "paper_2007_12856_b200" / "csrc"
    cmd = [vbuild.NVCC, *vbuild.ARCH, *vbuild.FLAGS, "-shared", "-I", str(csrc), "-I", str(ROOT / "include"),
           "-I", str(HERE / "csrc"), str(SRC), "-o", str(LIB), "-L", str(vlib.parent), "-lvpx",
           "-Xlinker", f"-rpath={vlib.parent}"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"probe build failed:\n{r.stdout}\n{r.stderr}")
    return LIB


def load():
    global _probe
    if _probe is None:
        _lib.load()
        lib = ctypes.CDLL(str(build()))
        for name, (rt, args) in _lib._parse_header(HDR).items():
            fn = getattr(lib, name)
            fn.argtypes, fn.restype = args, rt
        _probe = lib
    return _probe


def call(name, *args):
    rc = getattr(load(), name)(*args)
    if rc != 0:
        raise RuntimeError(f"{name}: {_lib.load().vpx_last_error().decode(errors='replace')}")
    return rc
