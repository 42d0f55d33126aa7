"""Build the oracle's native pieces (TEST INFRASTRUCTURE ONLY).

1. oracle/conv_oracle.so  <- oracle/conv_oracle.c   (gcc -O3 -ffp-contract=off -fopenmp)
2. oracle/_ref/_hot*.so   <- the reference's own Cython kernel source
   /root/reference/pkg/src/voxpar/kernels/_hot.pyx, compiled straight from where
   it lies (cython -> gcc, the flags of reference pkg/setup.py:45-52).  Only when
   /root/reference exists (this container); the built .so travels to GPU boxes.
   No reference source is copied into the repository: the generated C and the
   module land in oracle/_ref/, which is git-ignored.

python oracle/build_oracle.py [--force]
"""

from __future__ import annotations

import subprocess
import sys
import sysconfig
from pathlib import Path

HERE = Path(__file__).resolve().parent
REF_PYX = Path("/root/reference/pkg/src/voxpar/kernels/_hot.pyx")
REF_DIR = HERE / "_ref"
ORACLE_SO = HERE / "conv_oracle.so"


def _newer(dst: Path, *srcs: Path) -> bool:
    return dst.exists() and all(dst.stat().st_mtime >= s.stat().st_mtime for s in srcs)


def build_conv_oracle(force=False) -> Path:
    src = HERE / "conv_oracle.c"
    if force or not _newer(ORACLE_SO, src):
        subprocess.run(["gcc", "-O3", "-ffp-contract=off", "-fopenmp", "-fPIC", "-shared",
                        str(src), "-o", str(ORACLE_SO)], check=True)
    return ORACLE_SO


def ref_module_path():
    suffix = sysconfig.get_config_var("EXT_SUFFIX") or ".so"
    return REF_DIR / f"_hot{suffix}"


def build_reference_kernels(force=False):
    """Compile the reference's _hot.pyx into oracle/_ref/ (None if unavailable)."""
    out = ref_module_path()
    if not REF_PYX.exists():
        return out if out.exists() else None
    if not force and _newer(out, REF_PYX):
        return out
    REF_DIR.mkdir(exist_ok=True)
    csrc = REF_DIR / "_hot.c"
    subprocess.run([sys.executable, "-m", "cython", "-3", str(REF_PYX), "-o", str(csrc)], check=True)
    import numpy as np

    inc = sysconfig.get_paths()["include"]
    subprocess.run(["gcc", "-O3", "-ffp-contract=off", "-fPIC", "-shared",
                    "-DNPY_NO_DEPRECATED_API=NPY_1_7_API_VERSION",
                    f"-I{inc}", f"-I{np.get_include()}", str(csrc), "-o", str(out)], check=True)
    csrc.unlink()  # generated translation unit; only the compiled module is kept
    return out


def build(force=False):
    build_conv_oracle(force)
    return build_reference_kernels(force)


if __name__ == "__main__":
    print(build(force="--force" in sys.argv))
