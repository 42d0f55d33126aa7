"""B200-native hybrid data x spatial parallel 3D-CNN training path (voxpar API).

Modules mirror the reference package's layout of the hot path:
geometry (reference tensor.py), comm (fabric.py), layers
(layers/distributed.py), networks / accounting (model/networks.py,
layers/accounting.py), engine (model/engine.py, optim.py), prng (prng.py),
kernels (kernels/__init__.py).  Arithmetic runs in libvpx.so (sm_100a).
"""

from . import errors  # noqa: F401

PRECISIONS = {"tf32": 0, "fp32": 1}


def set_precision(mode: str) -> None:
    """'tf32' (default): tcgen05 tensor cores, activations stored rounded to
    nearest TF32.  'fp32': CUDA-core fp32 direct kernels everywhere (strict
    parity mode, the reference's fp32 tolerance)."""
    from . import _lib

    _lib.call("vpx_set_precision", PRECISIONS[mode])


def get_precision() -> str:
    from . import _lib

    v = _lib.load().vpx_get_precision()
    return {0: "tf32", 1: "fp32"}[v]
