"""Pinned counter-based PRNG (splitmix64), host key folding + device streams.

Algorithm pinned by the reference (reference pkg/src/voxpar/prng.py:1-25):
  mix(z)         = z ^= z>>30; z *= 0xBF58476D1CE4E5B9; z ^= z>>27;
                   z *= 0x94D049BB133111EB; z ^= z>>31          (mod 2^64)
  key_fold(k..)  = acc = 0x243F6A8885A308D3; acc = mix(acc ^ mix(k_i + golden))
  stream(key)[i] = mix(key + (i+1)*golden)
  uniform01      = (u64 >> 11) * 2^-53 (fp64)
Key folding is a handful of integer ops and stays on the host; streams are
generated on the device by vpx_prng_* and are bit-identical to numpy's
(tests/test_prng_gpu.py).  Keys in use: init weights [seed,-1,i]
(reference model/optim.py:97-113), synthetic batch [seed,-3,0|1]
(reference cli.py:112-125), dropout [seed,epoch,iteration,sample,layer]
(reference model/engine.py:314-320).
"""

from __future__ import annotations

MASK = (1 << 64) - 1
GOLDEN = 0x9E3779B97F4A7C15
M1 = 0xBF58476D1CE4E5B9
M2 = 0x94D049BB133111EB
FOLD_INIT = 0x243F6A8885A308D3


def mix(z: int) -> int:
    z &= MASK
    z = ((z ^ (z >> 30)) * M1) & MASK
    z = ((z ^ (z >> 27)) * M2) & MASK
    return z ^ (z >> 31)


def key_fold(parts) -> int:
    acc = FOLD_INIT
    for p in parts:
        acc = mix(acc ^ mix((int(p) & MASK) + GOLDEN))
    return acc


def resolve(key) -> int:
    return key if isinstance(key, int) else key_fold(key)


def u64_host(key, n: int):
    """Small host-side stream (used for schedule-sized draws and tests)."""
    k = resolve(key)
    return [mix(k + ((i + 1) * GOLDEN & MASK)) for i in range(n)]


def uniform_device(key, n: int, lo: float, hi: float, out=None, fp64: bool = False):
    """lo + (hi-lo) * uniform01 of the first n values of the stream, on the
    current CUDA stream; returns a float32 (or float64) CUDA tensor."""
    import torch

    from . import _lib

    if out is None:
        out = torch.empty(n, dtype=torch.float64 if fp64 else torch.float32, device="cuda")
    p32 = 0 if fp64 else out.data_ptr()
    p64 = out.data_ptr() if fp64 else 0
    _lib.call("vpx_prng_uniform", resolve(key), n, float(lo), float(hi), p32, p64,
              torch.cuda.current_stream().cuda_stream)
    return out


def keep_mask_device(key, n: int, keep: float):
    """uniform01 < keep as a uint8 CUDA tensor (dropout masks)."""
    import torch

    from . import _lib

    out = torch.empty(n, dtype=torch.uint8, device="cuda")
    _lib.call("vpx_prng_mask", resolve(key), n, float(keep), out.data_ptr(),
              torch.cuda.current_stream().cuda_stream)
    return out


# ----------------------------------------------------------- host (numpy)
# Vectorised host streams for schedule- and fixture-sized draws (epoch
# permutations, HSB1 fixture voxels); identical bits to the device streams.

def u64(key, n: int):
    """First n raw 64-bit words of the stream (reference prng.py:54-62)."""
    import numpy as np

    k = np.uint64(resolve(key))
    z = k + (np.arange(n, dtype=np.uint64) + np.uint64(1)) * np.uint64(GOLDEN)
    z = (z ^ (z >> np.uint64(30))) * np.uint64(M1)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(M2)
    return z ^ (z >> np.uint64(31))


def randint(key, n: int, lo: int, hi: int):
    """Integers in [lo, hi), modulo-mapped (reference prng.py:75-78)."""
    import numpy as np

    return (u64(key, n) % np.uint64(hi - lo)).astype(np.int64) + lo


def permutation(key, size: int):
    """Fisher-Yates shuffle of arange(size), j = stream[i] mod (i+1)
    (reference prng.py:81-90)."""
    import numpy as np

    perm = np.arange(size, dtype=np.int64)
    if size < 2:
        return perm
    draws = u64(key, size)
    for i in range(size - 1, 0, -1):
        j = int(draws[i] % np.uint64(i + 1))
        perm[i], perm[j] = perm[j], perm[i]
    return perm
