"""Per-kernel device timing for the roofline report (bench.py).

When a Recorder is active, the layer ops bracket their libvpx launches with
CUDA events on the launching (current) stream and tag them with the layer
name, pass and the algorithmic flops / bytes of that launch.  Inactive
(the default), `region` is a no-op context manager.  With VPX_NVTX=1 in the
environment every region is also an NVTX range named by its tag, so a single
layer's kernel can be selected for `ncu --nvtx --nvtx-include "<tag>/"`.

Recorder(graph=True) records its events with cudaEventRecordExternal, so a
step captured while it is active (engine.CapturedStep(recorder=...)) carries
the events as graph nodes and every replay re-times each region: the
per-layer breakdown of the graph-replayed step itself, without the host
launch gaps that inflate the small layers in an eager step.
"""

from __future__ import annotations

import contextlib
import os
from collections import defaultdict

import torch

_ACTIVE = None
_NVTX = os.environ.get("VPX_NVTX") == "1"
_RT = None


def _cudart():
    global _RT
    if _RT is None:
        import ctypes

        _RT = ctypes.CDLL("libcudart.so.12")
    return _RT


class _ExtEvent:
    """A timing CUDA event recorded with cudaEventRecordExternal (a graph
    node under stream capture, a plain record otherwise)."""

    __slots__ = ("h",)

    def __init__(self):
        import ctypes

        self.h = ctypes.c_void_p()
        rc = _cudart().cudaEventCreate(ctypes.byref(self.h))
        if rc:
            raise RuntimeError(f"cudaEventCreate: {rc}")

    def record(self):
        import ctypes

        rc = _cudart().cudaEventRecordWithFlags(self.h, ctypes.c_void_p(torch.cuda.current_stream().cuda_stream), 1)
        if rc:
            raise RuntimeError(f"cudaEventRecordWithFlags: {rc}")

    def elapsed_time(self, end: "_ExtEvent") -> float:
        import ctypes

        ms = ctypes.c_float()
        rc = _cudart().cudaEventElapsedTime(ctypes.byref(ms), self.h, end.h)
        if rc:
            raise RuntimeError(f"cudaEventElapsedTime: {rc}")
        return float(ms.value)

    def __del__(self):
        try:
            _cudart().cudaEventDestroy(self.h)
        except Exception:
            pass


class Recorder:
    def __init__(self, graph: bool = False):
        self.events = []  # (tag, flops, bytes, start, end)
        self.graph = graph
        self._acc = None

    def __enter__(self):
        global _ACTIVE
        _ACTIVE = self
        return self

    def __exit__(self, *exc):
        global _ACTIVE
        _ACTIVE = None

    def _add(self, out):
        for tag, fl, by, s, e in self.events:
            d = out[tag]
            d["ms"] += s.elapsed_time(e)
            d["launches"] += 1
            d["flops"], d["bytes"] = fl, by
            d["bytes_total"] += by

    def accumulate(self):
        """Graph mode: add the regions' times of the replay that just ran (the
        captured event nodes are re-recorded by every replay)."""
        torch.cuda.synchronize()
        if self._acc is None:
            self._acc = defaultdict(lambda: {"ms": 0.0, "launches": 0, "flops": 0, "bytes": 0, "bytes_total": 0})
        self._add(self._acc)

    def summary(self):
        """{tag: {"ms": total, "launches": k, "flops": per launch, "bytes": per launch}}"""
        if self._acc is not None:
            return dict(self._acc)
        torch.cuda.synchronize()
        out = defaultdict(lambda: {"ms": 0.0, "launches": 0, "flops": 0, "bytes": 0, "bytes_total": 0})
        self._add(out)
        return dict(out)


@contextlib.contextmanager
def region(tag: str, flops: int = 0, nbytes: int = 0):
    rec = _ACTIVE
    if _NVTX:
        torch.cuda.nvtx.range_push(tag)
    if rec is None:
        try:
            yield
        finally:
            if _NVTX:
                torch.cuda.nvtx.range_pop()
        return
    if rec.graph:
        s, e = _ExtEvent(), _ExtEvent()
    else:
        s = torch.cuda.Event(enable_timing=True)
        e = torch.cuda.Event(enable_timing=True)
    s.record()
    try:
        yield
    finally:
        if _NVTX:
            torch.cuda.nvtx.range_pop()
    e.record()
    rec.events.append((tag, flops, nbytes, s, e))
