"""Per-kernel device timing for the roofline report (bench.py).

When a Recorder is active, the layer ops bracket their libvpx launches with
CUDA events on the launching (current) stream and tag them with the layer
name, pass and the algorithmic flops / bytes of that launch.  Inactive
(the default), `region` is a no-op context manager.  With VPX_NVTX=1 in the
environment every region is also an NVTX range named by its tag, so a single
layer's kernel can be selected for `ncu --nvtx --nvtx-include "<tag>/"`.
"""

from __future__ import annotations

import contextlib
import os
from collections import defaultdict

import torch

_ACTIVE = None
_NVTX = os.environ.get("VPX_NVTX") == "1"


class Recorder:
    def __init__(self):
        self.events = []  # (tag, flops, bytes, start, end)

    def __enter__(self):
        global _ACTIVE
        _ACTIVE = self
        return self

    def __exit__(self, *exc):
        global _ACTIVE
        _ACTIVE = None

    def summary(self):
        """{tag: {"ms": total, "launches": k, "flops": per launch, "bytes": per launch}}"""
        torch.cuda.synchronize()
        out = defaultdict(lambda: {"ms": 0.0, "launches": 0, "flops": 0, "bytes": 0, "bytes_total": 0})
        for tag, fl, by, s, e in self.events:
            d = out[tag]
            d["ms"] += s.elapsed_time(e)
            d["launches"] += 1
            d["flops"], d["bytes"] = fl, by
            d["bytes_total"] += by
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
