"""Device time of one deep-layer conv pass (CosmoFlow-512 c4..c7 shapes, one
GPU): 50 back-to-back passes captured in one CUDA graph, replayed; reports
microseconds per pass for forward, backward-data and backward-filter
(each = the C-ABI call: weight pack + kernel + split-K reduce).
python tools/small_pass.py
SMALL_PASS_EAGER=1 runs each pass 3 times eagerly instead (for an ncu launch list)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2007_12856_b200 import _lib  # noqa: E402
from paper_2007_12856_b200.frames import Frame, stream_ptr  # noqa: E402

SHAPES = {"c4": (64, 128, 64, 2), "c5": (128, 256, 16, 1), "c6": (256, 256, 8, 1), "c7": (256, 256, 4, 1)}
REPS = 50


def timed(fn):
    if os.environ.get("SMALL_PASS_EAGER"):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        return 0.0
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for _ in range(REPS):
                fn()
    torch.cuda.synchronize()
    g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(5):
        g.replay()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) * 1e3 / (5 * REPS)


lib = _lib.load()
for name, (cin, cout, e, s) in SHAPES.items():
    od = e // s
    x = Frame(1, cin, e, e, e, (0, 0, 0), zero=True)
    x.t.normal_()
    y = Frame(1, cout, od, od, od)
    u = Frame(1, cout, od, od, od)
    u.t.normal_()
    g = Frame(1, cin, e, e, e)
    w = torch.randn(cout, cin, 3, 3, 3, device="cuda") * 0.01
    wg = torch.empty_like(w)
    nb = max(lib.vpx_conv3d_workspace_bytes(cin, cout, 3, y.desc), lib.vpx_conv3d_workspace_bytes(cin, cout, 3, g.desc))
    ws = torch.empty(nb // 4 + 1024, device="cuda")
    f = lambda: _lib.call("vpx_conv3d_fwd", x.ptr, x.desc, w.data_ptr(), 3, s, y.ptr, y.desc, ws.data_ptr(),
                          ws.numel() * 4, stream_ptr())
    d = lambda: _lib.call("vpx_conv3d_bwd_data", u.ptr, u.desc, w.data_ptr(), 3, s, g.ptr, g.desc, ws.data_ptr(),
                          ws.numel() * 4, stream_ptr())
    wf = lambda: _lib.call("vpx_conv3d_bwd_filter", x.ptr, x.desc, u.ptr, u.desc, 3, s, wg.data_ptr(), 0,
                           ws.data_ptr(), ws.numel() * 4, stream_ptr())
    print(f"{name} ({cin}->{cout}, {e}^3, s{s}): fwd {timed(f):6.1f} us  dgrad {timed(d):6.1f} us  "
          f"wgrad {timed(wf):6.1f} us", flush=True)
