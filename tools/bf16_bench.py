"""BF16 vs TF32 tap-box conv throughput on CosmoFlow-512 layer shapes (GPU):
forward and backward-data of c3 (32->64, 128^3), c4 (64->128 stride 2, 64^3),
c5 (128->256, 16^3) through vpx_conv3d_fwd(_bf16) / vpx_conv3d_bwd_data(_bf16),
CUDA-event timed (median of 20).  The TF32 numbers force the tap-box kernel
(VPX_NO_ROWWIN-style comparison is not needed: the tap-box is the kernel both
paths share)."""
import ctypes
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2007_12856_b200 import _lib  # noqa: E402
from paper_2007_12856_b200.frames import frame_desc, stream_ptr  # noqa: E402

SHAPES = {"c3": (32, 64, 128, 1), "c4": (64, 128, 64, 2), "c5": (128, 256, 16, 1)}


def timeit(fn, n=20):
    for _ in range(3):
        fn()
    ts = []
    for _ in range(n):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    return sorted(ts)[n // 2]


out = {}
for name, (cin, cout, W, s) in SHAPES.items():
    o = -(-W // s)
    xfr, yfr = frame_desc(1, cin, W, W, W), frame_desc(1, cout, o, o, o)
    flops = 2 * 27 * cin * cout * o ** 3
    w = torch.randn(cout, cin, 3, 3, 3, device="cuda") * 0.05
    nb = _lib.load().vpx_conv3d_workspace_bytes(cin, cout, 3, ctypes.addressof(yfr))
    ws = torch.empty(nb // 4 + 64, device="cuda")
    res = {}
    for dt, suffix in ((torch.float32, ""), (torch.bfloat16, "_bf16")):
        x = torch.randn(1, W, W, W, cin, device="cuda").to(dt)
        y = torch.empty(1, o, o, o, cout, device="cuda").to(dt)
        u = torch.randn(1, o, o, o, cout, device="cuda").to(dt)
        g = torch.empty(1, W, W, W, cin, device="cuda").to(dt)
        args_f = (x.data_ptr(), ctypes.addressof(xfr), w.data_ptr(), 3, s, y.data_ptr(), ctypes.addressof(yfr),
                  ws.data_ptr(), ws.numel() * 4, stream_ptr())
        args_d = (u.data_ptr(), ctypes.addressof(yfr), w.data_ptr(), 3, s, g.data_ptr(), ctypes.addressof(xfr),
                  ws.data_ptr(), ws.numel() * 4, stream_ptr())
        tf = timeit(lambda: _lib.call("vpx_conv3d_fwd" + suffix, *args_f))
        td = timeit(lambda: _lib.call("vpx_conv3d_bwd_data" + suffix, *args_d))
        res["bf16" if suffix else "tf32"] = {"fwd_ms": tf, "fwd_tflops": flops / tf / 1e9, "dgrad_ms": td,
                                             "dgrad_tflops": flops / td / 1e9}
    out[name] = res
    print(name, json.dumps(res), flush=True)
print(json.dumps(out))
