"""Per-kernel micro-benchmark at the CosmoFlow-512 layer shapes (one GPU).

python tools/kbench.py [case ...]   cases: c1fwd c1wgrad c2fwd c2dgrad c2wgrad
                                           c3fwd c3dgrad c3wgrad c4fwd c4dgrad c4wgrad
Prints ms / TFLOP/s / GB/s (CUDA events, best of 5 after 2 warm-ups).  Used
for kernel iteration and as the single-kernel command profiled with ncu.
"""

import ctypes
import sys

import torch

sys.path.insert(0, ".")
from paper_2007_12856_b200 import _lib  # noqa: E402
from paper_2007_12856_b200.frames import Frame, frame_desc, stream_ptr  # noqa: E402

L = {  # name: (cin, cout, in extent, stride)
    "c1": (4, 16, 512, 1), "c2": (16, 32, 256, 1), "c3": (32, 64, 128, 1), "c4": (64, 128, 64, 2),
    "c5": (128, 256, 16, 1),
}


def timeit(fn, reps=5):
    for _ in range(2):
        fn()
    best = 1e9
    for _ in range(reps):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        e.synchronize()
        best = min(best, s.elapsed_time(e))
    return best


def run(case):
    layer, kind = case[:2], case[2:]
    cin, cout, E, s = L[layer]
    O = -(-E // s)
    torch.manual_seed(0)
    x = Frame(1, cin, E, E, E)
    x.t.uniform_(-1, 1)
    w = (torch.rand(cout, cin, 3, 3, 3, device="cuda") - 0.5) * 0.1
    y = Frame(1, cout, O, O, O)
    u = Frame(1, cout, O, O, O)
    u.t.uniform_(-1, 1)
    lib = _lib.load()
    ws = torch.empty(lib.vpx_conv3d_workspace_bytes(cin, cout, 3, u.desc) // 4 + 1024, device="cuda")
    flops = 2 * 27 * cin * cout * O ** 3
    st = stream_ptr()
    if kind == "fwd":
        fn = lambda: _lib.call("vpx_conv3d_fwd_act", x.ptr, x.desc, w.data_ptr(), 3, s, y.ptr, y.desc, 1, 0.3,
                               ws.data_ptr(), ws.numel() * 4, st)
        nbytes = 4 * (x.t.numel() + y.t.numel())
    elif kind == "dgrad":
        g = Frame(1, cin, E, E, E)
        fn = lambda: _lib.call("vpx_conv3d_bwd_data", u.ptr, u.desc, w.data_ptr(), 3, s, g.ptr, g.desc,
                               ws.data_ptr(), ws.numel() * 4, st)
        nbytes = 4 * (u.t.numel() + g.t.numel())
    elif kind == "pool":  # the fused first block: conv + leaky + avg pool + sign mask
        pf = Frame(1, cout, O // 2, O // 2, O // 2)
        mask = torch.empty((1, O, O, O), dtype=torch.int16, device="cuda")
        fn = lambda: _lib.call("vpx_conv3d_fwd_leaky_pool_c4", x.ptr, x.desc, w.data_ptr(), 0.3, pf.ptr, pf.desc,
                               mask.data_ptr(), ws.data_ptr(), ws.numel() * 4, st)
        nbytes = 4 * (x.t.numel() + pf.t.numel()) + 2 * mask.numel()
    elif kind == "wgm":  # the fused first-block backward: pooled gradient + sign mask -> filter gradient
        up = Frame(1, cout, O // 2, O // 2, O // 2)
        up.t.uniform_(-1, 1)
        mask = torch.randint(-32768, 32767, (1, O, O, O), dtype=torch.int16, device="cuda")
        wg = torch.empty_like(w)
        mfr = frame_desc(1, cout, O, O, O)
        fn = lambda: _lib.call("vpx_conv3d_bwd_filter_c4_pooled_mask", x.ptr, x.desc, mask.data_ptr(),
                               ctypes.addressof(mfr), up.ptr, up.desc, 0.3, wg.data_ptr(), 0, ws.data_ptr(),
                               ws.numel() * 4, st)
        nbytes = 4 * (x.t.numel() + up.t.numel()) + 2 * mask.numel()
    elif kind == "wgrad" and layer == "c1":
        up = Frame(1, cout, O // 2, O // 2, O // 2)
        up.t.uniform_(-1, 1)
        gb = torch.empty(u.t.numel(), device="cuda")
        wg = torch.empty_like(w)
        ufr = frame_desc(1, cout, O, O, O)

        def fn():
            _lib.call("vpx_pool_leaky_bwd_blocked", u.ptr, u.desc, up.ptr, up.desc, gb.data_ptr(), 0.3, 0, st)
            _lib.call("vpx_conv3d_bwd_filter_c4", x.ptr, x.desc, gb.data_ptr(), ctypes.addressof(ufr),
                      wg.data_ptr(), 0, ws.data_ptr(), ws.numel() * 4, st)
        nbytes = 4 * (x.t.numel() + u.t.numel())
    else:
        wg = torch.empty_like(w)
        fn = lambda: _lib.call("vpx_conv3d_bwd_filter", x.ptr, x.desc, u.ptr, u.desc, 3, s, wg.data_ptr(), 0,
                               ws.data_ptr(), ws.numel() * 4, st)
        nbytes = 4 * (x.t.numel() + u.t.numel())
    ms = timeit(fn)
    print(f"{case:10s} {ms:8.3f} ms  {flops / ms / 1e9:8.1f} TFLOP/s  {nbytes / ms / 1e6:8.1f} GB/s", flush=True)


if __name__ == "__main__":
    cases = sys.argv[1:] or ["c1fwd", "c1wgrad", "c2fwd", "c2dgrad", "c2wgrad", "c3fwd", "c3dgrad", "c3wgrad",
                             "c4fwd", "c4dgrad", "c4wgrad"]
    for c in cases:
        run(c)
