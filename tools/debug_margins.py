"""Probe: conv passes on frames with halo margins, output/workspace pre-filled
with NaN, vs the oracle (one GPU).  Usage: python tools/debug_margins.py"""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from oracle import serial as O
from paper_2007_12856_b200 import _lib
from paper_2007_12856_b200.frames import Frame, stream_ptr

R = O.tf32_round


def rel(a, b):
    b = np.asarray(b, np.float64)
    return float(np.nanmax(np.abs(np.asarray(a, np.float64) - b)) / np.max(np.abs(b))) if np.all(np.isfinite(a)) else float("nan")


def run(cin, cout, d, h, w, s, m, fill):
    rng = np.random.default_rng(0)
    xf = Frame(1, cin, d, h, w, m, zero=True)
    full = R(rng.uniform(-1, 1, tuple(xf.t.shape)).astype(np.float32))
    xf.t.copy_(torch.from_numpy(full).cuda())
    wt = (rng.uniform(-1, 1, (cout, cin, 3, 3, 3)) * 0.2).astype(np.float32)
    wd = torch.from_numpy(wt).cuda()
    od, oh, ow = d // s, h // s, w // s
    yf = Frame(1, cout, od, oh, ow)
    yf.t.fill_(fill)
    nb = _lib.load().vpx_conv3d_workspace_bytes(cin, cout, 3, yf.desc)
    nb = max(nb, BIG)
    ws = torch.full((nb // 4 + 64,), fill, device="cuda")
    _lib.call("vpx_conv3d_fwd", xf.ptr, xf.desc, wd.data_ptr(), 3, s, yf.ptr, yf.desc, ws.data_ptr(), ws.numel() * 4,
              stream_ptr())
    torch.cuda.synchronize()
    got = yf.to_ncdhw().cpu().numpy()
    xn = full.transpose(0, 4, 1, 2, 3)
    pads = [(0, 0), (0, 0)] + [(0, 0) if mm else (1, 1) for mm in m]
    xpad = np.pad(xn, pads)
    ref = R(O._f64(O.k_conv3d_fwd, xpad, R(wt), (s, s, s)))
    # dgrad
    u = Frame(1, cout, od, oh, ow)
    u.t.copy_(torch.from_numpy(R(rng.uniform(-1, 1, tuple(u.t.shape)).astype(np.float32))).cuda())
    g = Frame(1, cin, d, h, w, m, zero=False)
    g.t.fill_(fill)
    ws.fill_(fill)
    _lib.call("vpx_conv3d_bwd_data", u.ptr, u.desc, wd.data_ptr(), 3, s, g.ptr, g.desc, ws.data_ptr(), ws.numel() * 4,
              stream_ptr())
    # wgrad
    wg = torch.full((cout, cin, 3, 3, 3), fill, device="cuda")
    ws.fill_(fill)
    _lib.call("vpx_conv3d_bwd_filter", xf.ptr, xf.desc, u.ptr, u.desc, 3, s, wg.data_ptr(), 0, ws.data_ptr(),
              ws.numel() * 4, stream_ptr())
    torch.cuda.synchronize()
    un = u.to_ncdhw().cpu().numpy()
    gfull = R(O._f64(O.k_conv3d_bwd_data, un, R(wt), (s, s, s), xpad.shape[2:]))
    sl = [slice(None), slice(None)] + [slice(None) if mm else slice(1, -1) for mm in m]
    gref = gfull[tuple(sl)]
    gdev = g.t.permute(0, 4, 1, 2, 3).cpu().numpy()
    wref = O._f64(O.k_conv3d_bwd_filter, xpad, un, (s, s, s), (3, 3, 3))
    return rel(got, ref), rel(gdev, gref), rel(wg.cpu().numpy(), wref)


for cin, cout, d, h, w, s in ((4, 16, 16, 16, 32), (16, 32, 8, 8, 16), (32, 64, 4, 4, 8), (4, 16, 8, 16, 128),
                             (16, 32, 4, 8, 256), (64, 128, 4, 4, 4)), :
    pass
cases = [(4, 16, 16, 16, 32, 1), (16, 32, 8, 8, 16, 1), (32, 64, 4, 4, 8, 1), (64, 128, 8, 8, 8, 2),
         (4, 16, 8, 16, 128, 1), (16, 32, 4, 8, 256, 1), (32, 64, 4, 8, 128, 1), (128, 256, 2, 2, 4, 1)]
import os
BIG = int(os.environ.get("BIG", "0"))
for c in cases:
    for m in ((0, 0, 0), (1, 0, 0), (0, 1, 0), (1, 1, 0), (0, 0, 1), (1, 1, 1)):
        for fill in (0.0, float("nan")):
            try:
                e = run(*c, m, fill)
            except Exception as exc:
                e = f"{type(exc).__name__}: {str(exc)[:80]}"
            print(c, m, fill, e, flush=True)
