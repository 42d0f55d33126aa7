"""Quick GPU check of the conv C-ABI against torch fp32 conv3d (CPU, fp64 accumulate).

python tools/check_conv.py  -> prints max-abs/max-ref relative errors per case.
"""

import ctypes
import sys
import time

import numpy as np
import torch
import torch.nn.functional as F

sys.path.insert(0, ".")
from paper_2007_12856_b200 import _lib  # noqa: E402

torch.manual_seed(0)


def frame(n, c, d, h, w, md=0, mh=0, mw=0):
    t = torch.zeros(n, d + 2 * md, h + 2 * mh, w + 2 * mw, c, device="cuda")
    fr = (ctypes.c_int * 8)(n, c, d, h, w, md, mh, mw)
    inner = t[:, md:md + d, mh:mh + h, mw:mw + w, :]
    return t, fr, inner


def rel(a, b):
    return float((a - b).abs().max() / b.abs().max().clamp_min(1e-30))


def ws_for(cin, cout, k, ufr):
    lib = _lib.load()
    nb = lib.vpx_conv3d_workspace_bytes(cin, cout, k, ctypes.addressof(ufr))
    return torch.empty(max(nb, 16) // 4 + 64, device="cuda")


def case(n, cin, cout, D, H, W, k=3, s=1, margins=(0, 0, 0), reps=0):
    st = torch.cuda.current_stream().cuda_stream
    x = torch.randn(n, cin, D, H, W, dtype=torch.float64)
    w = torch.randn(cout, cin, k, k, k, dtype=torch.float64) / np.sqrt(cin * k ** 3)
    r = (k - 1) // 2
    y_ref = F.conv3d(x, w, stride=s, padding=r)
    od, oh, ow = y_ref.shape[2:]
    u = torch.randn_like(y_ref)
    xg_ref = torch.nn.grad.conv3d_input(x.shape, w, u, stride=s, padding=r)
    wg_ref = torch.nn.grad.conv3d_weight(x, w.shape, u, stride=s, padding=r)

    md, mh, mw = margins
    xt, xfr, xin = frame(n, cin, D, H, W, md, mh, mw)
    xin.copy_(x.permute(0, 2, 3, 4, 1).float())
    yt, yfr, yin = frame(n, cout, od, oh, ow)
    ut, ufr, uin = frame(n, cout, od, oh, ow)
    uin.copy_(u.permute(0, 2, 3, 4, 1).float())
    gt, gfr, gin = frame(n, cin, D, H, W)  # no margins for the check
    wd = w.float().cuda().contiguous()
    wgt = torch.zeros_like(wd)
    ws = ws_for(cin, cout, k, ufr)
    args_f = (xt.data_ptr(), ctypes.addressof(xfr), wd.data_ptr(), k, s, yt.data_ptr(),
              ctypes.addressof(yfr), ws.data_ptr(), ws.numel() * 4, st)
    _lib.call("vpx_conv3d_fwd", *args_f)
    _lib.call("vpx_conv3d_bwd_data", ut.data_ptr(), ctypes.addressof(ufr), wd.data_ptr(), k, s,
              gt.data_ptr(), ctypes.addressof(gfr), ws.data_ptr(), ws.numel() * 4, st)
    _lib.call("vpx_conv3d_bwd_filter", xt.data_ptr(), ctypes.addressof(xfr), ut.data_ptr(),
              ctypes.addressof(ufr), k, s, wgt.data_ptr(), 0, ws.data_ptr(), ws.numel() * 4, st)
    torch.cuda.synchronize()
    ey = rel(yin.permute(0, 4, 1, 2, 3).double().cpu(), y_ref)
    eg = rel(gin.permute(0, 4, 1, 2, 3).double().cpu(), xg_ref)
    ew = rel(wgt.double().cpu(), wg_ref)
    msg = f"n={n} cin={cin} cout={cout} {D}x{H}x{W} k={k} s={s} m={margins}: fwd {ey:.2e} dgrad {eg:.2e} wgrad {ew:.2e}"
    if reps:
        torch.cuda.synchronize()
        t0 = time.time()
        for _ in range(reps):
            _lib.call("vpx_conv3d_fwd", *args_f)
        torch.cuda.synchronize()
        dt = (time.time() - t0) / reps
        fl = 2 * 27 * cin * cout * od * oh * ow * n
        msg += f" | fwd {dt * 1e3:.3f} ms {fl / dt / 1e12:.1f} TF/s"
    print(msg, flush=True)
    return max(ey, eg, ew)


if __name__ == "__main__":
    print(_lib.load().vpx_version().decode())
    worst = 0.0
    for args in [
        (1, 4, 16, 4, 8, 128), (2, 4, 16, 3, 5, 256), (1, 16, 32, 4, 4, 128), (1, 32, 64, 3, 3, 128),
        (1, 4, 16, 4, 8, 128, 3, 1, (1, 0, 0)), (1, 16, 32, 4, 4, 128, 3, 1, (1, 1, 0)),
        (1, 64, 128, 8, 8, 8, 3, 2), (1, 8, 2, 6, 6, 6, 1, 1), (1, 128, 256, 4, 4, 4),
    ]:
        worst = max(worst, case(*args))
    case(1, 4, 16, 64, 64, 512, reps=5)
    case(1, 16, 32, 32, 64, 256, reps=5)
    case(1, 32, 64, 32, 32, 128, reps=5)
    print("worst", worst)
