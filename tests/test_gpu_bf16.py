"""BF16 path (GPU): 3x3x3 conv forward / backward-data with bf16 storage on
tcgen05 kind::f16 (vpx_conv3d_fwd_bf16 / vpx_conv3d_bwd_data_bf16, the
tap-box implicit GEMM with 64-channel K chunks, fp32 accumulation), against
the fp32 oracle at the north-star BF16 tolerance rtol 2e-2 in the reference
metric max|got-ref|/max|ref| (reference cli.py:199-202), and against a
BF16-emulating oracle (operands rounded to bf16, fp64 accumulation, output
rounded to bf16) at 1e-2.  Conv semantics: reference _hot.pyx:19-67."""

import ctypes

import numpy as np
import pytest
import torch

from oracle import serial as O
from paper_2007_12856_b200 import _lib
from paper_2007_12856_b200.frames import frame_desc, stream_ptr

pytestmark = pytest.mark.gpu


def rel(got, ref):
    ref = np.asarray(ref, dtype=np.float64)
    return float(np.max(np.abs(np.asarray(got, np.float64) - ref)) / max(np.max(np.abs(ref)), 1e-30))


def bf16_round(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).bfloat16().float().numpy()


CASES = [  # n, cin, cout, d, h, w, stride, margins
    (1, 16, 32, 4, 6, 16, 1, (0, 0, 0)),
    (2, 32, 64, 4, 4, 32, 1, (1, 1, 0)),
    (1, 64, 128, 8, 8, 8, 2, (0, 0, 0)),
    (1, 128, 256, 4, 4, 8, 1, (1, 0, 0)),
    (1, 32, 64, 3, 4, 128, 1, (0, 0, 0)),
    (1, 256, 256, 2, 4, 4, 1, (0, 0, 0)),
]


@pytest.mark.parametrize("case", CASES)
def test_bf16_conv_fwd_and_dgrad(case):
    n, cin, cout, d, h, w, s, m = case
    md, mh, mw = m
    rng = np.random.default_rng(17)
    full = rng.uniform(-1, 1, (n, cin, d + 2 * md, h + 2 * mh, w + 2 * mw)).astype(np.float32)
    wt = (rng.uniform(-1, 1, (cout, cin, 3, 3, 3)) / np.sqrt(27 * cin)).astype(np.float32)
    x = torch.from_numpy(full.transpose(0, 2, 3, 4, 1).copy()).cuda().bfloat16()   # NDHWC bf16 frame
    wd = torch.from_numpy(wt).cuda()
    od, oh, ow = (-(-e // s) for e in (d, h, w))
    y = torch.full((n, od, oh, ow, cout), float("nan"), device="cuda").bfloat16()
    xfr, yfr = frame_desc(n, cin, d, h, w, md, mh, mw), frame_desc(n, cout, od, oh, ow)
    nb = _lib.load().vpx_conv3d_workspace_bytes(cin, cout, 3, ctypes.addressof(yfr))
    W = torch.empty(nb // 4 + 64, device="cuda")
    _lib.call("vpx_conv3d_fwd_bf16", x.data_ptr(), ctypes.addressof(xfr), wd.data_ptr(), 3, s, y.data_ptr(),
              ctypes.addressof(yfr), W.data_ptr(), W.numel() * 4, stream_ptr())
    got = y.float().permute(0, 4, 1, 2, 3).cpu().numpy()
    pads = [(0, 0), (0, 0)] + [(0, 0) if mm else (1, 1) for mm in m]
    xpad = np.pad(full, pads)
    ref32 = O.k_conv3d_fwd(xpad, wt, (s, s, s))
    emu = bf16_round(O.k_conv3d_fwd(bf16_round(xpad).astype(np.float64), bf16_round(wt).astype(np.float64),
                                    (s, s, s)).astype(np.float32))
    assert np.all(np.isfinite(got))
    assert rel(got, ref32) < 2e-2, ("fwd vs fp32", rel(got, ref32))
    assert rel(got, emu) < 1e-2, ("fwd vs bf16-emulated", rel(got, emu))
    # backward-data over the (margin-including) input frame
    u = rng.uniform(-1, 1, (n, cout, od, oh, ow)).astype(np.float32)
    ud = torch.from_numpy(u.transpose(0, 2, 3, 4, 1).copy()).cuda().bfloat16()
    g = torch.full((n, d + 2 * md, h + 2 * mh, w + 2 * mw, cin), float("nan"), device="cuda").bfloat16()
    gfr = frame_desc(n, cin, d, h, w, md, mh, mw)
    ufr = frame_desc(n, cout, od, oh, ow)
    _lib.call("vpx_conv3d_bwd_data_bf16", ud.data_ptr(), ctypes.addressof(ufr), wd.data_ptr(), 3, s, g.data_ptr(),
              ctypes.addressof(gfr), W.data_ptr(), W.numel() * 4, stream_ptr())
    gg = g.float().permute(0, 4, 1, 2, 3).cpu().numpy()
    gref = O.k_conv3d_bwd_data(u, wt, (s, s, s), xpad.shape[2:])
    sl = (slice(None), slice(None)) + tuple(slice(None) if mm else slice(1, -1) for mm in m)
    gref = gref[sl]
    gemu = bf16_round(O.k_conv3d_bwd_data(bf16_round(u).astype(np.float64), bf16_round(wt).astype(np.float64),
                                          (s, s, s), xpad.shape[2:]).astype(np.float32))[sl]
    assert np.all(np.isfinite(gg)), "dgrad left part of the frame (margins included) unwritten"
    assert rel(gg, gref) < 2e-2, ("dgrad vs fp32", rel(gg, gref))
    assert rel(gg, gemu) < 1e-2, ("dgrad vs bf16-emulated", rel(gg, gemu))
