"""Device kernels vs the CPU oracle (GPU).  Conv runs on tcgen05 in TF32:
tolerance rtol 1e-3 in the reference's metric max|got-ref| / max|ref|
(reference cli.py:199-202); pointwise/pool/layout/prng/halo are exact."""

import ctypes
import json
import os

import numpy as np
import pytest
import torch

from oracle import serial as O
from paper_2007_12856_b200 import _lib, get_precision, prng
from paper_2007_12856_b200.frames import Frame, frame_desc, stream_ptr

pytestmark = pytest.mark.gpu

TF32_RTOL = 1e-3


def rel(got, ref):
    ref = np.asarray(ref, dtype=np.float64)
    return float(np.max(np.abs(np.asarray(got, np.float64) - ref)) / max(np.max(np.abs(ref)), 1e-30))


def ws(cin, cout, k, fr):
    nb = _lib.load().vpx_conv3d_workspace_bytes(cin, cout, k, fr.desc)
    return torch.empty(nb // 4 + 64, device="cuda")


def run_conv(x, w, k, s, margins=(0, 0, 0), grad_margins=(0, 0, 0)):
    n, cin, d, h, wd = x.shape
    cout = w.shape[0]
    xf = Frame(n, cin, d, h, wd, margins, zero=True).load_ncdhw(x)
    od, oh, ow = (-(-e // s) for e in (d, h, wd))
    yf = Frame(n, cout, od, oh, ow)
    wt = torch.from_numpy(np.ascontiguousarray(w)).float().cuda()
    W = ws(cin, cout, k, yf)
    _lib.call("vpx_conv3d_fwd", xf.ptr, xf.desc, wt.data_ptr(), k, s, yf.ptr, yf.desc, W.data_ptr(),
              W.numel() * 4, stream_ptr())
    return xf, yf, wt, W


CASES = [
    # n, cin, cout, d, h, w, k, s   (tcgen05 row-window for W%128==0 stride 1, else CUDA-core)
    (1, 4, 16, 4, 6, 128, 3, 1),
    (2, 4, 16, 3, 5, 256, 3, 1),
    (1, 16, 32, 4, 4, 128, 3, 1),
    (2, 16, 32, 3, 6, 256, 3, 1),      # u-in-TMEM filter gradient (W = 256)
    (1, 8, 8, 4, 4, 128, 3, 1),        # U-Net 8-channel levels: rowh N padded 24 -> 32
    (1, 16, 8, 3, 4, 256, 3, 1),
    # grouped-voxel filter gradient (Cin = Cout <= 32, conv_wgrad_g.cu)
    (2, 8, 8, 3, 5, 256, 3, 1),
    (1, 8, 8, 3, 3, 32, 3, 1),
    (1, 16, 16, 3, 4, 128, 3, 1),
    (1, 32, 32, 2, 3, 64, 3, 1),
    (1, 32, 64, 3, 3, 128, 3, 1),
    (1, 64, 128, 8, 8, 8, 3, 2),
    (1, 128, 256, 4, 4, 4, 3, 1),
    (2, 8, 2, 6, 6, 6, 1, 1),
    # U-Net edges on CUDA cores (conv_small.cu): 1x1x1 head, 1-channel first layer
    (1, 8, 2, 3, 4, 256, 1, 1),
    (1, 16, 4, 2, 3, 40, 1, 1),
    (1, 1, 8, 3, 5, 100, 3, 1),
    (2, 1, 8, 4, 6, 64, 3, 1),
    (1, 1, 16, 2, 9, 70, 3, 1),
    # tcgen05 filter gradient: mode A (Cin <= 32, W taps folded into M) ...
    (1, 4, 16, 3, 4, 32, 3, 1),
    (2, 16, 32, 3, 3, 16, 3, 1),
    (1, 32, 64, 2, 5, 8, 3, 1),
    # ... and mode B (Cin % 128 == 0, W <= 32)
    (1, 128, 256, 3, 4, 16, 3, 1),
    (1, 256, 256, 2, 4, 8, 3, 1),
    (1, 64, 128, 4, 4, 16, 3, 1),      # partial 128-channel tile
    (1, 64, 128, 8, 16, 32, 3, 2),     # stride 2 (TMA element stride), the c4 shape
    (2, 192, 128, 4, 8, 16, 3, 2),
    # tap-box fwd/dgrad: W < 128, channel chunks padded by TMA zero fill, stride 2
    (1, 16, 32, 4, 6, 16, 3, 1),
    (2, 32, 64, 4, 4, 32, 3, 1),
    (1, 64, 128, 16, 16, 16, 3, 2),
    (1, 256, 256, 8, 8, 8, 3, 1),
    # W < 8 filter gradients (one zero-padded 8-voxel K step per row): CosmoFlow-512 c7, stride-2 c4 at 8^3
    (1, 256, 256, 4, 4, 4, 3, 1),
    (2, 128, 256, 4, 4, 4, 3, 1),
    (1, 64, 128, 8, 8, 8, 3, 2),
]


@pytest.mark.parametrize("shape,margins", [((1, 4, 6, 64), (0, 0, 0)), ((2, 4, 2, 128), (1, 0, 0)),
                                           ((1, 2, 4, 512), (1, 1, 0))])
def test_first_block_fused_backward_and_c4_wgrad(shape, margins):
    """c1 fast path: pooled gradient -> (pool bwd + leaky bwd, blocked layout)
    -> dense Cin=4 filter gradient, against the oracle composition."""
    n, d, h, w = shape
    rng = np.random.default_rng(21)
    x = rng.uniform(-1, 1, (n, 4, d, h, w)).astype(np.float32)
    y = rng.uniform(-1, 1, (n, 16, d, h, w)).astype(np.float32)   # leaky output (= pool input)
    up = rng.uniform(-1, 1, (n, 16, d // 2, h // 2, w // 2)).astype(np.float32)
    xf = Frame(n, 4, d, h, w, margins, zero=True).load_ncdhw(x)
    yf, uf = _frame_of(y), _frame_of(up)
    gb = torch.empty(4 * n * d * h * w * 4, device="cuda")
    _lib.call("vpx_pool_leaky_bwd_blocked", yf.ptr, yf.desc, uf.ptr, uf.desc, gb.data_ptr(), 0.3, 0, stream_ptr())
    yr = yf.to_ncdhw().cpu().numpy()  # as stored (TF32-rounded)
    g_ref = O.leaky_bwd(yr, O.pool3d_bwd(yr, uf.to_ncdhw().cpu().numpy(), "average"), 0.3)
    got = gb.view(4, n, d, h, w, 4).permute(1, 0, 5, 2, 3, 4).reshape(n, 16, d, h, w).cpu().numpy()
    assert rel(got, g_ref) < 1e-3
    wg = torch.zeros(16, 4, 3, 3, 3, device="cuda")
    from paper_2007_12856_b200.frames import frame_desc

    ufr = frame_desc(n, 16, d, h, w)
    W = ws(4, 16, 3, Frame(n, 16, d, h, w))
    _lib.call("vpx_conv3d_bwd_filter_c4", xf.ptr, xf.desc, gb.data_ptr(), ctypes.addressof(ufr), wg.data_ptr(), 0,
              W.data_ptr(), W.numel() * 4, stream_ptr())
    wg_ref = O.conv3d_bwd_filter(xf.to_ncdhw().cpu().numpy(), got, (3, 3, 3), (1, 1, 1))
    assert rel(wg.cpu().numpy(), wg_ref) < TF32_RTOL
    # one-kernel variant: pooled gradient -> u in TMEM -> filter gradient; the
    # pooled gradient arrives with the same D/H margins as x here
    upf = Frame(n, 16, d // 2, h // 2, w // 2, margins, zero=True).load_ncdhw(uf.to_ncdhw())
    wg2 = torch.zeros(16, 4, 3, 3, 3, device="cuda")
    _lib.call("vpx_conv3d_bwd_filter_c4_pooled", xf.ptr, xf.desc, yf.ptr, yf.desc, upf.ptr, upf.desc, 0.3, 0,
              wg2.data_ptr(), 0, W.data_ptr(), W.numel() * 4, stream_ptr())
    assert rel(wg2.cpu().numpy(), wg_ref) < TF32_RTOL
    assert rel(wg2.cpu().numpy(), wg.cpu().numpy()) < 1e-5  # same rounded operands, other summation order


@pytest.mark.parametrize("shape,margins", [((1, 4, 6, 128), (0, 0, 0)), ((2, 2, 4, 256), (1, 1, 0)),
                                           ((1, 2, 34, 128), (0, 0, 0)), ((1, 2, 44, 256), (1, 1, 0))])
def test_first_block_fused_forward_and_mask_backward(shape, margins):
    """conv(4->16)+leaky+avg-pool in one kernel (pooled output + sign mask)
    against the unfused conv/pool kernels: the fused kernel sums the three
    height taps in TMEM (the unfused one in its epilogue), so the activations
    agree to within one TF32 rounding step -- pooled values within 2^-10 of
    the maximum, sign bits equal wherever the activation is not ~0.  The
    mask-driven filter gradient equals the y-driven one bit for bit."""
    n, d, h, w = shape
    rng = np.random.default_rng(5)
    x = rng.uniform(-1, 1, (n, 4, d, h, w)).astype(np.float32)
    wt = torch.from_numpy((rng.uniform(-1, 1, (16, 4, 3, 3, 3)) / 5).astype(np.float32)).cuda()
    xf = Frame(n, 4, d, h, w, margins, zero=True).load_ncdhw(x)
    W = ws(4, 16, 3, Frame(n, 16, d, h, w))
    # unfused reference path: conv + fused leaky epilogue, then pool
    yf = Frame(n, 16, d, h, w)
    _lib.call("vpx_conv3d_fwd_act", xf.ptr, xf.desc, wt.data_ptr(), 3, 1, yf.ptr, yf.desc, 1, 0.3, W.data_ptr(),
              W.numel() * 4, stream_ptr())
    pref = Frame(n, 16, d // 2, h // 2, w // 2, margins, zero=True)
    _lib.call("vpx_pool_fwd", yf.ptr, yf.desc, pref.ptr, pref.desc, 0, stream_ptr())
    # fused
    pf = Frame(n, 16, d // 2, h // 2, w // 2, margins, zero=True)
    mask = torch.zeros((n, d, h, w), dtype=torch.int16, device="cuda")
    _lib.call("vpx_conv3d_fwd_leaky_pool_c4", xf.ptr, xf.desc, wt.data_ptr(), 0.3, pf.ptr, pf.desc,
              mask.data_ptr(), W.data_ptr(), W.numel() * 4, stream_ptr())
    torch.cuda.synchronize()
    assert float((pf.t - pref.t).abs().max()) <= 2.0 ** -10 * float(pref.t.abs().max())
    ybits = (yf.t >= 0).to(torch.int32) * (2 ** torch.arange(16, device="cuda", dtype=torch.int32))
    ymask = ybits.sum(-1) & 0xFFFF
    yi = yf.t  # conv output frame (no margins)
    diff = (mask.to(torch.int32) & 0xFFFF) != ymask
    near0 = (yi.abs() <= 1e-5 * float(yi.abs().max())).any(-1)
    assert not bool((diff & ~near0).any())
    mask = ymask.to(torch.int16)  # the backward check below drives both paths from the same y
    # backward from a pooled gradient
    up = rng.uniform(-1, 1, (n, 16, d // 2, h // 2, w // 2)).astype(np.float32)
    upf = Frame(n, 16, d // 2, h // 2, w // 2, margins, zero=True).load_ncdhw(up)
    wg_y = torch.zeros(16, 4, 3, 3, 3, device="cuda")
    wg_m = torch.zeros(16, 4, 3, 3, 3, device="cuda")
    _lib.call("vpx_conv3d_bwd_filter_c4_pooled", xf.ptr, xf.desc, yf.ptr, yf.desc, upf.ptr, upf.desc, 0.3, 0,
              wg_y.data_ptr(), 0, W.data_ptr(), W.numel() * 4, stream_ptr())
    from paper_2007_12856_b200.frames import frame_desc

    mfr = frame_desc(n, 16, d, h, w)
    _lib.call("vpx_conv3d_bwd_filter_c4_pooled_mask", xf.ptr, xf.desc, mask.data_ptr(), ctypes.addressof(mfr),
              upf.ptr, upf.desc, 0.3, wg_m.data_ptr(), 0, W.data_ptr(), W.numel() * 4, stream_ptr())
    torch.cuda.synchronize()
    assert torch.equal(wg_y, wg_m)


@pytest.mark.parametrize("cin,cout,spatial,stride", [(256, 256, (4, 4, 4), 1), (256, 256, (8, 8, 8), 1),
                                                    (128, 256, (8, 8, 8), 2), (256, 256, (8, 8, 8), 2)])
def test_tapbox_row_pack_bit_exact(cin, cout, spatial, stride, monkeypatch):
    """Deep-layer tap-box passes (split K): the row-staged weight pack gives
    the same bits as the element-wise pack, forward and backward-data, and
    the forward stays within the TF32 tolerance of the oracle."""
    rng = np.random.default_rng(17)
    n = 1
    x = O.tf32_round(rng.standard_normal((n, cin) + spatial).astype(np.float32))
    w = (rng.standard_normal((cout, cin, 3, 3, 3)) / np.sqrt(27 * cin)).astype(np.float32)
    od = tuple(-(-e // stride) for e in spatial)
    u = O.tf32_round(rng.standard_normal((n, cout) + od).astype(np.float32))
    wt = torch.from_numpy(w).cuda()

    def run():
        xf = Frame(n, cin, *spatial, (1, 1, 0), zero=True).load_ncdhw(x)
        yf = Frame(n, cout, *od)
        W = ws(cin, cout, 3, yf)
        _lib.call("vpx_conv3d_fwd", xf.ptr, xf.desc, wt.data_ptr(), 3, stride, yf.ptr, yf.desc, W.data_ptr(),
                  W.numel() * 4, stream_ptr())
        uf = Frame(n, cout, *od).load_ncdhw(u)
        gf = Frame(n, cin, *spatial, (1, 1, 0), zero=True)
        _lib.call("vpx_conv3d_bwd_data", uf.ptr, uf.desc, wt.data_ptr(), 3, stride, gf.ptr, gf.desc, W.data_ptr(),
                  W.numel() * 4, stream_ptr())
        torch.cuda.synchronize()
        return yf.t.clone(), gf.t.clone()

    y1, g1 = run()
    monkeypatch.setenv("VPX_PACK_ELEMWISE", "1")
    y2, g2 = run()
    assert torch.equal(y1.view(torch.int32), y2.view(torch.int32))
    assert torch.equal(g1.view(torch.int32), g2.view(torch.int32))
    assert rel(Frame(n, cout, *od, tensor=y1).to_ncdhw().cpu().numpy(),
               O.k_conv3d_fwd(np.pad(x, ((0, 0), (0, 0), (1, 1), (1, 1), (1, 1))), w, (stride,) * 3)) < TF32_RTOL


def test_tapbox_dgrad_all_margins():
    """W-partitioned frames (margins in all three dims) go through the tap-box
    kernel for both passes."""
    rng = np.random.default_rng(11)
    n, cin, cout, d, h, w = 1, 32, 64, 4, 4, 16
    full = rng.uniform(-1, 1, (n, cin, d + 2, h + 2, w + 2)).astype(np.float32)
    wt = (rng.uniform(-1, 1, (cout, cin, 3, 3, 3)) / 30).astype(np.float32)
    xf = Frame(n, cin, d, h, w, (1, 1, 1), zero=True)
    xf.t.copy_(torch.from_numpy(full.transpose(0, 2, 3, 4, 1).copy()).cuda())
    yf = Frame(n, cout, d, h, w)
    wdev = torch.from_numpy(wt).cuda()
    W = ws(cin, cout, 3, yf)
    _lib.call("vpx_conv3d_fwd", xf.ptr, xf.desc, wdev.data_ptr(), 3, 1, yf.ptr, yf.desc, W.data_ptr(),
              W.numel() * 4, stream_ptr())
    assert rel(yf.to_ncdhw().cpu().numpy(), O.k_conv3d_fwd(full, wt, (1, 1, 1))) < TF32_RTOL
    u = rng.uniform(-1, 1, (n, cout, d, h, w)).astype(np.float32)
    uf = Frame(n, cout, d, h, w).load_ncdhw(u)
    gf = Frame(n, cin, d, h, w, (1, 1, 1), zero=False)
    _lib.call("vpx_conv3d_bwd_data", uf.ptr, uf.desc, wdev.data_ptr(), 3, 1, gf.ptr, gf.desc, W.data_ptr(),
              W.numel() * 4, stream_ptr())
    g_ref = O.k_conv3d_bwd_data(u, wt, (1, 1, 1), (d + 2, h + 2, w + 2))
    assert rel(gf.t.cpu().numpy().transpose(0, 4, 1, 2, 3), g_ref) < TF32_RTOL


@pytest.mark.parametrize("case", CASES)
def test_conv_passes_vs_oracle(case):
    n, cin, cout, d, h, w, k, s = case
    rng = np.random.default_rng(7)
    x = rng.uniform(-1, 1, (n, cin, d, h, w)).astype(np.float32)
    wt = (rng.uniform(-1, 1, (cout, cin, k, k, k)) / np.sqrt(cin * k ** 3)).astype(np.float32)
    xf, yf, wdev, W = run_conv(x, wt, k, s)
    y_ref = O.conv3d(x, wt, (k,) * 3, (s,) * 3)
    assert rel(yf.to_ncdhw().cpu().numpy(), y_ref) < TF32_RTOL
    u = rng.uniform(-1, 1, y_ref.shape).astype(np.float32)
    uf = Frame(*u.shape[:1], u.shape[1], *u.shape[2:]).load_ncdhw(u)
    gf = Frame(n, cin, d, h, w)
    _lib.call("vpx_conv3d_bwd_data", uf.ptr, uf.desc, wdev.data_ptr(), k, s, gf.ptr, gf.desc, W.data_ptr(),
              W.numel() * 4, stream_ptr())
    g_ref = O.conv3d_bwd_data(u, wt, (k,) * 3, (s,) * 3, (d, h, w))
    assert rel(gf.to_ncdhw().cpu().numpy(), g_ref) < TF32_RTOL
    wg = torch.zeros_like(wdev)
    _lib.call("vpx_conv3d_bwd_filter", xf.ptr, xf.desc, uf.ptr, uf.desc, k, s, wg.data_ptr(), 0, W.data_ptr(),
              W.numel() * 4, stream_ptr())
    wg_ref = O.conv3d_bwd_filter(x, u, (k,) * 3, (s,) * 3)
    assert rel(wg.cpu().numpy(), wg_ref) < TF32_RTOL


@pytest.mark.parametrize("cout,spatial,stride", [(128, (8, 8, 16), 2), (128, (4, 6, 8), 1), (256, (4, 4, 16), 1),
                                                 (128, (6, 8, 64), 2), (128, (4, 4, 8), 2)])
def test_wgrad_tap_pairs(cout, spatial, stride, monkeypatch):
    """64-input-channel filter gradients (CosmoFlow c4) put two taps in the
    128-row MMA tile; same result as the one-tap tiles (VPX_WGRAD_NOPAIR, a
    different split-K partition, so equal up to fp32 summation order) and the
    oracle, on a frame with D/H margins as under a spatial split."""
    rng = np.random.default_rng(11)
    n, cin = 1, 64
    x = O.tf32_round(rng.uniform(-1, 1, (n, cin) + spatial).astype(np.float32))
    od = tuple(-(-e // stride) for e in spatial)
    u = O.tf32_round(rng.uniform(-1, 1, (n, cout) + od).astype(np.float32))
    xf = Frame(n, cin, *spatial, (1, 1, 0), zero=True).load_ncdhw(x)
    uf = Frame(n, cout, *od).load_ncdhw(u)
    W = ws(cin, cout, 3, uf)

    def run():
        wg = torch.zeros(cout, cin, 3, 3, 3, device="cuda")
        _lib.call("vpx_conv3d_bwd_filter", xf.ptr, xf.desc, uf.ptr, uf.desc, 3, stride, wg.data_ptr(), 0,
                  W.data_ptr(), W.numel() * 4, stream_ptr())
        torch.cuda.synchronize()
        return wg.cpu().numpy()

    got = run()
    monkeypatch.setenv("VPX_WGRAD_NOPAIR", "1")
    one = run()
    assert np.abs(got - one).max() <= 1e-5 * np.abs(one).max()
    assert rel(got, O.conv3d_bwd_filter(x, u, (3,) * 3, (stride,) * 3)) < TF32_RTOL


@pytest.mark.parametrize("cin,cout,spatial", [(64, 128, (16, 16, 16)), (64, 128, (6, 10, 32)), (128, 256, (8, 8, 8))])
def test_tapbox_stride2_dgrad_balanced_tiles_bit_exact(cin, cout, spatial, monkeypatch):
    """Stride-2 backward-data deals its tiles heaviest parity class first,
    serpentine over the CTAs; every tile is still computed whole by one CTA,
    so the gradient has the same bits as the round-robin order
    (VPX_TAPBOX_RR) and stays within the TF32 tolerance of the oracle."""
    rng = np.random.default_rng(5)
    n = 1
    w = (rng.standard_normal((cout, cin, 3, 3, 3)) / np.sqrt(27 * cin)).astype(np.float32)
    od = tuple(-(-e // 2) for e in spatial)
    u = O.tf32_round(rng.standard_normal((n, cout) + od).astype(np.float32))
    wt = torch.from_numpy(w).cuda()
    uf = Frame(n, cout, *od).load_ncdhw(u)

    def run():
        gf = Frame(n, cin, *spatial, (1, 1, 0), zero=True)
        W = ws(cin, cout, 3, gf)
        _lib.call("vpx_conv3d_bwd_data", uf.ptr, uf.desc, wt.data_ptr(), 3, 2, gf.ptr, gf.desc, W.data_ptr(),
                  W.numel() * 4, stream_ptr())
        torch.cuda.synchronize()
        return gf

    g1 = run()
    monkeypatch.setenv("VPX_TAPBOX_RR", "1")
    g2 = run()
    assert torch.equal(g1.t, g2.t)
    g_ref = O.conv3d_bwd_data(u, O.tf32_round(w), (3,) * 3, (2,) * 3, spatial)
    assert rel(g1.to_ncdhw().cpu().numpy(), g_ref) < TF32_RTOL


def test_conv_fwd_frame_margins_and_dgrad_margins():
    """D/H-partitioned frames: the kernel must read the margin rows (here
    filled with neighbour data) and write dgrad over the margins too."""
    rng = np.random.default_rng(3)
    n, cin, cout, d, h, w = 1, 16, 32, 4, 4, 128
    full = rng.uniform(-1, 1, (n, cin, d + 2, h + 2, w)).astype(np.float32)  # as if halos were received
    wt = (rng.uniform(-1, 1, (cout, cin, 3, 3, 3)) / 20).astype(np.float32)
    xf = Frame(n, cin, d, h, w, (1, 1, 0), zero=True)
    xf.t.copy_(torch.from_numpy(full.transpose(0, 2, 3, 4, 1).copy()).cuda())
    yf = Frame(n, cout, d, h, w)
    wdev = torch.from_numpy(wt).cuda()
    W = ws(cin, cout, 3, yf)
    _lib.call("vpx_conv3d_fwd", xf.ptr, xf.desc, wdev.data_ptr(), 3, 1, yf.ptr, yf.desc, W.data_ptr(),
              W.numel() * 4, stream_ptr())
    # reference: conv over the margin-extended block, keep the interior rows
    xpad = np.pad(full, ((0, 0), (0, 0), (0, 0), (0, 0), (1, 1)))
    y_ref = O.k_conv3d_fwd(xpad, wt, (1, 1, 1))
    assert rel(yf.to_ncdhw().cpu().numpy(), y_ref) < TF32_RTOL
    u = rng.uniform(-1, 1, (n, cout, d, h, w)).astype(np.float32)
    uf = Frame(n, cout, d, h, w).load_ncdhw(u)
    gf = Frame(n, cin, d, h, w, (1, 1, 0), zero=False)
    _lib.call("vpx_conv3d_bwd_data", uf.ptr, uf.desc, wdev.data_ptr(), 3, 1, gf.ptr, gf.desc, W.data_ptr(),
              W.numel() * 4, stream_ptr())
    g_ref = O.k_conv3d_bwd_data(u, wt, (1, 1, 1), (d + 2, h + 2, w + 2))[:, :, :, :, 1:-1]
    got = gf.t.cpu().numpy().transpose(0, 4, 1, 2, 3)
    assert rel(got, g_ref) < TF32_RTOL


def test_prng_device_streams_bit_exact(golden):
    g = json.loads((golden / "prng.json").read_text())
    for k in g["uniform"]:
        key = json.loads(k)
        dev = prng.uniform_device(key, 16, -0.5, 2.0, fp64=True).cpu().numpy()
        assert dev.tolist() == g["uniform"][k]
    big = prng.uniform_device([0, -3, 0], 1 << 20, -1.0, 1.0).cpu().numpy()
    import hashlib

    assert hashlib.sha256(big.tobytes()).hexdigest() == g["uniform_1M_f32_bytes_sha"]
    m = prng.keep_mask_device([0, 1, 2, 3, 4], 64, 0.8).cpu().numpy().astype(bool)
    assert np.array_equal(m, O.dropout_mask([0, 1, 2, 3, 4], 64, 0.8))


def _frame_of(a):
    return Frame(a.shape[0], a.shape[1], *a.shape[2:]).load_ncdhw(a.astype(np.float32))


@pytest.fixture
def fp32_mode():
    import paper_2007_12856_b200 as pkg

    pkg.set_precision("fp32")
    yield
    pkg.set_precision("tf32")


def test_tf32_storage_rounds_to_nearest():
    """In TF32 mode every stored activation is the nearest TF32 value (low 13
    mantissa bits zero, round-to-nearest), so the tensor core sees it exactly."""
    x = np.random.default_rng(4).standard_normal((1, 8, 2, 4, 4)).astype(np.float32)
    f = _frame_of(x)
    got = f.to_ncdhw().cpu().numpy()
    assert np.all(got.view(np.uint32) & np.uint32(0x1FFF) == 0)
    assert np.max(np.abs(got - x) / np.abs(x)) <= 2.0 ** -11


def test_pool_leaky_bn_deconv_vs_oracle(golden, fp32_mode):
    A = np.load(golden / "layers.npz")
    x = A["pool_x"].astype(np.float32)
    xf = _frame_of(x)
    for kind in ("average", "max"):
        yf = Frame(x.shape[0], x.shape[1], x.shape[2] // 2, x.shape[3] // 2, x.shape[4] // 2)
        _lib.call("vpx_pool_fwd", xf.ptr, xf.desc, yf.ptr, yf.desc, int(kind == "max"), stream_ptr())
        assert rel(yf.to_ncdhw().cpu().numpy(), O.pool3d(x, kind)) < 1e-6
        u = A[f"pool_{kind}_u"].astype(np.float32)
        uf = _frame_of(u)
        gf = Frame(*x.shape[:2], *x.shape[2:])
        _lib.call("vpx_pool_bwd", xf.ptr, xf.desc, uf.ptr, uf.desc, gf.ptr, gf.desc, int(kind == "max"), stream_ptr())
        assert np.array_equal(gf.to_ncdhw().cpu().numpy(), O.pool3d_bwd(x, u, kind))
    # leaky is exact
    lx = np.random.default_rng(1).standard_normal((2, 3, 4, 4, 4)).astype(np.float32)
    lx[0, 0, 0, 0, 0] = 0.0
    lu = np.random.default_rng(2).standard_normal(lx.shape).astype(np.float32)
    a, b, c = _frame_of(lx), _frame_of(lu), Frame(2, 3, 4, 4, 4)
    _lib.call("vpx_leaky_fwd", a.ptr, a.desc, c.ptr, c.desc, 0.3, stream_ptr())
    assert np.array_equal(c.to_ncdhw().cpu().numpy(), O.leaky(lx, 0.3))
    _lib.call("vpx_leaky_bwd", a.ptr, a.desc, b.ptr, b.desc, c.ptr, c.desc, 0.3, stream_ptr())
    assert np.array_equal(c.to_ncdhw().cpu().numpy(), O.leaky_bwd(lx, lu, 0.3))
    # deconv
    dx, dw, du = A["deconv_x"].astype(np.float32), A["deconv_w"].astype(np.float32), A["deconv_u"].astype(np.float32)
    xf, uf = _frame_of(dx), _frame_of(du)
    yf = Frame(dx.shape[0], dw.shape[1], *(2 * e for e in dx.shape[2:]))
    wdev = torch.from_numpy(dw).cuda()
    W = torch.empty(_lib.load().vpx_deconv_workspace_bytes(dx.shape[1], dw.shape[1]) // 4, device="cuda")
    _lib.call("vpx_deconv_fwd", xf.ptr, xf.desc, wdev.data_ptr(), yf.ptr, yf.desc, W.data_ptr(), W.numel() * 4,
              stream_ptr())
    assert rel(yf.to_ncdhw().cpu().numpy(), A["deconv_y"]) < 1e-5
    gf = Frame(*dx.shape[:2], *dx.shape[2:])
    _lib.call("vpx_deconv_bwd_data", uf.ptr, uf.desc, wdev.data_ptr(), gf.ptr, gf.desc, W.data_ptr(), W.numel() * 4,
              stream_ptr())
    assert rel(gf.to_ncdhw().cpu().numpy(), A["deconv_g"]) < 1e-5
    wg = torch.zeros_like(wdev)
    _lib.call("vpx_deconv_bwd_filter", xf.ptr, xf.desc, uf.ptr, uf.desc, wg.data_ptr(), 0, W.data_ptr(), stream_ptr())
    assert rel(wg.cpu().numpy(), A["deconv_wg"]) < 1e-5


def test_halo_copy_round_trip():
    t = Frame(2, 3, 4, 5, 6, (1, 1, 1), zero=True)
    t.t.copy_(torch.arange(t.t.numel(), dtype=torch.float32, device="cuda").view_as(t.t))
    box = (1, 0, 1, 2, 1, 4, 3, 5)  # n0, z0, y0, x0, en, ez, ey, ex
    buf = torch.empty(1 * 4 * 3 * 5 * 3, device="cuda")
    from paper_2007_12856_b200.comm import copy_box

    copy_box(t, box, buf, 0)
    ref = t.t[1:2, 0:4, 1:4, 2:7, :].reshape(-1)
    assert torch.equal(buf, ref)
    before = t.t.clone()
    copy_box(t, box, buf, 2)
    assert torch.equal(t.t[1:2, 0:4, 1:4, 2:7, :], 2 * before[1:2, 0:4, 1:4, 2:7, :])


@pytest.mark.parametrize("dims,margins,c", [((2, 6, 5, 7), (1, 0, 0), 8), ((1, 4, 300, 9), (0, 1, 0), 16)])
def test_halo_round_peer_loopback(dims, margins, c):
    """vpx_halo_round_peer on one GPU wired as a ring of one: face -1 sends
    into mailbox A (read by face +1), face +1 into mailbox B (read by face -1),
    so the margins receive the opposite boundary slabs (a periodic wrap).
    Checks the pack/unpack boxes, the accumulate mode, and that the block
    counters and expected-arrival counts come back consistent across calls."""
    n, d, h, w = dims
    t = Frame(n, c, d, h, w, margins, zero=True)
    interior = torch.randn((n, d, h, w, c), device="cuda")
    t.interior.copy_(interior)
    dim = margins.index(1)
    ext = [d + 2 * margins[0], h + 2 * margins[1], w + 2 * margins[2]]
    slab = n * c * ext[0] * ext[1] * ext[2]
    mail = torch.zeros(2 * slab, device="cuda")
    flags = torch.zeros(64, dtype=torch.int64, device="cuda")  # 0,1 flags; 8,9 expected; 16.. counters; 32 error
    base = flags.data_ptr()

    def box(lo, size):
        b = [0, 0, 0, 0, n, ext[0], ext[1], ext[2]]
        b[1 + dim], b[5 + dim] = lo, size
        return b

    e = ext[dim]
    # side -1: send the first interior slab, receive into the low margin
    # side +1: send the last interior slab, receive into the high margin
    faces = [(box(1, 1), box(0, 1)), (box(e - 2, 1), box(e - 1, 1))]

    def run(mode):
        desc = [0] * 64
        desc[23] = base + 16 * 8
        for s, (sb, rb) in enumerate(faces):
            o = 32 * s
            desc[o + 0], desc[o + 11], desc[o + 24] = 1, 1, mode
            desc[o + 1:o + 9], desc[o + 12:o + 20] = sb, rb
            desc[o + 9] = mail.data_ptr() + 4 * slab * s          # face s writes mailbox s
            desc[o + 10] = base + 8 * s
            desc[o + 20] = mail.data_ptr() + 4 * slab * (1 - s)   # and reads the other one
            desc[o + 21] = base + 8 * (1 - s)
            desc[o + 22] = base + 8 * (8 + s)
        arr = (ctypes.c_longlong * 64)(*desc)
        _lib.call("vpx_halo_round_peer", t.ptr, t.desc, ctypes.addressof(arr), 4 * slab, 5_000_000_000,
                  base + 32 * 8, stream_ptr())
        torch.cuda.synchronize()

    def sl(lo):
        idx = [slice(None)] * 5
        idx[1 + dim] = slice(lo, lo + 1)
        return tuple(idx)

    run(1)
    assert torch.equal(t.t[sl(0)], t.t[sl(e - 2)]) and torch.equal(t.t[sl(e - 1)], t.t[sl(1)])
    run(2)  # accumulate: the margins now hold twice the opposite slab
    assert torch.equal(t.t[sl(0)], 2 * t.t[sl(e - 2)]) and torch.equal(t.t[sl(e - 1)], 2 * t.t[sl(1)])
    f = flags.cpu()
    assert f[0] == f[1] == 2 and f[8] == f[9] == 2  # two arrivals per face, both consumed
    assert int(f[16]) == 0 and int(f[17]) == 0 and int(f[32]) == 0  # block counters back at rest, no error


@pytest.mark.parametrize("cin,cout,spatial", [(16, 8, (3, 4, 40)), (32, 16, (2, 3, 64)), (32, 8, (2, 2, 33))])
def test_deconv_vectorised_vs_oracle(cin, cout, spatial, fp32_mode):
    """Transposed conv fwd / dgrad / wgrad on the float4 row kernels (ops_unet.cu),
    partial 32-voxel tiles included; fp32 CUDA-core arithmetic."""
    rng = np.random.default_rng(11)
    x = rng.standard_normal((2, cin) + spatial).astype(np.float32)
    w = (rng.standard_normal((cin, cout, 2, 2, 2)) / np.sqrt(8 * cin)).astype(np.float32)
    xf = _frame_of(x)
    yf = Frame(2, cout, *(2 * e for e in spatial))
    wdev = torch.from_numpy(w).cuda()
    W = torch.empty(_lib.load().vpx_deconv_workspace_bytes(cin, cout) // 4, device="cuda")
    _lib.call("vpx_deconv_fwd", xf.ptr, xf.desc, wdev.data_ptr(), yf.ptr, yf.desc, W.data_ptr(), W.numel() * 4,
              stream_ptr())
    assert rel(yf.to_ncdhw().cpu().numpy(), O.deconv3d(x, w)) < 1e-5
    u = rng.standard_normal((2, cout) + tuple(2 * e for e in spatial)).astype(np.float32)
    uf = _frame_of(u)
    gf = Frame(2, cin, *spatial, (1, 1, 1), zero=True)
    _lib.call("vpx_deconv_bwd_data", uf.ptr, uf.desc, wdev.data_ptr(), gf.ptr, gf.desc, W.data_ptr(), W.numel() * 4,
              stream_ptr())
    assert rel(gf.to_ncdhw().cpu().numpy(), O.deconv3d_bwd_data(u, w)) < 1e-5
    assert float(gf.t.abs().sum()) > 0 and gf.t[:, 0].abs().max().item() == 0.0  # margins untouched
    wg = torch.full_like(wdev, 0.5)
    _lib.call("vpx_deconv_bwd_filter", xf.ptr, xf.desc, uf.ptr, uf.desc, wg.data_ptr(), 1, W.data_ptr(),
              stream_ptr())
    assert rel(wg.cpu().numpy() - 0.5, O.deconv3d_bwd_filter(x, u)) < 1e-5


@pytest.mark.parametrize("ca,cb", [(8, 8), (16, 16), (3, 5)])
def test_concat_split_exact(ca, cb, fp32_mode):
    rng = np.random.default_rng(5)
    a = rng.standard_normal((2, ca, 3, 4, 20)).astype(np.float32)
    b = rng.standard_normal((2, cb, 3, 4, 20)).astype(np.float32)
    af, bf = _frame_of(a), _frame_of(b)
    yf = Frame(2, ca + cb, 3, 4, 20, (1, 1, 1), zero=True)
    _lib.call("vpx_concat", af.ptr, af.desc, bf.ptr, bf.desc, yf.ptr, yf.desc, stream_ptr())
    assert np.array_equal(yf.to_ncdhw().cpu().numpy(), np.concatenate([a, b], axis=1))
    u = rng.standard_normal((2, ca + cb, 3, 4, 20)).astype(np.float32)
    uf = _frame_of(u)
    ga = Frame(2, ca, 3, 4, 20)
    gb = _frame_of(b)
    _lib.call("vpx_split", uf.ptr, uf.desc, ga.ptr, ga.desc, gb.ptr, gb.desc, 1, stream_ptr())
    assert np.array_equal(ga.to_ncdhw().cpu().numpy(), u[:, :ca])
    assert np.array_equal(gb.to_ncdhw().cpu().numpy(), b + u[:, ca:])


def test_first_layer_one_channel_fused_leaky_margins():
    """1 -> 8 channel 3x3x3 conv with fused LeakyReLU reading halo margins
    (conv_small.cu), bit-identical to the generic direct kernel."""
    rng = np.random.default_rng(8)
    n, d, h, w = 1, 3, 5, 70
    full = rng.uniform(-1, 1, (n, 1, d + 2, h + 2, w + 2)).astype(np.float32)
    wt = (rng.uniform(-1, 1, (8, 1, 3, 3, 3)) / 5).astype(np.float32)
    xf = Frame(n, 1, d, h, w, (1, 1, 1), zero=True)
    xf.t.copy_(torch.from_numpy(full.transpose(0, 2, 3, 4, 1).copy()).cuda())
    wdev = torch.from_numpy(wt).cuda()
    outs = []
    for env in ("", "1"):
        os.environ["VPX_NO_SMALL"] = env
        if not env:
            del os.environ["VPX_NO_SMALL"]
        yf = Frame(n, 8, d, h, w)
        W = ws(1, 8, 3, yf)
        _lib.call("vpx_conv3d_fwd_act", xf.ptr, xf.desc, wdev.data_ptr(), 3, 1, yf.ptr, yf.desc, 1, 0.3,
                  W.data_ptr(), W.numel() * 4, stream_ptr())
        outs.append(yf.to_ncdhw().cpu().numpy())
    os.environ.pop("VPX_NO_SMALL", None)
    y_ref = O.leaky(O.k_conv3d_fwd(full, wt, (1, 1, 1)), 0.3)
    assert rel(outs[0], y_ref) < TF32_RTOL
    assert np.array_equal(outs[0].view(np.uint32), outs[1].view(np.uint32))


@pytest.mark.parametrize("ch,w", [(8, 256), (16, 128)])
def test_grouped_wgrad_reads_x_margins(ch, w):
    """Filter gradient with an input frame carrying D/H halo margins (as in a
    D/H-partitioned layer): the grouped-voxel kernel must read the margin rows."""
    rng = np.random.default_rng(4)
    n, d, h = 1, 3, 4
    full = rng.uniform(-1, 1, (n, ch, d + 2, h + 2, w)).astype(np.float32)
    xf = Frame(n, ch, d, h, w, (1, 1, 0), zero=True)
    xf.t.copy_(torch.from_numpy(full.transpose(0, 2, 3, 4, 1).copy()).cuda())
    u = rng.uniform(-1, 1, (n, ch, d, h, w)).astype(np.float32)
    uf = Frame(n, ch, d, h, w).load_ncdhw(u)
    W = ws(ch, ch, 3, uf)
    wg = torch.zeros((ch, ch, 3, 3, 3), device="cuda")
    _lib.call("vpx_conv3d_bwd_filter", xf.ptr, xf.desc, uf.ptr, uf.desc, 3, 1, wg.data_ptr(), 0, W.data_ptr(),
              W.numel() * 4, stream_ptr())
    xpad = np.pad(full, ((0, 0), (0, 0), (0, 0), (0, 0), (1, 1)))
    ref = O.k_conv3d_bwd_filter(xpad, u, (1, 1, 1), (3, 3, 3))
    assert rel(wg.cpu().numpy(), ref) < TF32_RTOL


def test_filter_gradient_channel_slices_equal_concat():
    """wgrad of a conv over a channel concat == the two slice gradients from the
    concat's sources (vpx_conv3d_bwd_filter_cslice)."""
    rng = np.random.default_rng(9)
    n, d, h, w = 1, 3, 4, 128
    a = rng.uniform(-1, 1, (n, 8, d, h, w)).astype(np.float32)
    b = rng.uniform(-1, 1, (n, 8, d, h, w)).astype(np.float32)
    u = rng.uniform(-1, 1, (n, 8, d, h, w)).astype(np.float32)
    af, bf, uf = _frame_of(a), _frame_of(b), _frame_of(u)
    cf = _frame_of(np.concatenate([a, b], axis=1))
    W = ws(16, 8, 3, uf)
    full = torch.zeros((8, 16, 3, 3, 3), device="cuda")
    _lib.call("vpx_conv3d_bwd_filter", cf.ptr, cf.desc, uf.ptr, uf.desc, 3, 1, full.data_ptr(), 0, W.data_ptr(),
              W.numel() * 4, stream_ptr())
    sl = torch.full((8, 16, 3, 3, 3), 7.0, device="cuda")
    for ci0, f in ((0, af), (8, bf)):
        _lib.call("vpx_conv3d_bwd_filter_cslice", f.ptr, f.desc, uf.ptr, uf.desc, 3, 1, sl.data_ptr(), ci0, 16, 0,
                  W.data_ptr(), W.numel() * 4, stream_ptr())
    ref = O.conv3d_bwd_filter(np.concatenate([a, b], axis=1), u, (3, 3, 3), (1, 1, 1))
    assert rel(full.cpu().numpy(), ref) < TF32_RTOL
    assert rel(sl.cpu().numpy(), ref) < TF32_RTOL


@pytest.mark.parametrize("cin,cout,shape,margins", [(16, 32, (1, 4, 6, 256), (0, 0, 0)),
                                                    (16, 32, (2, 2, 20, 128), (1, 1, 0)),
                                                    (16, 16, (1, 4, 4, 128), (1, 0, 0))])
def test_fused_conv_leaky_pool_bit_exact(cin, cout, shape, margins):
    """conv -> LeakyReLU -> avg pool in one kernel (conv_rowh.cu pooled variant)
    against the unfused conv(+leaky) and pool kernels: the fused kernel pools
    the unrounded activations in a tree order, so the pooled values agree to
    within one TF32 step (2^-10 of the maximum); the sign mask ==
    (activation >= 0) bit for bit (same convolution); the mask backward == the
    activation backward bit for bit."""
    n, d, h, w = shape
    rng = np.random.default_rng(12)
    md, mh, mw = margins
    full = rng.uniform(-1, 1, (n, cin, d + 2 * md, h + 2 * mh, w)).astype(np.float32)
    xf = Frame(n, cin, d, h, w, margins, zero=True)
    xf.t.copy_(torch.from_numpy(full.transpose(0, 2, 3, 4, 1).copy()).cuda())
    wt = torch.from_numpy((rng.uniform(-1, 1, (cout, cin, 3, 3, 3)) / 12).astype(np.float32)).cuda()
    slope = 0.3
    yf = Frame(n, cout, d, h, w)
    W = ws(cin, cout, 3, yf)
    _lib.call("vpx_conv3d_fwd_act", xf.ptr, xf.desc, wt.data_ptr(), 3, 1, yf.ptr, yf.desc, 1, slope, W.data_ptr(),
              W.numel() * 4, stream_ptr())
    pref = Frame(n, cout, d // 2, h // 2, w // 2)
    _lib.call("vpx_pool_fwd", yf.ptr, yf.desc, pref.ptr, pref.desc, 0, stream_ptr())
    pf = Frame(n, cout, d // 2, h // 2, w // 2)
    dt = {16: torch.int16, 32: torch.int32}[cout]
    mask = torch.zeros((n, d, h, w), dtype=dt, device="cuda")
    _lib.call("vpx_conv3d_fwd_leaky_pool", xf.ptr, xf.desc, wt.data_ptr(), slope, pf.ptr, pf.desc,
              mask.data_ptr(), W.data_ptr(), W.numel() * 4, stream_ptr())
    torch.cuda.synchronize()
    assert float((pf.t - pref.t).abs().max()) <= 2.0 ** -10 * float(pref.t.abs().max())
    y = yf.t  # (n, d, h, w, c)
    bits = (y >= 0).to(torch.int64) << torch.arange(cout, device="cuda")
    want = bits.sum(-1)
    got = mask.to(torch.int64) & ((1 << cout) - 1)
    assert torch.equal(got, want)
    up = rng.uniform(-1, 1, (n, cout, d // 2, h // 2, w // 2)).astype(np.float32)
    uf = Frame(n, cout, d // 2, h // 2, w // 2).load_ncdhw(up)
    g1 = Frame(n, cout, d, h, w, (md, mh, 0), zero=True)
    g2 = Frame(n, cout, d, h, w, (md, mh, 0), zero=True)
    _lib.call("vpx_pool_leaky_bwd", yf.ptr, yf.desc, uf.ptr, uf.desc, g1.ptr, g1.desc, slope, 0, stream_ptr())
    mdesc = frame_desc(n, cout, d, h, w)
    _lib.call("vpx_pool_leaky_bwd_mask", mask.data_ptr(), ctypes.addressof(mdesc), uf.ptr, uf.desc, g2.ptr, g2.desc,
              slope, stream_ptr())
    torch.cuda.synchronize()
    assert torch.equal(g1.t.view(torch.int32), g2.t.view(torch.int32))


@pytest.mark.parametrize("margins,precision", [((0, 0, 0), "tf32"), ((1, 1, 0), "tf32"), ((0, 0, 0), "fp32")])
def test_bn_apply_leaky_equals_bn_then_leaky(margins, precision):
    """vpx_bn_apply_leaky (one pass) == vpx_bn_apply then vpx_leaky_fwd, bit
    for bit, on flat and margin frames, with and without TF32 storage
    rounding (reference layers/reference.py:209-214, :231-233)."""
    rng = np.random.default_rng(11)
    n, c, d, h, w = 2, 8, 4, 6, 8
    x = rng.standard_normal((n, c, d, h, w)).astype(np.float32)
    xf = Frame(n, c, d, h, w, margins, zero=True).load_ncdhw(x)
    mean = torch.from_numpy(rng.standard_normal(c).astype(np.float32)).cuda()
    inv = torch.from_numpy(rng.uniform(0.5, 2, c).astype(np.float32)).cuda()
    gamma = torch.from_numpy(rng.uniform(-1, 1, c).astype(np.float32)).cuda()
    beta = torch.from_numpy(rng.uniform(-1, 1, c).astype(np.float32)).cuda()
    mid, ref, got = (Frame(n, c, d, h, w, margins, zero=True) for _ in range(3))
    import paper_2007_12856_b200 as pkg

    pkg.set_precision(precision)  # TF32 mode rounds every stored value to TF32
    try:
        _call_bn_pair(xf, mean, inv, gamma, beta, mid, ref, got)
    finally:
        pkg.set_precision("tf32")
    assert torch.equal(got.t, ref.t)


def _call_bn_pair(xf, mean, inv, gamma, beta, mid, ref, got):
    _lib.call("vpx_bn_apply", xf.ptr, xf.desc, mean.data_ptr(), inv.data_ptr(), gamma.data_ptr(), beta.data_ptr(),
              mid.ptr, mid.desc, stream_ptr())
    _lib.call("vpx_leaky_fwd", mid.ptr, mid.desc, ref.ptr, ref.desc, 0.3, stream_ptr())
    _lib.call("vpx_bn_apply_leaky", xf.ptr, xf.desc, mean.data_ptr(), inv.data_ptr(), gamma.data_ptr(),
              beta.data_ptr(), 0.3, got.ptr, got.desc, stream_ptr())
    torch.cuda.synchronize()


def test_xent_two_class_fast_path_equals_generic():
    """The vectorised two-class cross entropy (margin-free frames) gives the
    generic kernel's gradients bit for bit and its loss to double rounding,
    and both match a numpy log-softmax (reference layers/distributed.py:273-293)."""
    rng = np.random.default_rng(3)
    n, d, h, w = 1, 4, 6, 8
    logits = (rng.standard_normal((n, 2, d, h, w)) * 3).astype(np.float32)
    labels = torch.from_numpy(rng.integers(0, 2, (n, d, h, w))).cuda()
    count = n * d * h * w
    out = []
    for margins in ((0, 0, 0), (1, 1, 0)):  # flat: fast path; margins: generic kernel
        lf = Frame(n, 2, d, h, w, margins, zero=True).load_ncdhw(logits)
        gf = Frame(n, 2, d, h, w, margins, zero=True)
        part = torch.zeros(64, dtype=torch.float64, device="cuda")
        _lib.call("vpx_xent", lf.ptr, lf.desc, labels.data_ptr(), float(count), gf.ptr, gf.desc, part.data_ptr(),
                  64, stream_ptr())
        torch.cuda.synchronize()
        out.append((float(part.sum()) / count, gf.to_ncdhw().cpu().numpy()))
    assert np.array_equal(out[0][1].view(np.uint32), out[1][1].view(np.uint32))
    assert abs(out[0][0] - out[1][0]) <= 1e-12 * abs(out[1][0])
    lab = labels.cpu().numpy()
    lp = logits.astype(np.float64)
    lse = np.log(np.exp(lp).sum(1))
    ref = -(np.take_along_axis(lp, lab[:, None], 1)[:, 0] - lse).mean()
    assert abs(out[0][0] - ref) < 1e-5 * abs(ref)


@pytest.mark.parametrize("margins", [(0, 0, 0), (1, 1, 0)])
def test_int8_transfer_layout_equals_int16(margins):
    """vpx_layout_ncdhw_i8_to_frame (the datastore's int8 transfer copy) gives
    the same fp32 frame, bit for bit, as the int16 storage path."""
    rng = np.random.default_rng(7)
    v16 = rng.integers(-8, 9, (1, 4, 4, 6, 8)).astype(np.int16)
    a = Frame(1, 4, 4, 6, 8, margins, zero=True).load_ncdhw(v16)
    b = Frame(1, 4, 4, 6, 8, margins, zero=True).load_ncdhw(v16.astype(np.int8))
    torch.cuda.synchronize()
    assert torch.equal(a.t.view(torch.int32), b.t.view(torch.int32))
    assert np.array_equal(b.to_ncdhw().cpu().numpy(), v16.astype(np.float32))


@pytest.mark.parametrize("dtype", [np.int8, np.int16, np.float32])
@pytest.mark.parametrize("c,spatial,margins,offset", [(4, (3, 5, 16), (1, 1, 0), 0), (8, (2, 3, 12), (0, 1, 0), 0),
                                                      (3, (2, 3, 8), (1, 0, 0), 0), (4, (2, 2, 6), (0, 0, 0), 0),
                                                      (4, (2, 3, 8), (1, 1, 0), 1), (4, (1, 2, 520), (0, 0, 0), 0),
                                                      (4, (2, 1, 36), (1, 0, 0), 0), (1, (2, 3, 8), (1, 1, 0), 0),
                                                      (1, (2, 2, 12), (0, 0, 0), 1), (1, (2, 2, 10), (0, 0, 0), 0)])
def test_ncdhw_layout_kernels_exact(dtype, c, spatial, margins, offset):
    """NCDHW -> NDHWC frame layout kernels (C = 4 shuffle-coalesced, C % 4 == 0
    vector and C = 1 convert paths when W is a multiple of 4 and the source is
    aligned, scalar path otherwise): exact values in the interior, margins
    untouched (zero)."""
    rng = np.random.default_rng(3)
    n = 2
    shape = (n, c) + spatial
    if dtype == np.float32:
        v = rng.standard_normal(shape).astype(np.float32)
    else:
        v = rng.integers(-100, 101, shape).astype(dtype)
    src = torch.from_numpy(v.ravel()).cuda()
    if offset:  # a source not 16-byte aligned takes the scalar path
        buf = torch.zeros(src.numel() + offset, dtype=src.dtype, device="cuda")
        buf[offset:] = src
        src = buf[offset:]
    f = Frame(n, c, *spatial, margins, zero=True).load_ncdhw(src.view(shape))
    torch.cuda.synchronize()
    want = v.astype(np.float32)
    if dtype == np.float32 and get_precision() == "tf32":
        want = O.tf32_round(v)  # frames store values rounded to nearest TF32 in that mode
    assert np.array_equal(f.to_ncdhw().cpu().numpy(), want)
    t = f.t.cpu().numpy()
    md, mh, mw = f.m
    inner = t[:, md:md + spatial[0], mh:mh + spatial[1], mw:mw + spatial[2]]
    assert np.abs(t).sum() == np.abs(inner).sum()


@pytest.mark.parametrize("cin,cout,spatial,margins", [(32, 16, (4, 6, 64), (0, 0, 0)), (16, 8, (3, 4, 40), (0, 0, 0)),
                                                     (32, 16, (2, 8, 16), (1, 1, 0)), (16, 8, (4, 2, 24), (1, 0, 0)),
                                                     (16, 8, (2, 3, 128), (0, 0, 0)), (32, 16, (3, 2, 32), (1, 1, 0))])
def test_deconv_tensor_cores_vs_tf32_oracle(cin, cout, spatial, margins):
    """TF32 mode: the k2s2 transposed conv forward and backward-data run as
    tcgen05 implicit GEMMs (tap-box kernel, kind 1): rtol 1e-3 against the
    TF32-emulating oracle (operands rounded to nearest TF32, fp64
    accumulation), no CUDA-core fallback, output margins untouched by the
    forward, D/H input margins read correctly.  Reference: reference.py:99-131."""
    R = O.tf32_round
    rng = np.random.default_rng(12)
    x = R(rng.standard_normal((2, cin) + spatial).astype(np.float32))
    w = (rng.standard_normal((cin, cout, 2, 2, 2)) / np.sqrt(8 * cin)).astype(np.float32)
    xf = Frame(2, cin, *spatial, margins, zero=True).load_ncdhw(x)
    fine = tuple(2 * e for e in spatial)
    yf = Frame(2, cout, *fine, margins, zero=True)
    wdev = torch.from_numpy(w).cuda()
    W = torch.empty(_lib.load().vpx_deconv_workspace_bytes(cin, cout) // 4, device="cuda")
    fb0 = _lib.load().vpx_fallback_count()
    _lib.call("vpx_deconv_fwd", xf.ptr, xf.desc, wdev.data_ptr(), yf.ptr, yf.desc, W.data_ptr(), W.numel() * 4,
              stream_ptr())
    y_ref = R(O.deconv3d(x.astype(np.float64), R(w).astype(np.float64)).astype(np.float32))
    assert rel(yf.to_ncdhw().cpu().numpy(), y_ref) < 1e-3
    if any(margins):
        inner = yf.interior.clone()
        yf.interior.zero_()
        assert float(yf.t.abs().max()) == 0.0, "forward wrote into the output margins"
        yf.interior.copy_(inner)
    u = R(rng.standard_normal((2, cout) + fine).astype(np.float32))
    uf = Frame(2, cout, *fine).load_ncdhw(u)
    gf = Frame(2, cin, *spatial, margins, zero=True)
    _lib.call("vpx_deconv_bwd_data", uf.ptr, uf.desc, wdev.data_ptr(), gf.ptr, gf.desc, W.data_ptr(), W.numel() * 4,
              stream_ptr())
    g_ref = R(O.deconv3d_bwd_data(u.astype(np.float64), R(w).astype(np.float64)).astype(np.float32))
    assert rel(gf.to_ncdhw().cpu().numpy(), g_ref) < 1e-3
    assert _lib.load().vpx_fallback_count() == fb0, "deconv fell back to the CUDA-core kernels"
    if spatial[2] % 32 == 0:  # filter gradient on tcgen05 (deconv_wgrad.cu): 32-voxel W segments
        wg = torch.full_like(wdev, 0.25)
        _lib.call("vpx_deconv_bwd_filter", xf.ptr, xf.desc, uf.ptr, uf.desc, wg.data_ptr(), 1, W.data_ptr(),
                  stream_ptr())
        wg_ref = O.deconv3d_bwd_filter(x.astype(np.float64), u.astype(np.float64)).astype(np.float32)
        assert rel(wg.cpu().numpy() - 0.25, wg_ref) < 1e-3
        assert _lib.load().vpx_fallback_count() == fb0, "deconv filter gradient fell back to CUDA cores"


@pytest.mark.parametrize("margins", [(1, 0, 0), (1, 1, 0)])
def test_concat_wgrad_slices_from_partitioned_frame(margins):
    """Spatially partitioned U-Net u1c1: the concat frame carries exchanged D/H
    halo margins the concat sources do not have, so layers.concat_wgrad_sources
    takes each source's channel range from the concat frame itself (dense copy,
    margins included) -- the filter gradient must match the oracle over the
    whole haloed frame and the whole-concat kernel."""
    from paper_2007_12856_b200 import layers as D

    rng = np.random.default_rng(19)
    n, d, h, w = 1, 3, 4, 128
    md, mh, mw = margins
    full = rng.uniform(-1, 1, (n, 16, d + 2 * md, h + 2 * mh, w)).astype(np.float32)
    cf = Frame(n, 16, d, h, w, margins, zero=True)
    cf.t.copy_(torch.from_numpy(full.transpose(0, 2, 3, 4, 1).copy()).cuda())
    u = rng.uniform(-1, 1, (n, 8, d, h, w)).astype(np.float32)
    uf = _frame_of(u)
    srcs = [Frame(n, 8, d, h, w), Frame(n, 8, d, h, w)]  # stand-ins: channel counts only (no margins)
    params = type("P", (), {"kernel": (3, 3, 3), "stride": (1, 1, 1), "cin": 16, "cout": 8})()
    slices = D.concat_wgrad_sources(cf, srcs, uf, params)
    assert slices is not None and [c0 for c0, _ in slices] == [0, 8]
    W = ws(16, 8, 3, uf)
    whole = torch.zeros((8, 16, 3, 3, 3), device="cuda")
    _lib.call("vpx_conv3d_bwd_filter", cf.ptr, cf.desc, uf.ptr, uf.desc, 3, 1, whole.data_ptr(), 0, W.data_ptr(),
              W.numel() * 4, stream_ptr())
    sl = torch.full((8, 16, 3, 3, 3), 7.0, device="cuda")
    D.dist_conv3d_bwd_filter_slices(None, slices, uf, params, sl)
    xpad = np.pad(full, ((0, 0), (0, 0), (0 if md else 1,) * 2, (0 if mh else 1,) * 2, (1, 1)))
    ref = O.k_conv3d_bwd_filter(xpad, u, (1, 1, 1), (3, 3, 3))
    assert rel(sl.cpu().numpy(), ref) < TF32_RTOL
    assert rel(sl.cpu().numpy(), whole.cpu().numpy()) < 1e-5  # same TF32 products, other summation order
