"""Out-of-bounds and uninitialised-read checks of our own (GPU).

compute-sanitizer is closed on this GPU pool (runs under it left GPUs needing
a reset), so the kernels get the sanitizer's two main checks by construction:

* every buffer a kernel touches -- input and output frames, weights,
  workspace -- sits inside a larger allocation whose guard bands hold a
  signalling-NaN bit pattern; after the kernel the guard bands must be
  bit-identical (no out-of-bounds write), and every output must be finite
  (an out-of-bounds or never-written read would pull in the NaN pattern);
* outputs are pre-filled with the same NaN pattern, so a kernel that leaves
  part of its output unwritten fails the finiteness check (initcheck).

Shapes: every conv CASE of test_gpu_kernels (each tcgen05 kernel family and
the CUDA-core paths), frames with halo margins in D/H/W, the fused first-block
kernels, pooling/LeakyReLU/BN/halo/layout kernels.
"""

import ctypes

import numpy as np
import pytest
import torch

from paper_2007_12856_b200 import _lib
from paper_2007_12856_b200.frames import Frame, frame_desc, stream_ptr
from test_gpu_kernels import CASES

pytestmark = pytest.mark.gpu

GUARD = 1 << 16                # floats on each side
SENTINEL = 0x7FBADBAD          # a NaN bit pattern


class Guarded:
    """A float32 buffer of `numel` elements inside NaN guard bands."""

    def __init__(self, numel, fill=None):
        self.buf = torch.empty(numel + 2 * GUARD, dtype=torch.float32, device="cuda")
        self.buf.view(torch.int32).fill_(SENTINEL)
        self.t = self.buf[GUARD:GUARD + numel]
        if fill is not None:
            self.t.copy_(fill.reshape(-1))

    def guards_intact(self):
        g = torch.cat([self.buf[:GUARD], self.buf[-GUARD:]]).view(torch.int32)
        return bool((g == SENTINEL).all())


def gframe(n, c, d, h, w, margins=(0, 0, 0), data=None, zero_margins=True):
    """Frame whose storage is a Guarded buffer: interior = data (NCDHW) or the
    NaN pattern (output frames), margins zero (or NaN when zero_margins=False)."""
    md, mh, mw = margins
    shape = (n, d + 2 * md, h + 2 * mh, w + 2 * mw, c)
    g = Guarded(int(np.prod(shape)))
    fr = Frame(n, c, d, h, w, margins, tensor=g.t.view(shape))
    if data is not None:
        if zero_margins:
            fr.t.zero_()
        fr.load_ncdhw(data)
    return fr, g


def ws_guarded(cin, cout, k, fr):
    nb = _lib.load().vpx_conv3d_workspace_bytes(cin, cout, k, fr.desc)
    g = Guarded(nb // 4 + 64)
    return g


def finite(fr, full=False):
    t = fr.t if full else fr.interior
    return bool(torch.isfinite(t).all())


@pytest.mark.parametrize("case", CASES)
@pytest.mark.parametrize("margins", [(0, 0, 0), (1, 1, 0)])
def test_conv_passes_stay_in_bounds(case, margins):
    n, cin, cout, d, h, w, k, s = case
    if k == 1 or cin == 1:
        margins = (0, 0, 0)  # the pointwise / 1-channel kernels take margin-free frames
    if s == 2 and any(e % 2 for e in (d, h, w)):
        pytest.skip("odd extent")
    rng = np.random.default_rng(1)
    x = rng.uniform(-1, 1, (n, cin, d, h, w)).astype(np.float32)
    xf, gx = gframe(n, cin, d, h, w, margins, x)
    if any(margins):  # neighbour data in the margins, as after a halo exchange
        fill = torch.from_numpy(rng.uniform(-1, 1, tuple(xf.t.shape)).astype(np.float32)).cuda()
        inner = xf.interior.clone()
        xf.t.copy_(fill)
        xf.interior.copy_(inner)
    wt = Guarded(cout * cin * k ** 3, torch.from_numpy(
        (rng.uniform(-1, 1, (cout, cin, k, k, k)) / np.sqrt(cin * k ** 3)).astype(np.float32)).cuda())
    od, oh, ow = (-(-e // s) for e in (d, h, w))
    yf, gy = gframe(n, cout, od, oh, ow)
    W = ws_guarded(cin, cout, k, yf)
    _lib.call("vpx_conv3d_fwd", xf.ptr, xf.desc, wt.t.data_ptr(), k, s, yf.ptr, yf.desc, W.t.data_ptr(),
              W.t.numel() * 4, stream_ptr())
    torch.cuda.synchronize()
    assert gy.guards_intact() and gx.guards_intact() and W.guards_intact() and wt.guards_intact()
    assert finite(yf, full=True), "conv fwd left output unwritten or read out of bounds"
    u = rng.uniform(-1, 1, (n, cout, od, oh, ow)).astype(np.float32)
    uf, gu = gframe(n, cout, od, oh, ow, data=u)
    gf, gg = gframe(n, cin, d, h, w, margins)  # NaN everywhere, margins included
    W2 = ws_guarded(cin, cout, k, uf)
    _lib.call("vpx_conv3d_bwd_data", uf.ptr, uf.desc, wt.t.data_ptr(), k, s, gf.ptr, gf.desc, W2.t.data_ptr(),
              W2.t.numel() * 4, stream_ptr())
    torch.cuda.synchronize()
    assert gg.guards_intact() and gu.guards_intact() and W2.guards_intact()
    assert finite(gf, full=True), "conv dgrad left part of the gradient frame (margins included) unwritten"
    wg = Guarded(cout * cin * k ** 3)
    W3 = ws_guarded(cin, cout, k, uf)
    _lib.call("vpx_conv3d_bwd_filter", xf.ptr, xf.desc, uf.ptr, uf.desc, k, s, wg.t.data_ptr(), 0, W3.t.data_ptr(),
              W3.t.numel() * 4, stream_ptr())
    torch.cuda.synchronize()
    assert wg.guards_intact() and W3.guards_intact() and gx.guards_intact()
    assert bool(torch.isfinite(wg.t).all()), "conv wgrad left filter-gradient entries unwritten"


@pytest.mark.parametrize("shape,margins", [((1, 4, 6, 128), (0, 0, 0)), ((2, 2, 4, 256), (1, 1, 0)),
                                           ((1, 2, 4, 512), (1, 0, 0))])
def test_first_block_kernels_stay_in_bounds(shape, margins):
    n, d, h, w = shape
    rng = np.random.default_rng(2)
    x = rng.uniform(-1, 1, (n, 4, d, h, w)).astype(np.float32)
    xf, gx = gframe(n, 4, d, h, w, margins, x)
    wt = Guarded(16 * 4 * 27, torch.from_numpy((rng.uniform(-1, 1, (16, 4, 3, 3, 3)) / 5).astype(np.float32)).cuda())
    pf, gp = gframe(n, 16, d // 2, h // 2, w // 2, margins)
    pf.t.zero_()
    mask = torch.full((n * d * h * w + 2 * GUARD,), -21555, dtype=torch.int16, device="cuda")
    W = ws_guarded(4, 16, 3, Frame(n, 16, d, h, w))
    _lib.call("vpx_conv3d_fwd_leaky_pool_c4", xf.ptr, xf.desc, wt.t.data_ptr(), 0.3, pf.ptr, pf.desc,
              mask[GUARD:].data_ptr(), W.t.data_ptr(), W.t.numel() * 4, stream_ptr())
    torch.cuda.synchronize()
    assert gp.guards_intact() and W.guards_intact() and gx.guards_intact()
    assert bool((mask[:GUARD] == -21555).all()) and bool((mask[-GUARD:] == -21555).all())
    assert finite(pf)
    up = rng.uniform(-1, 1, (n, 16, d // 2, h // 2, w // 2)).astype(np.float32)
    upf, gu = gframe(n, 16, d // 2, h // 2, w // 2, margins, up)
    wg = Guarded(16 * 4 * 27)
    mfr = frame_desc(n, 16, d, h, w)
    W2 = ws_guarded(4, 16, 3, Frame(n, 16, d, h, w))
    _lib.call("vpx_conv3d_bwd_filter_c4_pooled_mask", xf.ptr, xf.desc, mask[GUARD:].data_ptr(),
              ctypes.addressof(mfr), upf.ptr, upf.desc, 0.3, wg.t.data_ptr(), 0, W2.t.data_ptr(),
              W2.t.numel() * 4, stream_ptr())
    torch.cuda.synchronize()
    assert wg.guards_intact() and W2.guards_intact() and gu.guards_intact()
    assert bool(torch.isfinite(wg.t).all())


@pytest.mark.parametrize("c,spatial,margins", [(16, (4, 6, 8), (0, 0, 0)), (32, (4, 4, 16), (1, 1, 0)),
                                               (8, (2, 8, 4), (1, 1, 1))])
def test_pointwise_kernels_stay_in_bounds(c, spatial, margins):
    d, h, w = spatial
    rng = np.random.default_rng(3)
    x = rng.uniform(-1, 1, (2, c, d, h, w)).astype(np.float32)
    xf, gx = gframe(2, c, d, h, w, (0, 0, 0), x)
    # leaky fwd/bwd
    yf, gy = gframe(2, c, d, h, w, margins)
    _lib.call("vpx_leaky_fwd", xf.ptr, xf.desc, yf.ptr, yf.desc, 0.3, stream_ptr())
    uf, gu = gframe(2, c, d, h, w, (0, 0, 0), x[:, :, ::-1].copy())
    lg, glg = gframe(2, c, d, h, w, (0, 0, 0))
    _lib.call("vpx_leaky_bwd", xf.ptr, xf.desc, uf.ptr, uf.desc, lg.ptr, lg.desc, 0.3, stream_ptr())
    # pool fwd/bwd (avg, max)
    for is_max in (0, 1):
        pf, gp = gframe(2, c, d // 2, h // 2, w // 2, margins)
        _lib.call("vpx_pool_fwd", xf.ptr, xf.desc, pf.ptr, pf.desc, is_max, stream_ptr())
        pu, gpu = gframe(2, c, d // 2, h // 2, w // 2, (0, 0, 0), x[:, :, ::2, ::2, ::2].copy())
        pg, gpg = gframe(2, c, d, h, w, (0, 0, 0))
        _lib.call("vpx_pool_bwd", xf.ptr, xf.desc, pu.ptr, pu.desc, pg.ptr, pg.desc, is_max, stream_ptr())
        pl, gpl = gframe(2, c, d, h, w, (0, 0, 0))
        _lib.call("vpx_pool_leaky_bwd", xf.ptr, xf.desc, pu.ptr, pu.desc, pl.ptr, pl.desc, 0.3, is_max, stream_ptr())
        torch.cuda.synchronize()
        for g in (gp, gpu, gpg, gpl):
            assert g.guards_intact()
        assert finite(pf) and finite(pg) and finite(pl)
    torch.cuda.synchronize()
    for g in (gx, gy, gu, glg):
        assert g.guards_intact()
    assert finite(yf) and finite(lg)
    # layout round trip through a guarded NCDHW buffer
    dst = Guarded(x.size)
    _lib.call("vpx_layout_frame_to_ncdhw", yf.ptr, yf.desc, dst.t.data_ptr(), stream_ptr())
    torch.cuda.synchronize()
    assert dst.guards_intact() and bool(torch.isfinite(dst.t).all())


@pytest.mark.parametrize("cin,cout,spatial,margins", [(32, 16, (2, 4, 64), (0, 0, 0)), (16, 8, (3, 2, 32), (1, 1, 0)),
                                                     (16, 8, (2, 2, 40), (0, 0, 0))])
def test_deconv_kernels_stay_in_bounds(cin, cout, spatial, margins):
    """k2s2 transposed conv (tcgen05 tap-box kind 1 + deconv_wgrad.cu, or the
    CUDA-core kernels where W is not a multiple of the 32-voxel segment)."""
    rng = np.random.default_rng(4)
    x = rng.uniform(-1, 1, (2, cin) + spatial).astype(np.float32)
    fine = tuple(2 * e for e in spatial)
    xf, gx = gframe(2, cin, *spatial, margins, x)
    wt = Guarded(cin * cout * 8, torch.from_numpy((rng.uniform(-1, 1, (cin, cout, 2, 2, 2)) / 8).astype(np.float32)).cuda())
    yf, gy = gframe(2, cout, *fine, margins)
    yf.t.zero_()
    W = Guarded(_lib.load().vpx_deconv_workspace_bytes(cin, cout) // 4 + 64)
    _lib.call("vpx_deconv_fwd", xf.ptr, xf.desc, wt.t.data_ptr(), yf.ptr, yf.desc, W.t.data_ptr(), W.t.numel() * 4,
              stream_ptr())
    u = rng.uniform(-1, 1, (2, cout) + fine).astype(np.float32)
    uf, gu = gframe(2, cout, *fine, (0, 0, 0), u)
    gf, gg = gframe(2, cin, *spatial, margins)
    gf.t.zero_()
    _lib.call("vpx_deconv_bwd_data", uf.ptr, uf.desc, wt.t.data_ptr(), gf.ptr, gf.desc, W.t.data_ptr(),
              W.t.numel() * 4, stream_ptr())
    wg = Guarded(cin * cout * 8)
    _lib.call("vpx_deconv_bwd_filter", xf.ptr, xf.desc, uf.ptr, uf.desc, wg.t.data_ptr(), 0, W.t.data_ptr(),
              stream_ptr())
    torch.cuda.synchronize()
    for g in (gx, wt, gy, W, gu, gg, wg):
        assert g.guards_intact()
    assert finite(yf) and finite(gf) and bool(torch.isfinite(wg.t).all())
