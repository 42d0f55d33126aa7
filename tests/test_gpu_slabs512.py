"""Per-layer slab parity at the CosmoFlow-512 shapes the bench runs (GPU).

Every conv block of CosmoFlow 512^3 (c1..c7: channels, strides, and the full
H x W extents of the 512^3 step) is run through the SAME layer functions the
engine calls in the timed step (layers.first_block_fwd / dist_conv3d with the
fused LeakyReLU / dist_pool3d forward, dist_pool_leaky_bwd or
first_block_wgrad / dist_conv3d_bwd_filter / dist_conv3d_bwd_data backward),
so the same kernel instantiations launch (c1_fwd_pool_kernel at W=512,
c1_pooled_wgrad_kernel<512,1>, conv_rowh_pool_kernel<16,32> at W=256,
conv_rowh_kernel<32,16>, wgrad_ut_kernel<256>, conv_rowwin at W=128,
conv_tapbox / wgrad_kernel for c4..c7).  Only the depth is thinned to a slab
(c1..c3; c4..c7 run at their full 512^3-step extents), once without margins
(the 1-GPU step) and once with D halo margins filled with neighbour data (a
rank of the 1x8x1x1 split; the halo exchange itself is covered elsewhere).

Each output is checked against the TF32-emulating oracle evaluated on the
device's own inputs to that layer (teacher forcing) at the north-star rtol
1e-3 in the reference metric max|got-ref|/max|ref| (reference
cli.py:199-202); the conv semantics are reference _hot.pyx:19-93.
"""

import numpy as np
import pytest
import torch

from oracle import serial as O
from paper_2007_12856_b200 import _lib
from paper_2007_12856_b200 import layers as D
from paper_2007_12856_b200.comm import RankCtx
from paper_2007_12856_b200.frames import DistTensor
from paper_2007_12856_b200.geometry import ProcessGrid, Shape5D, make_partition
from paper_2007_12856_b200.layers import NO_HALO
from paper_2007_12856_b200.networks import build_cosmoflow

pytestmark = pytest.mark.gpu

R = O.tf32_round
RTOL = 1e-3
SLOPE = 0.3
# (block, cin, cout, stride, input extent at 512^3, slab depth of the input)
BLOCKS = [("c1", 4, 16, 1, 512, 4), ("c2", 16, 32, 1, 256, 4), ("c3", 32, 64, 1, 128, 4),
          ("c4", 64, 128, 2, 64, 8), ("c5", 128, 256, 1, 16, 16), ("c6", 256, 256, 1, 8, 8),
          ("c7", 256, 256, 1, 4, 4)]


def rel(got, ref):
    ref = np.asarray(ref, dtype=np.float64)
    return float(np.max(np.abs(np.asarray(got, np.float64) - ref)) / max(np.max(np.abs(ref)), 1e-30))


def _meta(c, d, h, w, split, radii):
    """Rank 0's tensor of a 1x2x1x1 depth split (margins md = radius) or of
    the whole slab (no margins)."""
    grid = ProcessGrid(1, 2 if split else 1, 1, 1)
    return make_partition(Shape5D(1, c, d * (2 if split else 1), h, w), grid, radii)


def _full(t: DistTensor):
    """Whole frame (margins included) as NCDHW numpy."""
    return t.t.permute(0, 4, 1, 2, 3).contiguous().cpu().numpy()


def _pad_hw(a, md):
    """Zero 'same' padding in the dims without margins (D has margins when md)."""
    return np.pad(a, ((0, 0), (0, 0), (0 if md else 1, 0 if md else 1), (1, 1), (1, 1)))


def _mask_bits(mask, c):
    b = mask.t.cpu().numpy().astype(np.int64) & ((1 << c) - 1)
    return np.stack([(b >> k) & 1 for k in range(c)], axis=1).astype(bool)  # (n, c, d, h, w)


@pytest.fixture
def no_halo(monkeypatch):
    """The slabs' margins are filled by the test; skip the (multi-rank) exchange."""
    monkeypatch.setattr(D, "halo_exchange", lambda ctx, x, *a, **k: None)
    monkeypatch.setattr(D, "reverse_halo_exchange", lambda *a, **k: None)


@pytest.mark.parametrize("split", [False, True], ids=["1gpu", "dsplit"])
@pytest.mark.parametrize("blk", BLOCKS, ids=[b[0] for b in BLOCKS])
def test_cosmoflow512_block_slab(blk, split, no_halo):
    name, cin, cout, s, ext, dslab = blk
    fb0 = _lib.load().vpx_fallback_count()
    if split and name in ("c6", "c7"):
        pytest.skip("8-way split redistributes before these blocks (engine.make_plan)")
    net = build_cosmoflow(512)
    conv = net.layers[net.layer_index(name)]
    assert (conv.params.cin, conv.params.cout, conv.params.stride[0]) == (cin, cout, s)
    rng = np.random.default_rng(int(name[1:]) * 10 + int(split))
    ctx = RankCtx(0, 1)
    md = 1 if split else 0
    d_in, od = dslab, dslab // s
    xm = _meta(cin, d_in, ext, ext, split, (1, 1, 1))
    x = DistTensor(xm, 0, zero=True)
    assert x.m == (md, 0, 0)
    # TF32 data everywhere in the frame (interior and, when split, both D margins)
    x.t.copy_(torch.from_numpy(R(rng.uniform(-1, 1, tuple(x.t.shape)).astype(np.float32))).cuda())
    w = rng.uniform(-1, 1, (cout, cin, 3, 3, 3)).astype(np.float32) * np.float32(np.sqrt(3.0 / (27 * cin)))
    wd = torch.from_numpy(w).cuda()
    xfull = _full(x)
    xpad = _pad_hw(xfull, md)
    # -------------------------------------------------------- forward
    pre = O._f64(O.k_conv3d_fwd, xpad, R(w), (s, s, s))  # fp32 conv, not yet rounded
    act_ref = R(O.leaky(pre, SLOPE))                     # stored activation (rounded once, fused epilogue)
    fused = (D.first_block_fwd_supported(x, conv.params, "average", SLOPE) if name == "c1" else
             D.block_fwd_pool_supported(x, conv.params, "average", SLOPE))
    if name in ("c1", "c2"):
        assert fused, f"{name}: the bench's fused conv+leaky+pool path must apply at 512^3"
    om = _meta(cout, od, ext // s, ext // s, split, NO_HALO)
    pm = _meta(cout, od // 2, ext // s // 2, ext // s // 2, split, (1, 1, 1))
    if fused:
        pooled, act = D.first_block_fwd(ctx, x, wd, conv.params, SLOPE, (1, 1, 1), tag=name)
        bits = _mask_bits(act, cout)
        band = np.abs(pre) <= 2.0 ** -11 * np.max(np.abs(pre))
        assert not np.any((bits != (act_ref >= 0)) & ~band), "sign mask disagrees outside the TF32 band"
        sign = np.where(band, bits, act_ref >= 0)
    else:
        act = D.dist_conv3d(ctx, x, wd, conv.params, NO_HALO, tag=name, leaky_slope=SLOPE)
        a_dev = act.numpy()
        assert rel(a_dev, act_ref) < RTOL, (name, "conv+leaky", rel(a_dev, act_ref))
        pooled = D.dist_pool3d(ctx, act, "average", (1, 1, 1), tag=f"p{name[1:]}")
        act_ref = a_dev  # teacher forcing: the pool sees the device activation
        sign = a_dev >= 0
    pool_ref = R(O._f64(O.pool3d, act_ref if not fused else R(O.leaky(pre, SLOPE)), "average", nargs=1))
    assert rel(pooled.numpy(), pool_ref) < RTOL, (name, "pooled fwd", rel(pooled.numpy(), pool_ref))
    # -------------------------------------------------------- backward
    up = DistTensor(pm, 0, zero=True)
    up.load_ncdhw(R(rng.uniform(-1, 1, (1, cout, od // 2, ext // s // 2, ext // s // 2)).astype(np.float32)))
    u_pool = up.numpy()
    g_ref = R(O.leaky_bwd(None, O.pool3d_bwd(pre, u_pool, "average"), SLOPE, mask=sign))
    wg = torch.zeros(cout, cin, 3, 3, 3, device="cuda")
    if name == "c1" and D.first_block_fast_path(net.layers[0], net.layers[1], act, up, xm):
        D.first_block_wgrad(ctx, x, act, up, SLOPE, "average", wg, tag=name)
        wg_ref = O._f64(O.k_conv3d_bwd_filter, xpad, g_ref, (s, s, s), (3, 3, 3))
        assert rel(wg.cpu().numpy(), wg_ref) < RTOL, (name, "wgrad (pooled, mask)", rel(wg.cpu().numpy(), wg_ref))
        assert _lib.load().vpx_fallback_count() == fb0, "a CUDA-core fallback ran"
        return
    g = D.dist_pool_leaky_bwd(act, up, SLOPE, "average", om, tag=f"{name}_act")
    g_dev = g.numpy()
    assert rel(g_dev, g_ref) < RTOL, (name, "pool+leaky bwd", rel(g_dev, g_ref))
    D.dist_conv3d_bwd_filter(ctx, x, g, conv.params, reduce=False, out=wg, tag=name)
    wg_ref = O._f64(O.k_conv3d_bwd_filter, xpad, g_dev, (s, s, s), (3, 3, 3))
    assert rel(wg.cpu().numpy(), wg_ref) < RTOL, (name, "wgrad", rel(wg.cpu().numpy(), wg_ref))
    gx = D.dist_conv3d_bwd_data(ctx, g, wd, conv.params, xm, tag=name)
    full = R(O._f64(O.k_conv3d_bwd_data, g_dev, R(w), (s, s, s), xpad.shape[2:]))
    ref = full[:, :, (0 if md else 1):full.shape[2] - (0 if md else 1), 1:-1, 1:-1]
    got = _full(gx)
    assert got.shape == ref.shape
    assert rel(got, ref) < RTOL, (name, "dgrad (frame incl. margins)", rel(got, ref))
    assert _lib.load().vpx_fallback_count() == fb0, f"{name}: a conv pass fell back to the CUDA-core kernels"
