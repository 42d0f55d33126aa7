"""Distributed layer ops on device-resident DistTensors.

Same operator names, argument order and semantics as the reference's
distributed layer library (reference pkg/src/voxpar/layers/distributed.py):
every op is collective over the ranks in its tensor's rank map, and gathering
the outputs reproduces the serial oracle.  Arithmetic runs in libvpx.so
(sm_100a); communication goes through comm.RankCtx (NCCL).  Outputs are
allocated with the halo margins their *consumer* needs (out_radii), so a
producer writes directly into the next conv's frame.

Weights are CUDA fp32 tensors in the reference layouts (conv OIDHW, deconv
(Cin,Cout,2,2,2)); parameter gradients are written into caller-provided
buffers (views of the flat gradient-allreduce bucket) when `out` is given.
"""

from __future__ import annotations

import ctypes
import os

import torch

from . import _lib
from .comm import RankCtx, halo_exchange, reverse_halo_exchange, copy_box
from .errors import NonDivisible, ShapeMismatch, Unsupported
from .frames import DistTensor, Frame, frame_desc, stream_ptr
from .geometry import DistTensorMeta, Shape5D, make_partition
from .timing import region

NO_HALO = (0, 0, 0)


class Workspace:
    """Grow-only device scratch (packed weights, reduction partials)."""

    def __init__(self):
        self._t = None

    def get(self, nbytes: int) -> torch.Tensor:
        nbytes = max(int(nbytes), 256)
        if self._t is None or self._t.numel() * 4 < nbytes:
            self._t = torch.empty((nbytes + 3) // 4 + 1024, dtype=torch.float32, device="cuda")
        return self._t


WS = Workspace()


def _group(meta: DistTensorMeta):
    return sorted(set(meta.rank_map))


def _out(meta: DistTensorMeta, shape: Shape5D, radii, grid_rank, zero=None) -> DistTensor:
    return DistTensor(make_partition(shape, meta.grid, radii, meta.rank_map), grid_rank, zero=zero)


def _like(t: DistTensor, radii=NO_HALO, channels=None) -> DistTensor:
    gs = t.meta.global_shape
    shape = gs if channels is None else Shape5D(gs.n, channels, gs.d, gs.h, gs.w)
    return _out(t.meta, shape, radii, t.grid_rank)


def _cubic(t):
    if len(set(t)) != 1:
        raise ShapeMismatch(f"only cubic kernels/strides are implemented, got {t}")
    return t[0]


# -------------------------------------------------------------- convolution

def _conv_flops(params, out_vox):
    k = _cubic(params.kernel)
    return 2 * k ** 3 * params.cin * params.cout * out_vox


def _overlap_d(ctx: RankCtx, meta: DistTensorMeta) -> bool:
    """Depth-only spatial split on several GPUs: the halo exchange can run on
    the communication stream while the planes that do not touch it compute."""
    # Off by default: measured on 4 B200s (graph replay) it does not pay --
    # the exchanges are latency-bound NCCL calls that the step has to wait for
    # either way.  VPX_OVERLAP=1 enables it.
    parts = meta.grid.spatial_parts
    return (ctx.size > 1 and parts[0] > 1 and parts[1] == 1 and parts[2] == 1
            and os.environ.get("VPX_OVERLAP") == "1" and torch.cuda.is_available())


OVERLAP_FREE_SMS = int(os.environ.get("VPX_OVERLAP_FREE_SMS", "16"))


class _sm_budget:
    """Leave OVERLAP_FREE_SMS SMs to the communication kernels while a
    convolution overlaps an exchange (vpx_set_sm_limit)."""

    def __enter__(self):
        n = torch.cuda.get_device_properties(torch.cuda.current_device()).multi_processor_count
        _lib.call("vpx_set_sm_limit", max(1, n - OVERLAP_FREE_SMS))

    def __exit__(self, *exc):
        _lib.call("vpx_set_sm_limit", 0)


def dist_conv3d(ctx: RankCtx, x: DistTensor, w: torch.Tensor, params, out_radii=NO_HALO,
                tag: str = "conv", leaky_slope: float = None) -> DistTensor:
    """Halo exchange, then the local tcgen05 implicit-GEMM conv on the frame
    (reference layers/distributed.py:42-69).  With leaky_slope set, the
    following LeakyReLU is fused into the epilogue and the result is
    leaky(conv(x)) (engine.forward uses this outside trace mode)."""
    meta = x.meta
    if tuple(meta.radii) != params.radii:
        raise ShapeMismatch(f"input partitioned with radii {meta.radii}, conv needs {params.radii}")
    if x.c != params.cin:
        raise ShapeMismatch(f"conv input channels {x.c} != {params.cin}")
    for name, e, p, s in zip("dhw", x.spatial, meta.grid.spatial_parts, params.stride):
        if p > 1 and e % s:
            raise NonDivisible(f"local extent {name}={e} not divisible by stride {s}")
    k, s = _cubic(params.kernel), _cubic(params.stride)
    gs = meta.global_shape
    y = _out(meta, Shape5D(gs.n, params.cout, *(-(-e // s) for e in gs.spatial)), out_radii, x.grid_rank)
    nb = _lib.load().vpx_conv3d_workspace_bytes(params.cin, params.cout, k, y.desc)
    ws = WS.get(nb)
    act, slope = int(leaky_slope is not None), float(leaky_slope or 0.0)

    def conv(zlo=None, zhi=None):
        if zlo is None:
            _lib.call("vpx_conv3d_fwd_act", x.ptr, x.desc, w.data_ptr(), k, s, y.ptr, y.desc, act, slope,
                      ws.data_ptr(), ws.numel() * 4, stream_ptr())
        else:
            _lib.call("vpx_conv3d_fwd_act_range", x.ptr, x.desc, w.data_ptr(), k, s, y.ptr, y.desc, act, slope,
                      zlo, zhi, ws.data_ptr(), ws.numel() * 4, stream_ptr())

    flops, nbytes = _conv_flops(params, y.voxels()), 4 * (x.voxels() * x.c + y.voxels() * y.c + w.numel())
    if _overlap_d(ctx, meta) and s == 1 and y.d >= 3:
        # exchange on the communication stream; output planes 1 .. d-2 read no
        # halo and run meanwhile, the two boundary planes after the join
        main, comm = torch.cuda.current_stream(), ctx.comm_stream()
        comm.wait_stream(main)
        with torch.cuda.stream(comm):
            halo_exchange(ctx, x)
        with region(f"{tag}.fwd", flops, nbytes):
            try:
                with _sm_budget():
                    conv(1, y.d - 1)
                main.wait_stream(comm)
                conv(0, 1)
                conv(y.d - 1, y.d)
            except Unsupported:
                main.wait_stream(comm)
                conv()
        return y
    halo_exchange(ctx, x)
    with region(f"{tag}.fwd", flops, nbytes):
        conv()
    return y


def dist_conv3d_bwd_data(ctx: RankCtx, u: DistTensor, w: torch.Tensor, params,
                         in_meta: DistTensorMeta, tag: str = "conv") -> DistTensor:
    """Input gradient over the halo-wide frame, then the adjoint exchange folds
    margin gradients into their owners (reference layers/distributed.py:72-82).
    The returned tensor keeps the frame; only its interior is meaningful."""
    k, s = _cubic(params.kernel), _cubic(params.stride)
    g = DistTensor(in_meta, u.grid_rank, zero=False)
    nb = _lib.load().vpx_conv3d_workspace_bytes(params.cin, params.cout, k, u.desc)
    ws = WS.get(nb)

    def dgrad(zlo=None, zhi=None):
        if zlo is None:
            _lib.call("vpx_conv3d_bwd_data", u.ptr, u.desc, w.data_ptr(), k, s, g.ptr, g.desc, ws.data_ptr(),
                      ws.numel() * 4, stream_ptr())
        else:
            _lib.call("vpx_conv3d_bwd_data_range", u.ptr, u.desc, w.data_ptr(), k, s, g.ptr, g.desc, zlo, zhi,
                      ws.data_ptr(), ws.numel() * 4, stream_ptr())

    flops, nbytes = _conv_flops(params, u.voxels()), 4 * (u.voxels() * u.c + g.t.numel() + w.numel())
    md = g.m[0]
    if _overlap_d(ctx, in_meta) and s == 1 and md == 1 and g.d >= 3:
        # boundary planes (and the margin planes that go to the neighbours)
        # first; the adjoint exchange then overlaps the interior planes
        main, comm = torch.cuda.current_stream(), ctx.comm_stream()
        with region(f"{tag}.dgrad", flops, nbytes):
            try:
                dgrad(-1, 1)
                dgrad(g.d - 1, g.d + 1)
            except Unsupported:
                dgrad()
                reverse_halo_exchange(ctx, in_meta, u.grid_rank, g)
                return g
            comm.wait_stream(main)
            with torch.cuda.stream(comm):
                reverse_halo_exchange(ctx, in_meta, u.grid_rank, g)
            with _sm_budget():
                dgrad(1, g.d - 1)
            main.wait_stream(comm)
        return g
    with region(f"{tag}.dgrad", flops, nbytes):
        dgrad()
    reverse_halo_exchange(ctx, in_meta, u.grid_rank, g)
    return g


def dist_conv3d_bwd_filter(ctx: RankCtx, x: DistTensor, u: DistTensor, params, reduce: bool = True,
                           out: torch.Tensor = None, tag: str = "conv") -> torch.Tensor:
    """Filter-gradient partial from the exchanged input frame; allreduced over
    the tensor's group when reduce=True (reference layers/distributed.py:85-98)."""
    k, s = _cubic(params.kernel), _cubic(params.stride)
    if out is None:
        out = torch.empty((params.cout, params.cin, k, k, k), dtype=torch.float32, device="cuda")
    nb = _lib.load().vpx_conv3d_workspace_bytes(params.cin, params.cout, k, u.desc)
    ws = WS.get(nb)
    with region(f"{tag}.wgrad", _conv_flops(params, u.voxels()),
                4 * (x.t.numel() + u.voxels() * u.c + out.numel())):
        _lib.call("vpx_conv3d_bwd_filter", x.ptr, x.desc, u.ptr, u.desc, k, s, out.data_ptr(), 0,
                  ws.data_ptr(), ws.numel() * 4, stream_ptr())
    if reduce:
        ctx.allreduce_sum_(out.view(-1), _group(x.meta))
    return out


def concat_wgrad_sources(x: DistTensor, sources, u: DistTensor, params):
    """The (ci0, source) list for taking a conv's filter gradient from the
    operands of the channel concat that produced its input x, or None.  Worth
    it when each source's channel count equals the conv's Cout (the
    grouped-voxel tcgen05 kernel then applies per source, while the concat as
    a whole would not) and no frame carries halo margins (the sources' margins
    are never exchanged)."""
    if sources is None or _cubic(params.kernel) != 3 or _cubic(params.stride) != 1:
        return None
    if _lib.load().vpx_get_precision() != 0 or any(u.m):  # the per-slice kernels are tcgen05 (TF32 mode)
        return None
    if any(t.c != u.c for t in sources) or sum(t.c for t in sources) != x.c:
        return None
    out, c0 = [], 0
    if not any(any(t.m) for t in (x,) + tuple(sources)):
        for t in sources:
            out.append((c0, t))
            c0 += t.c
        return out
    if x.m[2]:  # the grouped-voxel kernel reads whole W rows (no W margins)
        return None
    # spatially partitioned: x carries the exchanged halo margins, the concat
    # sources do not -- take each source's channel range from x itself, as a
    # dense frame with the same margins (one copy, ~1/4 of the slow
    # whole-concat kernel's time at U-Net's u1c1)
    for t in sources:
        sl = x.t[..., c0:c0 + t.c].contiguous()
        out.append((c0, Frame(x.n, t.c, x.d, x.h, x.w, x.m, tensor=sl)))
        c0 += t.c
    return out


def dist_conv3d_bwd_filter_slices(ctx: RankCtx, slices, u: DistTensor, params, out: torch.Tensor,
                                  tag: str = "conv") -> torch.Tensor:
    """Filter gradient of a conv whose input is a channel concat, one input
    channel slice per concat source (vpx_conv3d_bwd_filter_cslice)."""
    k, s = _cubic(params.kernel), _cubic(params.stride)
    nvox = u.voxels()
    with region(f"{tag}.wgrad", _conv_flops(params, nvox),
                4 * (sum(t.t.numel() for _, t in slices) + nvox * u.c + out.numel())):
        for ci0, t in slices:
            ws = WS.get(_lib.load().vpx_conv3d_workspace_bytes(t.c, params.cout, k, u.desc))
            _lib.call("vpx_conv3d_bwd_filter_cslice", t.ptr, t.desc, u.ptr, u.desc, k, s, out.data_ptr(), ci0,
                      params.cin, 0, ws.data_ptr(), ws.numel() * 4, stream_ptr())
    return out


# ------------------------------------------------------------------- deconv

def dist_deconv3d(ctx: RankCtx, x: DistTensor, w: torch.Tensor, out_radii=NO_HALO, tag: str = "deconv") -> DistTensor:
    """k2s2 transposed conv: purely local (reference layers/distributed.py:103-112)."""
    if tuple(x.meta.radii) != NO_HALO:
        raise ShapeMismatch("deconv input must carry no halos")
    gs = x.meta.global_shape
    y = _out(x.meta, Shape5D(gs.n, w.shape[1], 2 * gs.d, 2 * gs.h, 2 * gs.w), out_radii, x.grid_rank)
    with region(f"{tag}.fwd", 2 * 8 * x.voxels() * x.c * y.c, 4 * (x.voxels() * x.c + y.voxels() * y.c)):
        ws = WS.get(_lib.load().vpx_deconv_workspace_bytes(x.c, y.c))
        _lib.call("vpx_deconv_fwd", x.ptr, x.desc, w.data_ptr(), y.ptr, y.desc, ws.data_ptr(), ws.numel() * 4,
                  stream_ptr())
    return y


def dist_deconv3d_bwd_data(ctx: RankCtx, u: DistTensor, w: torch.Tensor, in_meta, tag: str = "deconv") -> DistTensor:
    g = DistTensor(in_meta, u.grid_rank, zero=False)
    with region(f"{tag}.dgrad", 2 * u.voxels() * u.c * g.c, 4 * (u.voxels() * u.c + g.voxels() * g.c)):
        ws = WS.get(_lib.load().vpx_deconv_workspace_bytes(g.c, u.c))
        _lib.call("vpx_deconv_bwd_data", u.ptr, u.desc, w.data_ptr(), g.ptr, g.desc, ws.data_ptr(), ws.numel() * 4,
                  stream_ptr())
    return g


def dist_deconv3d_bwd_filter(ctx: RankCtx, x: DistTensor, u: DistTensor, reduce: bool = True,
                             out: torch.Tensor = None, tag: str = "deconv") -> torch.Tensor:
    if out is None:
        out = torch.empty((x.c, u.c, 2, 2, 2), dtype=torch.float32, device="cuda")
    ws = WS.get(_lib.load().vpx_deconv_workspace_bytes(x.c, u.c))
    with region(f"{tag}.wgrad", 2 * u.voxels() * u.c * x.c, 4 * (u.voxels() * u.c + x.voxels() * x.c)):
        _lib.call("vpx_deconv_bwd_filter", x.ptr, x.desc, u.ptr, u.desc, out.data_ptr(), 0, ws.data_ptr(),
                  stream_ptr())
    if reduce:
        ctx.allreduce_sum_(out.view(-1), _group(x.meta))
    return out


# ------------------------------------------------------------------ pooling

def dist_pool3d(ctx: RankCtx, x: DistTensor, kind: str = "average", out_radii=NO_HALO,
                tag: str = "pool") -> DistTensor:
    """2^3 stride-2 pooling; windows never straddle blocks (reference
    layers/distributed.py:132-140)."""
    if tuple(x.meta.radii) != NO_HALO:
        raise ShapeMismatch("pool input must carry no halos")
    if kind not in ("average", "max"):
        raise ShapeMismatch(f"unknown pool kind {kind!r}")
    gs = x.meta.global_shape
    y = _out(x.meta, Shape5D(gs.n, gs.c, gs.d // 2, gs.h // 2, gs.w // 2), out_radii, x.grid_rank)
    with region(f"{tag}.fwd", 0, 4 * (x.voxels() * x.c + y.voxels() * y.c)):
        _lib.call("vpx_pool_fwd", x.ptr, x.desc, y.ptr, y.desc, int(kind == "max"), stream_ptr())
    return y


def dist_pool3d_bwd(ctx: RankCtx, x: DistTensor, u: DistTensor, kind: str, in_meta,
                    tag: str = "pool") -> DistTensor:
    g = DistTensor(in_meta, u.grid_rank, zero=False)
    nb = 4 * (u.voxels() * u.c + g.voxels() * g.c + (x.voxels() * x.c if kind == "max" else 0))
    with region(f"{tag}.bwd", 0, nb):
        _lib.call("vpx_pool_bwd", x.ptr, x.desc, u.ptr, u.desc, g.ptr, g.desc, int(kind == "max"), stream_ptr())
    return g


# ---------------------------------------------------------------- batchnorm

class BNState:
    """Per-channel batch-norm state (reference layers/reference.py:39-57);
    gamma/beta alias the optimizer's parameter storage."""

    def __init__(self, gamma, beta, running_mean=None, running_var=None, eps=1e-5, momentum=0.9):
        c = gamma.numel()
        self.gamma, self.beta = gamma, beta
        self.running_mean = running_mean if running_mean is not None else torch.zeros(c, device="cuda")
        self.running_var = running_var if running_var is not None else torch.ones(c, device="cuda")
        self.eps, self.momentum = eps, momentum


def _bn_sums(x, u, mean, inv, mode):
    c = x.c
    out = torch.empty(2 * c, dtype=torch.float32, device="cuda")
    ws = WS.get(_lib.load().vpx_bn_workspace_bytes(c))
    _lib.call("vpx_bn_sums", x.ptr, x.desc, u.ptr if u is not None else 0, u.desc if u is not None else 0,
              mean.data_ptr() if mean is not None else 0, inv.data_ptr() if inv is not None else 0, mode,
              out.data_ptr(), ws.data_ptr(), stream_ptr())
    return out


def dist_batchnorm(ctx: RankCtx, x: DistTensor, state: BNState, mode: str = "train",
                   out_radii=NO_HALO, tag: str = "bn", leaky_slope: float = None):
    """Local (sum x, sum x^2) -> allreduce(2C) over the tensor's whole rank
    group -> normalise (reference layers/distributed.py:152-180).  Returns
    (y, cache); the cache keeps x and the batch statistics (xhat is recomputed).
    With leaky_slope the following LeakyReLU runs in the same pass (y is then
    the activation; its signs are the normalised values' signs)."""
    gs = x.meta.global_shape
    c = gs.c
    mean = torch.empty(c, dtype=torch.float32, device="cuda")
    inv = torch.empty(c, dtype=torch.float32, device="cuda")
    if mode == "train":
        count = gs.n * gs.d * gs.h * gs.w
        with region(f"{tag}.stats", 0, 4 * x.voxels() * c):
            sums = _bn_sums(x, None, None, None, 0)
        ctx.allreduce_sum_(sums, _group(x.meta))
        _lib.call("vpx_bn_stats", sums.data_ptr(), c, float(count), float(state.eps), float(state.momentum),
                  mean.data_ptr(), inv.data_ptr(), state.running_mean.data_ptr(),
                  state.running_var.data_ptr(), stream_ptr())
    elif mode == "eval":
        count = 0
        mean.copy_(state.running_mean)
        inv.copy_(torch.rsqrt(state.running_var + state.eps))
    else:
        raise ShapeMismatch(f"unknown bn mode {mode!r}")
    y = _out(x.meta, gs, out_radii, x.grid_rank)
    with region(f"{tag}.fwd", 0, 8 * x.voxels() * c):
        if leaky_slope is not None:
            _lib.call("vpx_bn_apply_leaky", x.ptr, x.desc, mean.data_ptr(), inv.data_ptr(), state.gamma.data_ptr(),
                      state.beta.data_ptr(), float(leaky_slope), y.ptr, y.desc, stream_ptr())
        else:
            _lib.call("vpx_bn_apply", x.ptr, x.desc, mean.data_ptr(), inv.data_ptr(), state.gamma.data_ptr(),
                      state.beta.data_ptr(), y.ptr, y.desc, stream_ptr())
    return y, (x, mean, inv, count)


def dist_batchnorm_bwd(ctx: RankCtx, u: DistTensor, state: BNState, cache, in_meta,
                       dgamma: torch.Tensor = None, dbeta: torch.Tensor = None, tag: str = "bn"):
    """(dx, dgamma partial, dbeta partial); the two reduction terms are
    allreduced for dx, the parameter gradients stay rank-local partials
    (reference layers/distributed.py:183-201)."""
    x, mean, inv, count = cache
    c = x.c
    with region(f"{tag}.bwd_stats", 0, 8 * x.voxels() * c):
        local = _bn_sums(x, u, mean, inv, 1)  # [sum u, sum u*xhat]
    if dgamma is None:
        dgamma = torch.empty(c, dtype=torch.float32, device="cuda")
    if dbeta is None:
        dbeta = torch.empty(c, dtype=torch.float32, device="cuda")
    dbeta.copy_(local[:c])
    dgamma.copy_(local[c:])
    ctx.allreduce_sum_(local, _group(u.meta))
    g = DistTensor(in_meta, u.grid_rank, zero=False)
    with region(f"{tag}.bwd", 0, 12 * x.voxels() * c):
        _lib.call("vpx_bn_bwd_apply", x.ptr, x.desc, u.ptr, u.desc, mean.data_ptr(), inv.data_ptr(),
                  state.gamma.data_ptr(), local.data_ptr(), float(count), g.ptr, g.desc, stream_ptr())
    return g, dgamma, dbeta


# ---------------------------------------------------------------- pointwise

def dist_leaky_relu(x: DistTensor, slope: float, out_radii=NO_HALO, tag: str = "leaky") -> DistTensor:
    y = _out(x.meta, x.meta.global_shape, out_radii, x.grid_rank)
    with region(f"{tag}.fwd", 0, 8 * x.voxels() * x.c):
        _lib.call("vpx_leaky_fwd", x.ptr, x.desc, y.ptr, y.desc, float(slope), stream_ptr())
    return y


def dist_leaky_relu_bwd(x: DistTensor, u: DistTensor, slope: float, in_meta, tag: str = "leaky") -> DistTensor:
    g = DistTensor(in_meta, u.grid_rank, zero=False)
    with region(f"{tag}.bwd", 0, 12 * x.voxels() * x.c):
        _lib.call("vpx_leaky_bwd", x.ptr, x.desc, u.ptr, u.desc, g.ptr, g.desc, float(slope), stream_ptr())
    return g


def dist_pool_leaky_bwd(y: DistTensor, u: DistTensor, slope: float, kind: str, in_meta,
                        tag: str = "leaky") -> DistTensor:
    """Backward of leaky -> pool in one pass: g = leaky'(y) * pool_bwd(y, u)
    (reference layers/distributed.py:141-147 then :211-214); y is the LeakyReLU
    output, which is also the pool input."""
    g = DistTensor(in_meta, u.grid_rank, zero=False)
    if isinstance(y, MaskFrame):  # the forward ran fused: signs from the mask (average pool)
        if kind != "average":
            raise ShapeMismatch("mask backward needs average pooling")
        with region(f"{tag}.bwd", 0, 4 * (u.voxels() * u.c + y.voxels() * y.c) + y.voxels() * y.c // 8):
            _lib.call("vpx_pool_leaky_bwd_mask", y.ptr, y.desc, u.ptr, u.desc, g.ptr, g.desc, float(slope),
                      stream_ptr())
        return g
    with region(f"{tag}.bwd", 0, 4 * (u.voxels() * u.c + 2 * y.voxels() * y.c)):
        _lib.call("vpx_pool_leaky_bwd", y.ptr, y.desc, u.ptr, u.desc, g.ptr, g.desc, float(slope),
                  int(kind == "max"), stream_ptr())
    return g


def dist_concat_channels(a: DistTensor, b: DistTensor, out_radii=NO_HALO, tag: str = "concat") -> DistTensor:
    if a.meta.grid != b.meta.grid or a.meta.rank_map != b.meta.rank_map:
        raise ShapeMismatch("concat operands must share a partition layout")
    ga, gb = a.meta.global_shape, b.meta.global_shape
    if (ga.n, ga.d, ga.h, ga.w) != (gb.n, gb.d, gb.h, gb.w):
        raise ShapeMismatch(f"concat shapes {ga} vs {gb}")
    y = _out(a.meta, Shape5D(ga.n, ga.c + gb.c, ga.d, ga.h, ga.w), out_radii, a.grid_rank)
    with region(f"{tag}.fwd", 0, 8 * y.voxels() * y.c):
        _lib.call("vpx_concat", a.ptr, a.desc, b.ptr, b.desc, y.ptr, y.desc, stream_ptr())
    return y


def dist_concat_bwd(u: DistTensor, c_main: int, main_meta, skip_meta, skip_grad: DistTensor = None,
                    tag: str = "concat"):
    """Split a concat's gradient into (main part, skip part); the skip part is
    accumulated into skip_grad when given (reference engine.py:432-438)."""
    ga = DistTensor(main_meta, u.grid_rank, zero=False)
    acc = skip_grad is not None
    gb = skip_grad if acc else DistTensor(skip_meta, u.grid_rank, zero=False)
    with region(f"{tag}.bwd", 0, 4 * u.voxels() * u.c * (3 if acc else 2)):
        _lib.call("vpx_split", u.ptr, u.desc, ga.ptr, ga.desc, gb.ptr, gb.desc, int(acc), stream_ptr())
    return ga, gb


def add_into(dst: DistTensor, src: DistTensor) -> DistTensor:
    _lib.call("vpx_add", src.ptr, src.desc, dst.ptr, dst.desc, stream_ptr())
    return dst


# ------------------------------------------------------------------- losses

def dist_mse(ctx: RankCtx, pred, target, global_size: int, group=None):
    """MSE over rank-local rows (pred None -> contributes 0); loss identical on
    every rank (reference layers/distributed.py:257-270).  Device tensors."""
    if pred is None:
        local = torch.zeros(1, dtype=torch.float64, device="cuda")
        diff = None
    else:
        if pred.shape != target.shape:
            raise ShapeMismatch(f"mse shapes {tuple(pred.shape)} vs {tuple(target.shape)}")
        diff = pred - target
        local = (diff.double() * diff.double()).sum().reshape(1)
    ctx.allreduce_sum_(local, group)
    return local / global_size, (None if diff is None else diff * (2.0 / global_size))


def dist_cross_entropy(ctx: RankCtx, pred: DistTensor, labels: torch.Tensor, count: int, group=None,
                       nparts: int = 512):
    """Per-voxel softmax cross entropy over a spatially partitioned prediction;
    only the scalar is allreduced (reference layers/distributed.py:273-293).
    labels: int64 CUDA tensor (n_local, d, h, w) of this rank's block."""
    g = DistTensor(make_partition(pred.meta.global_shape, pred.meta.grid, NO_HALO, pred.meta.rank_map),
                   pred.grid_rank, zero=False)
    part = torch.empty(nparts, dtype=torch.float64, device="cuda")
    with region("loss.xent", 0, 4 * pred.voxels() * pred.c * 2 + 8 * pred.voxels()):
        _lib.call("vpx_xent", pred.ptr, pred.desc, labels.data_ptr(), float(count), g.ptr, g.desc,
                  part.data_ptr(), nparts, stream_ptr())
        local = part.sum().reshape(1)
    ctx.allreduce_sum_(local, group)
    return local / count, g


# ------------------------------------------------------------ redistribution

def redistribute(ctx: RankCtx, x, src_meta: DistTensorMeta, dst_meta: DistTensorMeta, zero=None):
    """Move a tensor between partition layouts, values preserved exactly
    (reference layers/distributed.py:298-368).  Collective over the union of
    both rank maps; x is this rank's source DistTensor (None if it holds no
    source part).  Returns the destination DistTensor or None."""
    if src_meta.global_shape != dst_meta.global_shape:
        raise ShapeMismatch(f"redistribute shapes differ: {src_meta.global_shape} vs {dst_meta.global_shape}")
    me = ctx.rank
    src_gr = src_meta.rank_map.index(me) if me in src_meta.rank_map else None
    dst_gr = dst_meta.rank_map.index(me) if me in dst_meta.rank_map else None
    if src_gr is not None and x is None:
        raise ShapeMismatch(f"rank {me} holds a source block but passed none")
    out = DistTensor(dst_meta, dst_gr, zero=zero) if dst_gr is not None else None
    ops, unpacks, locals_ = [], [], []
    for a in range(src_meta.grid.size):
        a_lo, a_hi = src_meta.sample_range(src_meta.group_of(a))
        ra = src_meta.region(a)
        for b in range(dst_meta.grid.size):
            b_lo, b_hi = dst_meta.sample_range(dst_meta.group_of(b))
            lo, hi = max(a_lo, b_lo), min(a_hi, b_hi)
            if hi <= lo:
                continue
            rb = dst_meta.region(b)
            ov = ra.intersect(rb)
            if ov is None:
                continue
            src_rank, dst_rank = src_meta.fabric_rank(a), dst_meta.fabric_rank(b)
            if me not in (src_rank, dst_rank):
                continue
            ext = ov.extent
            if a == src_gr:
                m = x.m
                sbox = (lo - a_lo,) + tuple(o - r + mm for o, r, mm in zip(ov.offset, ra.offset, m)) + (hi - lo,) + ext
            if b == dst_gr:
                m = out.m
                dbox = (lo - b_lo,) + tuple(o - r + mm for o, r, mm in zip(ov.offset, rb.offset, m)) + (hi - lo,) + ext
            numel = (hi - lo) * ext[0] * ext[1] * ext[2] * src_meta.global_shape.c
            if src_rank == dst_rank == me:
                buf = torch.empty(numel, dtype=torch.float32, device="cuda")
                copy_box(x, sbox, buf, 0)
                copy_box(out, dbox, buf, 1)
            elif src_rank == me:
                buf = torch.empty(numel, dtype=torch.float32, device="cuda")
                copy_box(x, sbox, buf, 0)
                ops.append(("send", dst_rank, buf))
            else:
                buf = torch.empty(numel, dtype=torch.float32, device="cuda")
                ops.append(("recv", src_rank, buf))
                unpacks.append((dbox, buf))
    ctx.exchange(ops)
    for dbox, buf in unpacks:
        copy_box(out, dbox, buf, 1)
    return out


# ------------------------------------------------- first-block fast path

class MaskFrame:
    """Sign mask of the first block's LeakyReLU output: int16 [n][d][h][w],
    bit co set where the stored activation is >= 0 (the backward needs only
    the sign because slope > 0).  Stands in for the activation frame in the
    stash when the forward ran fused (vpx_conv3d_fwd_leaky_pool_c4)."""

    def __init__(self, n, c, d, h, w):
        self.n, self.c, self.d, self.h, self.w = n, c, d, h, w
        dt = {8: torch.int8, 16: torch.int16, 32: torch.int32}[c]  # c/8 bytes per voxel
        self.t = torch.empty((n, d, h, w), dtype=dt, device="cuda")
        self._desc = frame_desc(n, c, d, h, w)

    @property
    def ptr(self):
        return self.t.data_ptr()

    @property
    def desc(self):
        return ctypes.addressof(self._desc)

    def voxels(self):
        return self.n * self.d * self.h * self.w


def first_block_fwd_supported(x: DistTensor, conv_params, pool_kind: str, slope: float) -> bool:
    """conv(4 -> 16, k3 s1) -> leaky(0 < slope <= 1) -> average pool in one
    kernel (TF32 mode)."""
    if pool_kind != "average" or _lib.load().vpx_get_precision() != 0 or not 0.0 < slope <= 1.0:
        return False
    if conv_params.cin != 4 or conv_params.cout != 16:
        return False
    if tuple(conv_params.kernel) != (3, 3, 3) or tuple(conv_params.stride) != (1, 1, 1):
        return False
    # the backward (first_block_wgrad with the mask) covers W in 128..512 per rank
    return x.m[2] == 0 and x.w in (128, 256, 512) and x.d % 2 == 0 and x.h % 2 == 0


FUSED_POOL_BLOCKS = ((16, 32), (16, 16))  # conv_rowh.cu conv_rowh_pool_kernel instances


def block_fwd_pool_supported(x: DistTensor, conv_params, pool_kind: str, slope: float) -> bool:
    """conv(k3 s1) -> leaky -> average pool of a later block (not the first)
    in one kernel: pooled output + sign mask; the backward reads the mask
    (vpx_pool_leaky_bwd_mask) instead of the activation."""
    if pool_kind != "average" or _lib.load().vpx_get_precision() != 0 or not 0.0 < slope <= 1.0:
        return False
    if (conv_params.cin, conv_params.cout) not in FUSED_POOL_BLOCKS:
        return False
    if tuple(conv_params.kernel) != (3, 3, 3) or tuple(conv_params.stride) != (1, 1, 1):
        return False
    return x.m[2] == 0 and x.w % 128 == 0 and x.d % 2 == 0 and x.h % 2 == 0


def first_block_fwd(ctx: RankCtx, x: DistTensor, w: torch.Tensor, conv_params, slope: float, out_radii,
                    tag: str = "c1"):
    """Pooled output + sign mask of conv -> leaky -> avg pool in one kernel
    (conv_c1fwd.cu for Cin 4 -> 16, conv_rowh.cu's pooled variant otherwise)."""
    halo_exchange(ctx, x)
    gs = x.meta.global_shape
    pooled = _out(x.meta, Shape5D(gs.n, conv_params.cout, gs.d // 2, gs.h // 2, gs.w // 2), out_radii,
                  x.grid_rank)
    mask = MaskFrame(x.n, conv_params.cout, x.d, x.h, x.w)
    yfr = frame_desc(x.n, conv_params.cout, x.d, x.h, x.w)
    ws = WS.get(_lib.load().vpx_conv3d_workspace_bytes(x.c, conv_params.cout, 3, ctypes.addressof(yfr)))
    nvox = x.voxels()
    with region(f"{tag}.fwd", _conv_flops(conv_params, nvox),
                4 * (x.voxels() * x.c + pooled.voxels() * pooled.c) + 2 * nvox):
        _lib.call("vpx_conv3d_fwd_leaky_pool", x.ptr, x.desc, w.data_ptr(), float(slope), pooled.ptr,
                  pooled.desc, mask.ptr, ws.data_ptr(), ws.numel() * 4, stream_ptr())
    return pooled, mask

def first_block_fast_path(conv, act, y: DistTensor, u: DistTensor, x_meta) -> bool:
    """True when the first conv block (Cin=4 -> 16, LeakyReLU, 2^3 pool) can
    take the fused backward: blocked pool/leaky backward + dense c1 wgrad."""
    if conv.kind != "conv" or act.kind != "leaky" or conv.params.cin != 4 or conv.params.cout != 16:
        return False
    if tuple(conv.params.kernel) != (3, 3, 3) or tuple(conv.params.stride) != (1, 1, 1):
        return False
    if not isinstance(y, MaskFrame) and _lib.load().vpx_get_precision() != 0:
        return False  # the fast-path kernels are tcgen05 (TF32); FP32 mode takes the CUDA-core path
    # frames may carry D/H halo margins (the pooled gradient arrives in the
    # next conv's dgrad frame); the dense x view needs no W margin
    return y.w in (64, 128, 256, 512) and x_meta.margins()[2] == 0


def first_block_wgrad(ctx: RankCtx, x: DistTensor, y: DistTensor, u_pool: DistTensor, slope: float,
                      pool_kind: str, out: torch.Tensor, tag: str = "c1"):
    """c1 filter gradient straight from the pooled gradient (see
    vpx_pool_leaky_bwd_blocked / vpx_conv3d_bwd_filter_c4 in include/vpx.h)."""
    nvox = y.voxels()
    ufr = frame_desc(y.n, y.c, y.d, y.h, y.w)
    ws = WS.get(_lib.load().vpx_conv3d_workspace_bytes(x.c, y.c, 3, ctypes.addressof(ufr)))
    flops = 2 * 27 * x.c * y.c * nvox
    if isinstance(y, MaskFrame):
        # forward ran fused: the LeakyReLU signs come from the mask
        with region(f"{tag}.wgrad", flops, 4 * (x.voxels() * x.c + u_pool.voxels() * u_pool.c) + 2 * nvox):
            _lib.call("vpx_conv3d_bwd_filter_c4_pooled_mask", x.ptr, x.desc, y.ptr, y.desc, u_pool.ptr,
                      u_pool.desc, float(slope), out.data_ptr(), 0, ws.data_ptr(), ws.numel() * 4, stream_ptr())
        return out
    if pool_kind != "max" and _lib.load().vpx_get_precision() == 0:
        # one kernel: pooled gradient -> u (in TMEM) -> filter gradient
        with region(f"{tag}.wgrad", flops, 4 * (x.voxels() * x.c + nvox * y.c + u_pool.voxels() * u_pool.c)):
            _lib.call("vpx_conv3d_bwd_filter_c4_pooled", x.ptr, x.desc, y.ptr, y.desc, u_pool.ptr, u_pool.desc,
                      float(slope), 0, out.data_ptr(), 0, ws.data_ptr(), ws.numel() * 4, stream_ptr())
        return out
    gb = WS2.get(nvox * y.c * 4)
    with region(f"{tag}_act.bwd", 0, 4 * (u_pool.voxels() * u_pool.c + 2 * nvox * y.c)):
        _lib.call("vpx_pool_leaky_bwd_blocked", y.ptr, y.desc, u_pool.ptr, u_pool.desc, gb.data_ptr(),
                  float(slope), int(pool_kind == "max"), stream_ptr())
    with region(f"{tag}.wgrad", flops, 4 * (x.voxels() * x.c + nvox * y.c + out.numel())):
        _lib.call("vpx_conv3d_bwd_filter_c4", x.ptr, x.desc, gb.data_ptr(), ctypes.addressof(ufr), out.data_ptr(),
                  0, ws.data_ptr(), ws.numel() * 4, stream_ptr())
    return out


WS2 = Workspace()
